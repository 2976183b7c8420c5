"""CPU checks of the C-ABI library: it builds for sm_100a, loads, and exports every
symbol include/edit_sync.h declares.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names += re.findall(r"^\s*(?:const\s+)?[\w\*]+\s+\**(edit_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2412_07210_b200 import build
    return build.build()


def test_header_declares_the_north_star_entry_points():
    names = _declared_functions()
    for required in ("edit_sync_init", "edit_layer_sync", "edit_sync_stats"):
        assert required in names


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(edit_\w+)\b", out))
    missing = [n for n in _declared_functions() if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(lib_path)
    for n in _declared_functions():
        assert hasattr(lib, n)


def test_binding_names_match_header(lib_path):
    from paper_2412_07210_b200 import edit_sync
    assert sorted(edit_sync.EXPORTED) == _declared_functions()
    lib = edit_sync.load_library()
    assert b"sm_100a" in lib.edit_sync_version()


def test_library_is_sm100a_code(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header(lib_path):
    # compile a tiny C program against the header and compare sizes/offsets with ctypes
    from paper_2412_07210_b200 import edit_sync as es
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "edit_sync.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(edit_sync_config_t), sizeof(edit_layer_stats_t),
         offsetof(edit_layer_stats_t, G_bar), offsetof(edit_layer_stats_t, ema_count),
         offsetof(edit_sync_config_t, flags), sizeof(edit_ema_t));
  return 0;
}'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    want = [ctypes.sizeof(es.Config), ctypes.sizeof(es.LayerStatsC), es.LayerStatsC.G_bar.offset,
            es.LayerStatsC.ema_count.offset, es.Config.flags.offset, es.EMA_DTYPE.itemsize]
    assert got == want


def test_validation_without_gpu(lib_path):
    # argument validation runs before any CUDA call
    from paper_2412_07210_b200 import edit_sync as es
    lib = es.load_library()
    numel = (ctypes.c_int64 * 2)(10, 20)
    bad = [dict(shard_dim=0), dict(sync_dim=9), dict(rank=4), dict(outer_lr=0.0), dict(outer_momentum=1.0),
           dict(clip_threshold=-1.0), dict(clip_eps=0.0), dict(ema_alpha=0.0), dict(anomaly_threshold=0.0),
           dict(param_dtype=7), dict(flags=8), dict(num_layers=0), dict(algo=2)]
    base = dict(shard_dim=2, sync_dim=2, rank=0, device=0, num_layers=2, param_dtype=0, layer_numel=numel,
                outer_lr=0.8, outer_momentum=0.85, clip_threshold=10.0, clip_eps=1e-6, anomaly_threshold=3.0,
                ema_alpha=0.02, ema_warmup_rounds=10, flags=0, algo=0)
    nb = ctypes.c_size_t()
    assert lib.edit_sync_workspace_bytes(ctypes.byref(es.Config(**base)), ctypes.byref(nb)) == 0
    assert nb.value > 20 * 4
    for b in bad:
        cfg = es.Config(**{**base, **b})
        assert lib.edit_sync_workspace_bytes(ctypes.byref(cfg), ctypes.byref(nb)) == 1, b
        assert lib.edit_sync_last_error()
    assert lib.edit_layer_sync(None, 0, None, None, None, None) == 1
