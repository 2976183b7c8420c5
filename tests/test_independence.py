"""The oracle and the CUDA path share no code (task rule): neither side includes,
imports or links the other, and the product package never touches oracle/."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sources(d, exts):
    for base, _, files in os.walk(os.path.join(ROOT, d)):
        if "__pycache__" in base:
            continue
        for f in files:
            if f.endswith(exts):
                yield os.path.join(base, f)


def _code(path):
    """Source text without comments/docstrings (mentions in prose are allowed)."""
    s = open(path, encoding="utf-8").read()
    if path.endswith(".py"):
        s = re.sub(r'("""|\'\'\')(?:.|\n)*?\1', "", s)
        s = re.sub(r"#.*", "", s)
    else:
        s = re.sub(r"/\*(?:.|\n)*?\*/", "", s)
        s = re.sub(r"//.*", "", s)
    return s


def test_oracle_does_not_reference_the_cuda_path():
    for p in _sources("oracle", (".py", ".c", ".h")):
        code = _code(p)
        for bad in ("paper_2412_07210_b200", "csrc", "edit_sync", "libedit_sync", "device_common", "internal.h"):
            assert bad not in code, f"{p} references {bad}"


def test_product_package_does_not_reference_the_oracle():
    for p in _sources("paper_2412_07210_b200", (".py", ".cu", ".cuh", ".cpp", ".h")):
        code = _code(p)
        assert not re.search(r"\boracle\b", code), f"{p} references the oracle"
    for p in _sources("include", (".h",)):
        assert not re.search(r"\boracle\b", _code(p)), p


def test_input_generators_hold_no_method_arithmetic():
    # synth/ (shared by both sides) draws inputs only: no norms, weights, clip or outer step
    for p in _sources("synth", (".py",)):
        code = _code(p)
        for bad in ("softmax", "nesterov", "clip", "sqrt(sum", ".norm(", "exp(-"):
            assert bad not in code.lower(), f"{p} contains {bad}"
