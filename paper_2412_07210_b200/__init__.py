"""paper_2412_07210_b200 -- B200-native (sm_100a) EDiT layer-wise sync with pseudo-gradient penalty.

The hot path (Alg. 2) runs in libedit_sync.so (csrc/, C ABI in include/edit_sync.h);
this package is the thin Python binding around it.
"""
from .edit_sync import (EDIT_BF16, EDIT_F32, NO_AE, NO_GC, NO_WA, EditSync, EditSyncError,  # noqa: F401
                        LayerStats, Trigger, broadcast_unique_id, get_unique_id, load_library)

__all__ = ["EditSync", "EditSyncError", "LayerStats", "Trigger", "broadcast_unique_id", "get_unique_id", "load_library",
           "NO_AE", "NO_WA", "NO_GC", "EDIT_BF16", "EDIT_F32"]
