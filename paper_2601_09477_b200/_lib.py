"""ctypes binding of the in-tree C-ABI library ``_smm_b200.so``.

The library is the only compute path: if it is missing, or no CUDA device is
visible, every hot-path call raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import InvalidParameterError, SketchmmError

_HERE = Path(__file__).resolve().parent
# SMM_LIB selects an experimental in-tree build (tools/variant.sh); default is the product library
LIB_PATH = _HERE / os.environ.get("SMM_LIB", "_smm_b200.so")

SMM_OK = 0
SMM_ERR_INVALID = 1
SMM_ERR_CUDA = 2
SMM_ERR_WORKSPACE = 3
VARIANT = {"fft": 0, "fwht": 1}
MAX_DEPTH = 63  # repetitions per kernel launch (SMM_MAX_DEPTH)
MAX_DEPTH_TOTAL = 511  # deepest sketch the device path handles (SMM_MAX_DEPTH_TOTAL)
FLAG_ACCUMULATE = 0x100

EXPORTS = (
    "smm_abi_version",
    "smm_last_error",
    "smm_hash_tables",
    "smm_compress_kernel",
    "smm_compress_workspace",
    "smm_compress_accumulate",
    "smm_compress_workspace_ex",
    "smm_compress_accumulate_ex",
    "smm_finalize",
    "smm_extract_workspace",
    "smm_extract",
    "smm_hh_pairs",
    "smm_query",
    "smm_kernel_launches",
    "smm_kernel_timing",
    "smm_kernel_timing_read",
    "smm_transpose",
    "smm_copy2d",
    "smm_fwht_batched",
    "smm_fft_batched",
)

_lock = threading.Lock()
_lib = None


class ExtensionMissingError(SketchmmError, RuntimeError):
    """The CUDA extension is not built / not loadable (no CPU fallback exists)."""


def load():
    """Load and type the shared library (idempotent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ExtensionMissingError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the sketched-product path has no CPU fallback)"
            )
        lib = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        I = ctypes.c_int
        I64 = ctypes.c_int64
        D = ctypes.c_double
        sig = {
            "smm_abi_version": ([], I),
            "smm_last_error": ([], ctypes.c_char_p),
            "smm_hash_tables": ([P, I, I, I, I64, P, P, P], I),
            "smm_compress_kernel": ([I, I, I, I64, I64, I64, I64, P], I),
            "smm_compress_workspace": ([I, I, I, I64, I64, I64, I64, P], I),
            "smm_compress_accumulate": ([I, P, I64, P, I64, I64, I64, I64, I64, P, I, I, P, P, I64, P], I),
            "smm_compress_workspace_ex": ([I, I, I, I64, I64, I64, I64, I, I, P], I),
            "smm_compress_accumulate_ex": ([I, P, I64, I, P, I64, I, I64, I64, I64, I64, P, I, I, P, P, I64, P], I),
            "smm_finalize": ([I, P, P, I, I, P], I),
            "smm_extract_workspace": ([I, I64, I64, I64, I64, P], I),
            "smm_extract": ([I, P, P, I, I, I64, I64, I64, I64, P, I64, D, I, P, I64, P, P, I64, P], I),
            "smm_hh_pairs": ([P, I64, I64, I64, P, I64, P], I),
            "smm_kernel_launches": ([], I64),
            "smm_kernel_timing": ([I], I),
            "smm_kernel_timing_read": ([I, P, P], I),
            "smm_transpose": ([P, I64, I64, I64, P, I64, P], I),
            "smm_copy2d": ([P, I64, P, I64, I64, I64, P], I),
            "smm_query": ([I, P, P, I, I, I64, I64, P, I64, P, P, P], I),
            "smm_fwht_batched": ([P, I64, I, D, P], I),
            "smm_fft_batched": ([P, I64, I, I, D, P], I),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C status to the reference's exception types."""
    if rc == SMM_OK:
        return
    msg = (load().smm_last_error() or b"").decode(errors="replace")
    if rc == SMM_ERR_INVALID:
        raise InvalidParameterError(msg)
    raise RuntimeError(f"sketchmm_b200 CUDA error ({rc}): {msg}")


def exported_symbols() -> list[str]:
    lib = load()
    return [name for name in EXPORTS if hasattr(lib, name)]
