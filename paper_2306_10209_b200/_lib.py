"""ctypes binding of libzpp.so (the C ABI declared in include/zpp.h).

The product path has no fallback: if the shared library is missing or fails to
load, importing an op raises immediately.  ``load()`` is lazy so that host-only
code (configs, partitions, ledgers) stays importable on machines without the
library.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, DeviceError, IntegrityError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZPP_LIB", os.path.join(_HERE, "libzpp.so"))

OK, ERR_CONFIG, ERR_VALIDATION, ERR_INTEGRITY, ERR_CUDA, ERR_COMM = range(6)
F32, F16, BF16, F64 = range(4)
FLAG_NONFINITE, FLAG_BADCODE, FLAG_TIMEOUT = 1, 2, 4
IPC_HANDLE_BYTES = 64

c_void_p, c_int, c_int64, c_size_t, c_double = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                                 ctypes.c_size_t, ctypes.c_double)
P = c_void_p
PP = ctypes.POINTER(c_void_p)

# name -> (restype, argtypes); must cover every entry point of include/zpp.h
SIGNATURES = {
    "zpp_version": (c_int, []),
    "zpp_last_error": (ctypes.c_char_p, []),
    "zpp_device_sm_count": (c_int, []),
    "zpp_quantize": (c_int, [P, c_int, c_int64, c_int, c_int64, P, P, P, P]),
    "zpp_swizzle_quantize": (c_int, [P, c_int, c_int64, c_int, c_int, c_int, c_int, c_int, c_int, c_int64,
                                     P, P, P, P]),
    "zpp_dequantize": (c_int, [P, P, c_int, c_int64, c_int, c_int64, P, c_int, P, P]),
    "zpp_gather_dequantize": (c_int, [PP, PP, c_int, c_int, c_int, c_int64, c_int, c_int64, P, c_int, c_int64,
                                      P, c_int64, c_int64, P, P]),
    "zpp_dequant_reduce": (c_int, [PP, PP, c_int, c_int, c_int64, c_int, c_int64, P, c_int, c_double, P, P]),
    "zpp_dequant_reduce_quant": (c_int, [PP, PP, c_int, c_int, c_int64, c_int, c_int64, c_int, c_int64,
                                         P, P, P, c_size_t, P, P]),
    "zpp_drq_workspace_bytes": (c_size_t, [c_int64, c_int64]),
    "zpp_scales": (c_int, [P, c_int, c_int64, c_int, P, P]),
    "zpp_wire_pack": (c_int, [P, P, c_int, c_int64, c_int, c_int64, P, P]),
    "zpp_wire_unpack": (c_int, [P, c_int64, c_int, c_int64, P, P, P]),
    "zpp_comm_create": (c_int, [c_int, c_int, c_int, c_size_t, ctypes.POINTER(c_void_p)]),
    "zpp_comm_ipc_handle": (c_int, [P, P]),
    "zpp_comm_open_peers": (c_int, [P, P]),
    "zpp_comm_sym_ptr": (c_void_p, [P, c_int]),
    "zpp_comm_sym_bytes": (c_size_t, [P]),
    "zpp_comm_barrier": (c_int, [P, c_int, c_int, P, P]),
    "zpp_comm_reset": (c_int, [P]),
    "zpp_comm_destroy": (c_int, [P]),
    "zpp_comm_trace": (c_int, [P, c_int]),
    "zpp_comm_trace_read": (c_int, [P, P, P, c_int]),
    "zpp_qwz_allgather": (c_int, [P, c_size_t, P, c_int, c_int64, c_int, c_int64, P, c_int, c_int64, P, c_int64,
                                  c_int64, P, P]),
    "zpp_qwz_allgather_next": (c_int, [P, c_size_t, P, c_int, c_int64, c_int, c_int64, P, c_int, c_int64, P,
                                       c_int64, c_int64, P, c_int64, P, P]),
    "zpp_hpz_allgather": (c_int, [P, c_size_t, c_int64, c_int, P, P, P]),
    "zpp_qgz_reduce_scatter": (c_int, [P, c_size_t, P, c_int, c_int64, c_int, c_int, c_int, c_int64, c_int,
                                       c_int64, P, c_int, P, P]),
    "zpp_qgz_reduce_scatter_buckets": (c_int, [P, c_size_t, P, c_int, c_int64, c_int, c_int, c_int, c_int, c_int64,
                                               c_int, c_int64, P, c_int, P, P]),
    "zpp_qwz_sym_bytes": (c_size_t, [c_int64, c_int, c_int64, c_int]),
    "zpp_qgz_sym_bytes": (c_size_t, [c_int64, c_int, c_int, c_int, c_int64, c_int, c_int64]),
    "zpp_hpz_sym_bytes": (c_size_t, [c_int64, c_int]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libzpp.so once; raise if it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"libzpp.so not found at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'`")
            lib = ctypes.CDLL(LIB_PATH)
            # ZPP_LIB (development A/B against an older build) may lack newer
            # entries; the in-tree library must export every one
            alt = "ZPP_LIB" in os.environ
            for name, (res, args) in SIGNATURES.items():
                if alt and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().zpp_last_error()
    return msg.decode() if msg else ""


_EXC = {ERR_CONFIG: ConfigError, ERR_VALIDATION: ValidationError, ERR_INTEGRITY: IntegrityError}


def check(rc: int, what: str = ""):
    if rc == OK:
        return
    exc = _EXC.get(rc, DeviceError)
    raise exc(f"{what}: {last_error()}" if what else last_error())


def ptr_array(ptrs):
    arr = (c_void_p * len(ptrs))(*[int(p) for p in ptrs])
    return ctypes.cast(arr, PP), arr  # keep arr alive alongside the pointer


def raise_for_flags(flags: int, what: str = ""):
    """Map the device error word to the reference's exceptions."""
    if flags & FLAG_NONFINITE:
        raise ValidationError(f"{what}: values must be finite")
    if flags & FLAG_BADCODE:
        raise IntegrityError(f"{what}: code outside symmetric range")
    if flags & FLAG_TIMEOUT:
        raise DeviceError(f"{what}: a peer never reached the device barrier")
