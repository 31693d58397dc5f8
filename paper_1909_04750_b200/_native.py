"""ctypes binding of csrc/libmk2.so (C ABI: include/mk2.h).

There is deliberately no fallback here: if the CUDA library is missing it is
built with nvcc (which needs no GPU); if that is impossible, or no sm_100
device is present when a context is created, the call raises.  Nothing in this
package computes keystream on the CPU.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from . import build as _build

_PKG = Path(__file__).resolve().parent
_lock = threading.Lock()
_lib = None

ABI_VERSION = 2
MK2_OK = 0
MK2_E_CUDA, MK2_E_ARG, MK2_E_STATE, MK2_E_NODEVICE, MK2_E_NOMEM = -1, -2, -3, -4, -5
MK2_IV_UNUSED = 0xFF

# every symbol include/mk2.h declares: (restype, argtypes)
_vp, _u8p, _u32p, _u64 = C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64
SYMBOLS = {
    "mk2_abi_version": (C.c_int, []),
    "mk2_device_count": (C.c_int, []),
    "mk2_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "mk2_destroy": (C.c_int, [_vp]),
    "mk2_set_stream": (C.c_int, [_vp, _vp]),
    "mk2_use_own_stream": (C.c_int, [_vp]),
    "mk2_set_chunk_clocks": (C.c_int, [_vp, C.c_uint32]),
    "mk2_set_stage_bytes": (C.c_int, [_vp, _u64]),
    "mk2_bulk_rowmajor": (C.c_int, [_vp, _vp, _vp, C.c_uint32, C.c_uint32, _u64, _u64, _vp, _u64, C.POINTER(_u64)]),
    "mk2_set_row_staging": (C.c_int, [_vp, C.c_int]),
    "mk2_set_bulk_fused": (C.c_int, [_vp, C.c_int]),
    "mk2_set_small_batch": (C.c_int, [_vp, C.c_int]),
    "mk2_last_plan": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_uint32)]),
    "mk2_sync": (C.c_int, [_vp]),
    "mk2_trim": (C.c_int, [_vp]),
    "mk2_last_error": (C.c_char_p, [_vp]),
    "mk2_set_group_offset": (C.c_int, [_vp, _u64]),
    "mk2_init_from_material": (C.c_int, [_vp, _u8p, _u8p, C.c_uint32, C.c_uint32, _u64]),
    "mk2_init_ragged": (C.c_int, [_vp, _u8p, _u8p, C.c_uint32, _u8p, _u64]),
    "mk2_init_counter_iv": (C.c_int, [_vp, _u8p, _u64, _u64]),
    "mk2_derive_material": (C.c_int, [_vp, _u8p, C.c_uint32, _u64, _u64, _u8p, _u8p]),
    "mk2_init_from_seed": (C.c_int, [_vp, _u8p, _u64, _u64]),
    "mk2_generate_colmajor": (C.c_int, [_vp, _u64, _vp, _u64]),
    "mk2_generate_rowmajor": (C.c_int, [_vp, _u64, _vp, _u64]),
    "mk2_generate_rowmajor_order": (C.c_int, [_vp, _u64, _vp, _u64, C.c_int]),
    "mk2_set_host_threads": (C.c_int, [_vp, C.c_int]),
    "mk2_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "mk2_host_free": (C.c_int, [_vp]),
    "mk2_grain_init_from_material": (C.c_int, [_vp, _u8p, _u8p, _u64]),
    "mk2_grain_generate_colmajor": (C.c_int, [_vp, _u64, _vp, _u64]),
    "mk2_grain_generate_rowmajor": (C.c_int, [_vp, _u64, _vp, _u64, C.c_int]),
    "mk2_grain_state_export": (C.c_int, [_vp, _u32p]),
    "mk2_clock": (C.c_int, [_vp, C.c_int, _u32p, _u64]),
    "mk2_query": (C.c_int, [_vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "mk2_state_export": (C.c_int, [_vp, _u32p]),
    "mk2_state_import": (C.c_int, [_vp, _u32p, _u64]),
    "mk2_checksum": (C.c_int, [_vp, C.POINTER(_u64)]),
    "mk2_last_kernel_ms": (C.c_float, [_vp]),
    "mk2_last_kernel_launches": (C.c_int, [_vp]),
    "mk2_set_async": (C.c_int, [_vp, C.c_int]),
    "mk2_set_block_threads": (C.c_int, [_vp, C.c_int]),
    "mk2_set_trace": (C.c_int, [_vp, _u64]),
    "mk2_read_trace": (C.c_int, [_vp, _vp, _u64, C.POINTER(_u64)]),
    "mk2_set_max_ctas": (C.c_int, [_vp, C.c_uint32]),
    "mk2_lop3_peak": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_float)]),
    "mk2_lop3_per_clock": (C.c_int, []),
    "mk2_rblock": (C.c_int, [C.c_int]),
    "mk2_lop3_per_block": (C.c_int, [C.c_int]),
}


class Mk2Error(RuntimeError):
    """A C-ABI call failed (CUDA error, missing device, bad state)."""


def library_path() -> Path:
    return _build.LIB


def lib() -> C.CDLL:
    """Load (building first if needed) the CUDA library; never falls back."""
    global _lib
    with _lock:
        if _lib is None:
            import os

            override = os.environ.get("MK2_LIB")  # experiments: an alternative build of the same sources
            if override:
                path = Path(override)
            else:
                path = _build.build_native()  # no-op unless a source changed since the library was built
            L = C.CDLL(str(path))
            for name, (res, args) in SYMBOLS.items():
                fn = getattr(L, name)  # AttributeError = ABI mismatch, fail loudly
                fn.restype = res
                fn.argtypes = args
            if L.mk2_abi_version() != ABI_VERSION:
                raise Mk2Error(f"{path} has ABI version {L.mk2_abi_version()}, this package needs {ABI_VERSION}")
            _lib = L
    return _lib


def check(rc: int, ctx=None, what: str = "mk2 call"):
    if rc != MK2_OK:
        msg = lib().mk2_last_error(ctx)
        text = msg.decode() if msg else ""
        if rc == MK2_E_ARG:
            raise ValueError(f"{what}: {text}")
        raise Mk2Error(f"{what} failed (code {rc}): {text}")
