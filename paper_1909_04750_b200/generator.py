"""Bulk generator: the reference's sliced MICKEY engine lifted to N >> 64.

`MickeyGenerator` owns one C-ABI context (include/mk2.h) = one GPU, one
stream, the column-major state of N instances.  It is the object the
reference-shaped front ends (`mickey.MickeySliced`, `kernels.mickey_sliced_words`)
are thin views of.  All cipher work happens in the CUDA kernels; this module
only validates arguments, allocates buffers and passes pointers.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _native, hostmem
from ._native import MK2_IV_UNUSED, check

KEY_BYTES = 10
IV_MAX_BITS = 80


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(buf) -> int:
    """Raw address of a numpy array / torch tensor / int pointer."""
    if buf is None:
        return 0
    if isinstance(buf, int):
        return buf
    if isinstance(buf, np.ndarray):
        if not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("buffer must be C-contiguous")
        return buf.ctypes.data
    if _is_torch(buf):
        if not buf.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return buf.data_ptr()
    raise TypeError(f"unsupported buffer type {type(buf)!r}")


# Contexts are created with the warp-per-group small-batch kernels enabled (csrc/mk2_coop.cuh).  MK2_SMALL_BATCH=0
# in the environment, or this flag, makes new contexts use the thread-per-group throughput kernels at every size:
# the GPU test suite runs itself both ways so that the edge cases of both kernel families stay covered.
DEFAULT_SMALL_BATCH = os.environ.get("MK2_SMALL_BATCH", "1") != "0"


class MickeyGenerator:
    """N independent MICKEY 2.0 instances on one B200 (32 per GPU thread)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self._lib = _native.lib()
        self._ctx = C.c_void_p()
        check(self._lib.mk2_create(int(device), C.byref(self._ctx)), None, "mk2_create")
        self.device = int(device)
        self._knobs_touched = False   # hostmem's context pool only keeps contexts in their default configuration
        self._peak_groups = 0
        if not DEFAULT_SMALL_BATCH:
            self._ck(self._lib.mk2_set_small_batch(self._ctx, 0), "mk2_set_small_batch")
        if stream is not None:
            self.set_stream(stream)

    # -- lifetime ---------------------------------------------------------
    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx:
            self._lib.mk2_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _ck(self, rc, what):
        check(rc, self._ctx, what)

    def set_stream(self, cuda_stream: Optional[int]):
        """Launch on an external CUDA stream handle (e.g. torch.cuda.current_stream().cuda_stream;
        0 is the legacy default stream).  None goes back to the context's own stream."""
        self._knobs_touched = True
        if cuda_stream is None:
            self._ck(self._lib.mk2_use_own_stream(self._ctx), "mk2_use_own_stream")
        else:
            self._ck(self._lib.mk2_set_stream(self._ctx, C.c_void_p(int(cuda_stream))), "mk2_set_stream")

    def set_chunk_clocks(self, clocks: int):
        """Tuning knob: clocks per scheduling chunk of the persistent keystream kernels."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_chunk_clocks(self._ctx, int(clocks)), "mk2_set_chunk_clocks")

    def set_row_staging(self, mode: int):
        """Tuning knob: row-major staging tile in shared memory (1), tensor memory (2) or (Grain only) L2-resident
        global scratch (3); 4 (Grain only) = the lone-warp ring kernel for row-major and the circular-buffer kernel
        for column-major output, 5 (Grain only) = the eight-warp row-major kernel (include/mk2.h); 0 = automatic."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_row_staging(self._ctx, int(mode)), "mk2_set_row_staging")

    def set_small_batch(self, enable: bool):
        """Tuning knob: warp-per-group kernels for small batches (default) or the throughput kernels at every size."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_small_batch(self._ctx, int(bool(enable))), "mk2_set_small_batch")

    def set_bulk_fused(self, mode):
        """Tuning knob: device-to-device bulk_rowmajor as one fused kernel: 1 / True = automatic (init-dominated calls,
        the default), 2 = whenever eligible, 0 / False = never (pack / init / keystream kernels)."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_bulk_fused(self._ctx, int(mode)), "mk2_set_bulk_fused")

    def set_stage_bytes(self, nbytes: int):
        """Tuning knob: bytes per device staging tile when the output buffer is in host memory."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_stage_bytes(self._ctx, int(nbytes)), "mk2_set_stage_bytes")

    def set_async(self, flag: bool):
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_async(self._ctx, int(bool(flag))), "mk2_set_async")

    def last_plan(self):
        """(threads per CTA, clocks per chunk) of the most recent keystream launch."""
        b, c = C.c_int(), C.c_uint32()
        self._ck(self._lib.mk2_last_plan(self._ctx, C.byref(b), C.byref(c)), "mk2_last_plan")
        return b.value, c.value

    def set_block_threads(self, threads: int):
        """Tuning knob: threads per CTA of the clocking kernels (32..256)."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_block_threads(self._ctx, int(threads)), "mk2_set_block_threads")

    TRACE_DTYPE = np.dtype([("chain", "<u4"), ("k", "<u4"), ("smid", "<u4"), ("warp", "<u4"),
                            ("t_pop", "<u8"), ("t_start", "<u8"), ("t_end", "<u8"), ("pad", "<u8")])

    def set_trace(self, capacity: int):
        """Diagnostics: record (chain, chunk, SM, warp, timestamps) per scheduled job."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_trace(self._ctx, int(capacity)), "mk2_set_trace")
        self._trace_cap = int(capacity)

    def read_trace(self) -> np.ndarray:
        cap = getattr(self, "_trace_cap", 0)
        rec = np.zeros(cap, self.TRACE_DTYPE)
        n = C.c_uint64()
        self._ck(self._lib.mk2_read_trace(self._ctx, _ptr(rec), cap, C.byref(n)), "mk2_read_trace")
        return rec[: n.value]

    def set_max_ctas(self, ctas: int):
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_max_ctas(self._ctx, int(ctas)), "mk2_set_max_ctas")

    def set_host_threads(self, threads: int):
        """Host threads that move bounce tiles into PAGEABLE output arrays (0 = automatic)."""
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_host_threads(self._ctx, int(threads)), "mk2_set_host_threads")

    def synchronize(self):
        self._ck(self._lib.mk2_sync(self._ctx), "mk2_sync")

    def trim(self):
        """Release scratch (key/IV staging pool, host-output staging buffers) back to the device."""
        self._ck(self._lib.mk2_trim(self._ctx), "mk2_trim")

    def set_group_offset(self, group_offset: int):
        self._knobs_touched = True
        self._ck(self._lib.mk2_set_group_offset(self._ctx, int(group_offset)), "mk2_set_group_offset")

    # -- geometry ---------------------------------------------------------
    def _query(self):
        n, g, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._ck(self._lib.mk2_query(self._ctx, C.byref(n), C.byref(g), C.byref(c)), "mk2_query")
        return n.value, g.value, c.value

    @property
    def instances(self) -> int:
        return self._query()[0]

    @property
    def groups(self) -> int:
        return self._query()[1]

    @property
    def clocks(self) -> int:
        return self._query()[2]

    # -- initialisation ---------------------------------------------------
    def init_material(self, keys, ivs=None, iv_bits: int = 0):
        """Uniform IV length: keys u8[N,10], ivs u8[N,>=ceil(iv_bits/8)] (numpy or torch, host or device)."""
        n, iv_stride = _material_shape(keys, ivs, iv_bits)
        self._note_size(n)
        self._ck(self._lib.mk2_init_from_material(self._ctx, _ptr(keys), _ptr(ivs) if iv_bits else 0, iv_stride,
                                                  int(iv_bits), n), "mk2_init_from_material")
        return self

    def _note_size(self, n: int):
        self._peak_groups = max(self._peak_groups, (int(n) + 31) // 32)

    def init_ragged(self, keys, ivs, iv_nbits):
        """Per-instance IV bit lengths (u8[N], 0..80 or MK2_IV_UNUSED)."""
        n, iv_stride = _material_shape(keys, ivs, 0)
        iv_nbits = _iv_nbits_u8(iv_nbits, n)
        self._note_size(n)
        self._ck(self._lib.mk2_init_ragged(self._ctx, _ptr(keys), _ptr(ivs), iv_stride, _ptr(iv_nbits), n),
                 "mk2_init_ragged")
        return self

    def init_counter(self, key: bytes, first_index: int, n: int):
        """One key, IV_k = 80-bit big-endian (first_index + k): SURVEY.md 8(d) synthetic set."""
        if len(key) != KEY_BYTES:
            raise ValueError(f"key must be {KEY_BYTES} bytes")
        kb = (C.c_uint8 * KEY_BYTES).from_buffer_copy(bytes(key))
        self._note_size(n)
        self._ck(self._lib.mk2_init_counter_iv(self._ctx, C.cast(kb, C.c_void_p), int(first_index), int(n)),
                 "mk2_init_counter_iv")
        return self

    def init_seed(self, seed: bytes, first_lane: int, n: int):
        """Seed-derived key/IV material (seedgen.derive_lane_material) for lanes first_lane..+n-1, then init."""
        sb = _seed_buf(seed)
        self._note_size(n)
        self._ck(self._lib.mk2_init_from_seed(self._ctx, C.cast(sb, C.c_void_p), int(first_lane), int(n)),
                 "mk2_init_from_seed")
        return self

    def derive_material(self, seed: bytes, first_lane: int, n: int, keys=None, ivs=None, algo_tag: int = 3):
        """keys u8[n,10], ivs u8[n,10] (algo_tag 3, mickey) or u8[n,8] (algo_tag 2, grain: seedgen.py:24-29)
        derived on the GPU (numpy by default; torch/device buffers accepted)."""
        sb = _seed_buf(seed)
        if algo_tag not in (2, 3):
            raise ValueError("algo_tag must be 2 (grain) or 3 (mickey)")
        if keys is None:
            keys = np.empty((n, KEY_BYTES), np.uint8)
        if ivs is None:
            ivs = np.empty((n, 10 if algo_tag == 3 else 8), np.uint8)
        self._ck(self._lib.mk2_derive_material(self._ctx, C.cast(sb, C.c_void_p), int(algo_tag), int(first_lane), int(n),
                                               _ptr(keys), _ptr(ivs)), "mk2_derive_material")
        return keys, ivs

    # -- generation -------------------------------------------------------
    def generate_colmajor(self, nclocks: int, out=None, stride_words: Optional[int] = None):
        """uint32 out[nclocks][G]; bit j of out[t][g] = keystream bit t of instance 32 g + j."""
        G = self.groups
        stride = G if stride_words is None else int(stride_words)
        if out is None:
            out = hostmem.empty((nclocks, stride), np.uint32)
        self._ck(self._lib.mk2_generate_colmajor(self._ctx, int(nclocks), _ptr(out), stride), "mk2_generate_colmajor")
        return out

    def generate_rowmajor(self, nclocks: int, out=None, pitch_bytes: Optional[int] = None, byte_offset: int = 0,
                          bit_order: str = "msb"):
        """uint8 out[N][nclocks/8] (the reference's lane-major order); the first bit of every byte in its most
        significant position, or with bit_order="lsb" in the least significant one (kernels.py:604-612)."""
        if bit_order not in ("msb", "lsb"):
            raise ValueError(f"unknown bit order {bit_order!r}")
        if nclocks % 8:
            raise ValueError("bit count must be a multiple of 8")
        N = self.instances
        if out is None:
            pitch = nclocks // 8 if pitch_bytes is None else int(pitch_bytes)
            out = hostmem.empty((N, pitch), np.uint8)
        elif pitch_bytes is None:
            pitch = int(out.shape[-1]) * (out.element_size() if _is_torch(out) else out.itemsize)
        else:
            pitch = int(pitch_bytes)
        self._ck(self._lib.mk2_generate_rowmajor_order(self._ctx, int(nclocks), _ptr(out) + int(byte_offset), pitch,
                                                       int(bit_order == "lsb")), "mk2_generate_rowmajor_order")
        return out

    def bulk_rowmajor(self, keys, ivs, iv_bits: int, nclocks: int, out=None, pitch_bytes: Optional[int] = None):
        """One shot: init from (keys, ivs) + nclocks keystream bits per instance, row-major (the reference's
        mickey_sliced_words + words_lane_major_bytes for any N).  With host arrays the upload, the init +
        keystream and the download of consecutive instance blocks overlap.  Returns (out, checksum)."""
        if nclocks % 8:
            raise ValueError("bit count must be a multiple of 8")
        n, iv_stride = _material_shape(keys, ivs, iv_bits)
        self._note_size(min(n, 1 << 22))
        if out is None:
            pitch = nclocks // 8 if pitch_bytes is None else int(pitch_bytes)
            out = hostmem.empty((n, pitch), np.uint8)
        elif pitch_bytes is None:
            pitch = int(out.shape[-1]) * (out.element_size() if _is_torch(out) else out.itemsize)
        else:
            pitch = int(pitch_bytes)
        csum = C.c_uint64(0)
        self._ck(self._lib.mk2_bulk_rowmajor(self._ctx, _ptr(keys), _ptr(ivs) if iv_bits else 0, iv_stride, int(iv_bits),
                                             n, int(nclocks), _ptr(out), pitch, C.byref(csum)), "mk2_bulk_rowmajor")
        return out, int(csum.value)

    def clock(self, mixing: bool, input_words=None, n: int = 1):
        """n raw CLOCK_KG steps (no output); input_words uint32[n][G] or None."""
        self._ck(self._lib.mk2_clock(self._ctx, int(bool(mixing)), _ptr(input_words), int(n)), "mk2_clock")

    # -- state / checksum -------------------------------------------------
    def export_state(self) -> np.ndarray:
        """uint32 rs[200][G]: R words then S words (MickeySliced.rregs / .sregs)."""
        rs = np.empty((200, self.groups), np.uint32)
        self._ck(self._lib.mk2_state_export(self._ctx, _ptr(rs)), "mk2_state_export")
        return rs

    def import_state(self, rs, n: int):
        self._note_size(n)
        rs = np.ascontiguousarray(rs, np.uint32) if isinstance(rs, np.ndarray) else rs
        self._ck(self._lib.mk2_state_import(self._ctx, _ptr(rs), int(n)), "mk2_state_import")
        return self

    def checksum(self) -> int:
        v = C.c_uint64()
        self._ck(self._lib.mk2_checksum(self._ctx, C.byref(v)), "mk2_checksum")
        return v.value

    # -- measurement ------------------------------------------------------
    @property
    def last_kernel_ms(self) -> float:
        return float(self._lib.mk2_last_kernel_ms(self._ctx))

    @property
    def last_kernel_launches(self) -> int:
        return int(self._lib.mk2_last_kernel_launches(self._ctx))

    def lop3_peak(self):
        """(lane-ops/s, ms) of the dependency-free LOP3 probe: the roofline denominator."""
        v, ms = C.c_double(), C.c_float()
        self._ck(self._lib.mk2_lop3_peak(self._ctx, C.byref(v), C.byref(ms)), "mk2_lop3_peak")
        return v.value, ms.value


def _iv_nbits_u8(iv_nbits, n: int):
    """Per-instance IV bit lengths as the C ABI reads them: n contiguous uint8 values (0..80 or MK2_IV_UNUSED).
    Lists and integer numpy arrays of any width are range-checked and converted (a default int64 array read as
    raw bytes would silently load wrong lengths); torch tensors must already be uint8."""
    if _is_torch(iv_nbits):
        if _dtype_name(iv_nbits) != "uint8" or iv_nbits.numel() != n:
            raise ValueError("iv_nbits must be a uint8 tensor with one entry per instance")
        return iv_nbits.contiguous()
    a = np.asarray(iv_nbits)
    if a.size != n:
        raise ValueError("iv_nbits must have one entry per instance")
    if a.dtype == np.uint8:
        return np.ascontiguousarray(a).reshape(-1)
    if not np.issubdtype(a.dtype, np.integer):
        raise ValueError("iv_nbits must hold integers")
    a = a.reshape(-1)
    bad = np.flatnonzero(((a < 0) | (a > IV_MAX_BITS)) & (a != MK2_IV_UNUSED))
    if bad.size:
        raise ValueError(f"lane {int(bad[0])}: IV must be at most {IV_MAX_BITS} bits")
    return np.ascontiguousarray(a.astype(np.uint8))


def _seed_buf(seed: bytes):
    if len(seed) != 32:
        raise ValueError("master seed must be 32 bytes")
    return (C.c_uint8 * 32).from_buffer_copy(bytes(seed))


def _material_shape(keys, ivs, iv_bits):
    kshape = tuple(keys.shape)
    if len(kshape) != 2 or kshape[1] != KEY_BYTES:
        raise ValueError(f"keys must have shape [N, {KEY_BYTES}]")
    if _dtype_name(keys) != "uint8":
        raise ValueError("keys must be uint8")
    n = kshape[0]
    if n < 1:
        raise ValueError("at least one lane is required")
    if iv_bits > IV_MAX_BITS:
        raise ValueError(f"IV must be at most {IV_MAX_BITS} bits")
    iv_stride = 0
    if ivs is not None:
        ishape = tuple(ivs.shape)
        if len(ishape) != 2 or ishape[0] != n or _dtype_name(ivs) != "uint8":
            raise ValueError("ivs must be uint8 with shape [N, iv_bytes]")
        iv_stride = ishape[1]
    if iv_bits and iv_stride < (iv_bits + 7) // 8:
        raise ValueError("ivs rows are shorter than iv_bits")
    return n, iv_stride


def _dtype_name(x) -> str:
    return str(x.dtype).replace("torch.", "")
