"""Host mirror of the reference's bulk-generation module (pkg/src/slicerng/kernels.py).

`mickey_sliced_words` keeps the reference's signature and return type
(kernels.py:189-200) but runs init + keystream in the CUDA kernels; the
`bulk_*` functions are the same operation lifted past the reference's 64-lane
cap.  The lane-extraction helpers (kernels.py:600-621) are pure layout
conversions of an array the caller already holds on the host; bulk callers
should use `MickeyGenerator.generate_rowmajor`, which emits that layout
directly from the GPU.
"""
from __future__ import annotations

import numpy as np

from . import hostmem, mickey
from .generator import MickeyGenerator

_U64 = np.uint64


def mickey_sliced_words(materials, nclocks: int, width: int = 64, device: int = 0) -> np.ndarray:
    """Keystream words uint64[nclocks] of up to `width` lanes (kernels.py:189-200).

    Every call restarts from init, like the reference's compiled loop; odd
    `nclocks` is fine; at width 32 the high 32 bits are zero.
    """
    if width not in mickey.LANE_WIDTHS:
        raise ValueError(f"lane width must be one of {mickey.LANE_WIDTHS}")
    keys, ivs, nbits, uniform = mickey.pack_materials(materials, width)
    with hostmem.borrow_context(MickeyGenerator, device) as gen:   # an idle context of this thread when there is one
        if uniform:
            gen.init_material(keys, ivs, int(nbits[0]))
        else:
            gen.init_ragged(keys, ivs, nbits)
        if nclocks == 0:
            return np.zeros(0, np.uint64)
        return mickey._as_u64(gen.generate_colmajor(int(nclocks)))


def bulk_colmajor(keys, ivs, iv_bits, nclocks: int, device: int = 0, out=None):
    """N instances (u8[N,10] keys, u8[N,*] ivs) -> uint32 out[nclocks][ceil(N/32)].

    iv_bits: one int (uniform) or a u8[N] array (ragged)."""
    with hostmem.borrow_context(MickeyGenerator, device) as gen:
        _init(gen, keys, ivs, iv_bits)
        return gen.generate_colmajor(nclocks, out)


def bulk_rowmajor(keys, ivs, iv_bits, nclocks: int, device: int = 0, out=None, bit_order: str = "msb"):
    """N instances -> uint8 out[N][nclocks/8], lane-major rows; bit_order as in words_lane_major_bytes
    (kernels.py:615-621: first bit of a byte in its most ("msb", default) or least ("lsb") significant position).

    Uniform IV length, MSB-first: one mk2_bulk_rowmajor call (upload, init + keystream and download of consecutive
    instance blocks overlap); otherwise init, then generate."""
    if bit_order not in ("msb", "lsb"):
        raise ValueError(f"unknown bit order {bit_order!r}")
    with hostmem.borrow_context(MickeyGenerator, device) as gen:
        if np.isscalar(iv_bits) and nclocks > 0 and bit_order == "msb":
            return gen.bulk_rowmajor(keys, ivs, int(iv_bits), nclocks, out)[0]
        _init(gen, keys, ivs, iv_bits)
        return gen.generate_rowmajor(nclocks, out, bit_order=bit_order)


def _init(gen, keys, ivs, iv_bits):
    if np.isscalar(iv_bits):
        gen.init_material(keys, ivs, int(iv_bits))
    else:
        gen.init_ragged(keys, ivs, iv_bits)


def mickey_naive_bitwise_bytes(material, nbytes: int, device: int = 0) -> bytes:
    """Single-instance keystream bytes (kernels.py:203-210).  The reference's "naive" engines are its
    CPU baselines; the bytes are by definition those of one MICKEY instance, served here by the GPU."""
    return mickey.MickeyScalar.from_key_iv(material, device).keystream_bytes(nbytes)


def mickey_packed_bytes(material, nbytes: int, device: int = 0) -> bytes:
    """Same stream as mickey_naive_bitwise_bytes (kernels.py:213-229)."""
    return mickey_naive_bitwise_bytes(material, nbytes, device)


# --- lane extraction helpers (kernels.py:600-621) ---------------------------

def words_to_lane_bits(words: np.ndarray, lane: int) -> np.ndarray:
    return ((np.asarray(words, np.uint64) >> _U64(lane)) & _U64(1)).astype(np.uint8)


def words_to_lane_bytes(words: np.ndarray, lane: int, bit_order: str = "msb") -> bytes:
    if bit_order not in ("msb", "lsb"):
        raise ValueError(f"unknown bit order {bit_order!r}")
    bits = words_to_lane_bits(words, lane)
    return np.packbits(bits, bitorder="big" if bit_order == "msb" else "little").tobytes()


def words_lane_major_bytes(words: np.ndarray, lanes: int, bit_order: str = "msb") -> bytes:
    """All of lane 0's bytes, then lane 1's, ... (docs/conventions.md:58-60)."""
    if bit_order not in ("msb", "lsb"):
        raise ValueError(f"unknown bit order {bit_order!r}")
    w = np.asarray(words, np.uint64)
    bits = ((w[None, :] >> np.arange(lanes, dtype=np.uint64)[:, None]) & _U64(1)).astype(np.uint8)
    return np.packbits(bits, axis=1, bitorder="big" if bit_order == "msb" else "little").tobytes()
