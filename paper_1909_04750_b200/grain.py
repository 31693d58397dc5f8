"""Host mirror of the reference's Grain v1 module (pkg/src/slicerng/grain.py).

`GrainKeyIv`, `GrainKeyIvError`, `GrainSliced.from_key_ivs / keystream_words /
keystream_lane_bits / extract_lane / b / s`, `grain_constants` and
`grain_sliced_words` (kernels.py:334-342) keep the reference's names, argument
meaning and errors; every clock runs in csrc/mk2_grain.cuh.  `GrainGenerator`
lifts the same operation past the 64-lane cap.  No CPU cipher code here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import hostmem
from .generator import MickeyGenerator, _ptr
from .mickey import LANE_WIDTHS, LaneState  # noqa: F401  (LaneState re-exported for extract_lane users)

KEY_BYTES = 10
IV_BYTES = 8
STATE_BITS = 80
INIT_CLOCKS = 160

LFSR_TAPS = (62, 51, 38, 23, 13, 0)
NFSR_LINEAR_TAPS = (62, 60, 52, 45, 37, 33, 28, 21, 14, 9, 0)
NFSR_PRODUCT_TAPS = (
    (63, 60), (37, 33), (15, 9), (60, 52, 45), (33, 28, 21), (63, 45, 28, 9), (60, 52, 37, 33),
    (63, 60, 21, 15), (63, 60, 52, 45, 37), (33, 28, 21, 15, 9), (52, 45, 37, 33, 28, 21),
)
H_LFSR_TAPS = (3, 25, 46, 64)
H_NFSR_TAP = 63
OUTPUT_TAPS = (1, 2, 4, 10, 31, 43, 56)


def grain_constants() -> dict:
    """Feedback, filter and output tap definitions (grain.py:62-71)."""
    return {"LFSR_TAPS": LFSR_TAPS, "NFSR_LINEAR_TAPS": NFSR_LINEAR_TAPS, "NFSR_PRODUCT_TAPS": NFSR_PRODUCT_TAPS,
            "H_LFSR_TAPS": H_LFSR_TAPS, "H_NFSR_TAP": H_NFSR_TAP, "OUTPUT_TAPS": OUTPUT_TAPS}


class GrainKeyIvError(ValueError):
    """Invalid key or IV material (grain.py:74-75)."""


@dataclass(frozen=True)
class GrainKeyIv:
    """An 80-bit key and a 64-bit IV (grain.py:78-92); bits are taken LSB-first per byte."""

    key: bytes
    iv: bytes

    def __post_init__(self):
        if len(self.key) != KEY_BYTES:
            raise GrainKeyIvError(f"key must be {KEY_BYTES} bytes")
        if len(self.iv) != IV_BYTES:
            raise GrainKeyIvError(f"IV must be {IV_BYTES} bytes")

    def key_bits(self) -> list:
        return np.unpackbits(np.frombuffer(self.key, np.uint8), bitorder="little").tolist()

    def iv_bits(self) -> list:
        return np.unpackbits(np.frombuffer(self.iv, np.uint8), bitorder="little").tolist()


class GrainGenerator(MickeyGenerator):
    """N independent Grain v1 instances on one B200 (same context machinery as MICKEY)."""

    def init_material(self, keys, ivs):  # type: ignore[override]
        """keys u8[N,10], ivs u8[N,8] (numpy or torch, host or device)."""
        kshape, ishape = tuple(keys.shape), tuple(ivs.shape)
        if len(kshape) != 2 or kshape[1] != KEY_BYTES or len(ishape) != 2 or ishape != (kshape[0], IV_BYTES):
            raise ValueError("keys must be [N, 10] and ivs [N, 8]")
        if kshape[0] < 1:
            raise ValueError("at least one lane is required")
        self._note_size(kshape[0])
        self._ck(self._lib.mk2_grain_init_from_material(self._ctx, _ptr(keys), _ptr(ivs), kshape[0]),
                 "mk2_grain_init_from_material")
        return self

    def generate_colmajor(self, nclocks: int, out=None, stride_words=None):
        G = self.groups
        stride = G if stride_words is None else int(stride_words)
        if out is None:
            out = hostmem.empty((nclocks, stride), np.uint32)
        self._ck(self._lib.mk2_grain_generate_colmajor(self._ctx, int(nclocks), _ptr(out), stride),
                 "mk2_grain_generate_colmajor")
        return out

    def generate_rowmajor(self, nclocks: int, out=None, pitch_bytes=None, byte_offset: int = 0, bit_order: str = "msb"):
        if bit_order not in ("msb", "lsb"):
            raise ValueError(f"unknown bit order {bit_order!r}")
        if nclocks % 8:
            raise ValueError("bit count must be a multiple of 8")
        if out is None:
            pitch = nclocks // 8 if pitch_bytes is None else int(pitch_bytes)
            out = hostmem.empty((self.instances, pitch), np.uint8)
        elif pitch_bytes is None:
            pitch = int(out.shape[-1])
        else:
            pitch = int(pitch_bytes)
        self._ck(self._lib.mk2_grain_generate_rowmajor(self._ctx, int(nclocks), _ptr(out) + int(byte_offset), pitch,
                                                       int(bit_order == "lsb")), "mk2_grain_generate_rowmajor")
        return out

    def export_state(self) -> np.ndarray:
        """uint32 bs[160][G]: NFSR words then LFSR words."""
        bs = np.empty((2 * STATE_BITS, self.groups), np.uint32)
        self._ck(self._lib.mk2_grain_state_export(self._ctx, _ptr(bs)), "mk2_grain_state_export")
        return bs


def pack_materials(materials: Sequence, width: int):
    """Validation of GrainSliced.from_key_ivs (grain.py:254-265) + packing to byte arrays."""
    if not materials:
        raise GrainKeyIvError("at least one lane is required")
    if len(materials) > width:
        raise GrainKeyIvError(f"{len(materials)} lanes exceed width {width}")
    n = len(materials)
    keys = np.zeros((n, KEY_BYTES), np.uint8)
    ivs = np.zeros((n, IV_BYTES), np.uint8)
    for j, m in enumerate(materials):
        try:
            kb, ib = m.key_bits(), m.iv_bits()
        except GrainKeyIvError as exc:
            raise GrainKeyIvError(f"lane {j}: {exc}") from exc
        keys[j] = np.packbits(np.asarray(kb, np.uint8), bitorder="little")
        ivs[j] = np.packbits(np.asarray(ib, np.uint8), bitorder="little")
    return keys, ivs


class GrainSliced:
    """W parallel Grain v1 instances resident on the GPU (grain.py:232-308)."""

    def __init__(self, gen: GrainGenerator, width: int):
        self._gen = gen
        self.width = width
        self.mask = (1 << width) - 1

    def __del__(self):
        gen, self._gen = getattr(self, "_gen", None), None
        if gen is not None:
            try:
                hostmem.release_context(gen)   # back to this thread's idle contexts (hostmem.py)
            except Exception:  # interpreter shutdown
                pass

    @classmethod
    def from_key_ivs(cls, materials: Sequence[GrainKeyIv], width: int = 64, device: int = 0) -> "GrainSliced":
        if width not in LANE_WIDTHS:
            raise ValueError(f"lane width must be one of {LANE_WIDTHS}")
        keys, ivs = pack_materials(materials, width)
        # lanes beyond len(materials) are the reference's unused lanes: the generator is sized to the
        # lane count, and the kernel leaves the rest of the group without the LFSR's top ones
        gen = hostmem.acquire_context(GrainGenerator, device)
        try:
            gen.init_material(keys, ivs)
        except BaseException:
            gen.close()
            raise
        return cls(gen, width)

    def _words(self):
        bs = self._gen.export_state().astype(np.uint64)
        w = bs[:, 0].copy()
        if bs.shape[1] == 2:
            w |= bs[:, 1] << np.uint64(32)
        return [int(x) for x in w[:STATE_BITS]], [int(x) for x in w[STATE_BITS:]]

    @property
    def b(self) -> list:
        return self._words()[0]

    @property
    def s(self) -> list:
        return self._words()[1]

    def extract_lane(self, j: int) -> LaneState:
        b, s = self._words()
        return LaneState([(w >> j) & 1 for w in b], [(w >> j) & 1 for w in s])  # .r = NFSR bits, .s = LFSR bits

    def keystream_words(self, nclocks: int) -> list:
        if nclocks == 0:
            return []
        return [int(w) for w in _as_u64(self._gen.generate_colmajor(nclocks), self.width)]

    def keystream_lane_bits(self, nbits: int) -> list:
        words = np.array(self.keystream_words(nbits), np.uint64)
        return [((words >> np.uint64(j)) & np.uint64(1)).astype(np.uint8).tolist() for j in range(self.width)]


def _as_u64(out: np.ndarray, width: int) -> np.ndarray:
    if out.shape[1] == 2:
        return np.ascontiguousarray(out).view("<u8").reshape(-1)
    return out[:, 0].astype(np.uint64)


def grain_sliced_words(materials, nclocks: int, width: int = 64, device: int = 0) -> np.ndarray:
    """Keystream words uint64[nclocks] (kernels.grain_sliced_words, kernels.py:334-342)."""
    eng = GrainSliced.from_key_ivs(materials, width, device=device)
    if nclocks == 0:
        return np.zeros(0, np.uint64)
    return _as_u64(eng._gen.generate_colmajor(int(nclocks)), width)
