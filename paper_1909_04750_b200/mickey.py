"""Host mirror of the reference's MICKEY 2.0 module (pkg/src/slicerng/mickey.py).

Same names, argument meaning and error behaviour as the reference for the
hot path's public surface -- `MickeyKeyIv`, `MickeyKeyIvError`,
`MickeySliced.from_key_ivs / keystream_words / keystream_lane_bits /
extract_lane / clock_kg / rregs / sregs`, `mickey_constants` -- but every
clock runs in the sm_100a kernels behind the C ABI (include/mk2.h).  There is
no CPU cipher code in this package: without a B200 these classes raise.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import hostmem
from ._native import MK2_IV_UNUSED
from .generator import MickeyGenerator

KEY_BYTES = 10
IV_MAX_BITS = 80
STATE_BITS = 100
PRECLOCKS = 100
LANE_WIDTHS = (32, 64)  # pkg/src/slicerng/bitslab.py:16

# Cipher tables, packed as in pkg/src/slicerng/mickey.py:35-39 (bit i = word
# i // 32, bit i % 32).  The CUDA side holds the same five constants in
# csrc/mk2_clock.cuh; tests compare both against the golden file.
_R_MASK_WORDS = (0x1279327B, 0xB5546660, 0xDF87818F, 0x00000003)
_COMP0_WORDS = (0x6AA97A30, 0x7942A809, 0x057EBFEA, 0x00000006)
_COMP1_WORDS = (0xDD629E9A, 0xE3A21D63, 0x91C23DD7, 0x00000001)
_FB0_WORDS = (0x9FFA7FAF, 0xAF4A9381, 0x9CEC5802, 0x00000001)
_FB1_WORDS = (0x4C8CB877, 0x4911B063, 0x40FBC52B, 0x00000008)


def _unpack(words):
    return tuple((words[i >> 5] >> (i & 31)) & 1 for i in range(STATE_BITS))


RTAPS_BITS = _unpack(_R_MASK_WORDS)
RTAPS = tuple(i for i in range(STATE_BITS) if RTAPS_BITS[i])
COMP0 = _unpack(_COMP0_WORDS)
COMP1 = _unpack(_COMP1_WORDS)
FB0 = _unpack(_FB0_WORDS)
FB1 = _unpack(_FB1_WORDS)


def mickey_constants() -> dict:
    """RTAPS set plus the four 100-bit sequences (mickey.py:61-69)."""
    return {"RTAPS": RTAPS, "COMP0": COMP0, "COMP1": COMP1, "FB0": FB0, "FB1": FB1}


class MickeyKeyIvError(ValueError):
    """Invalid key or IV material (mickey.py:72-73)."""


@dataclass(frozen=True)
class MickeyKeyIv:
    """An 80-bit key with a 0..80 bit IV (bytes, or a 0/1 sequence); mickey.py:76-98."""

    key: bytes
    iv: bytes | Sequence[int] = b""

    def __post_init__(self):
        if len(self.key) != KEY_BYTES:
            raise MickeyKeyIvError(f"key must be {KEY_BYTES} bytes")
        if len(self.iv_bits()) > IV_MAX_BITS:
            raise MickeyKeyIvError(f"IV must be at most {IV_MAX_BITS} bits")

    def key_bits(self) -> list[int]:
        return _bytes_to_bits(self.key)

    def iv_bits(self) -> list[int]:
        if isinstance(self.iv, (bytes, bytearray)):
            return _bytes_to_bits(bytes(self.iv))
        bits = list(self.iv)
        if any(b not in (0, 1) for b in bits):
            raise MickeyKeyIvError("IV bit sequence must contain only 0/1")
        return bits


def _bytes_to_bits(data: bytes) -> list[int]:
    # MSB-first per byte (pkg/src/slicerng/bitops.py:33-36)
    return np.unpackbits(np.frombuffer(bytes(data), np.uint8)).tolist()


@dataclass(frozen=True)
class LaneState:
    """One lane's registers as 0/1 lists (what extract_lane exposes: .r, .s)."""

    r: list
    s: list


def pack_materials(materials: Sequence, width: int):
    """Validate lanes like from_key_ivs (mickey.py:268-285) and pack them.

    Returns (keys u8[width,10], ivs u8[width,10], nbits u8[width], uniform).
    Unused lanes: zero material when lengths are uniform (they load zeros for
    the same clock count), MK2_IV_UNUSED (all-zero state) when ragged --
    exactly what the reference's two routes leave in those lanes.
    """
    if not materials:
        raise MickeyKeyIvError("at least one lane is required")
    if len(materials) > width:
        raise MickeyKeyIvError(f"{len(materials)} lanes exceed width {width}")
    keys = np.zeros((width, KEY_BYTES), np.uint8)
    ivs = np.zeros((width, 10), np.uint8)
    nbits = np.zeros(width, np.uint8)
    n = len(materials)
    if all(type(m) is MickeyKeyIv and type(m.iv) is bytes for m in materials):
        # the common case, without a Python-level loop over bits: records validated at construction
        # (__post_init__), byte strings already in the MSB-first wire order
        keys[:n] = np.frombuffer(b"".join(m.key for m in materials), np.uint8).reshape(n, KEY_BYTES)
        lens = {len(m.iv) for m in materials}
        if len(lens) == 1:
            (ln,) = lens
            if ln:
                ivs[:n, :ln] = np.frombuffer(b"".join(m.iv for m in materials), np.uint8).reshape(n, ln)
            nbits[:] = 8 * ln      # uniform: unused lanes load zero bits for the same clock count
            return keys, ivs, nbits, True
        for lane, m in enumerate(materials):
            if m.iv:
                ivs[lane, : len(m.iv)] = np.frombuffer(m.iv, np.uint8)
            nbits[lane] = 8 * len(m.iv)
        nbits[n:] = MK2_IV_UNUSED
        return keys, ivs, nbits, False
    for lane, m in enumerate(materials):
        if type(m) is MickeyKeyIv and type(m.iv) is bytes:
            # validated at construction (__post_init__); byte strings are already in the MSB-first wire order
            keys[lane] = np.frombuffer(m.key, np.uint8)
            if m.iv:
                ivs[lane, : len(m.iv)] = np.frombuffer(m.iv, np.uint8)
            nbits[lane] = 8 * len(m.iv)
            continue
        try:
            iv = m.iv_bits()
            key = m.key_bits()
            if len(iv) > IV_MAX_BITS:
                raise MickeyKeyIvError(f"IV must be at most {IV_MAX_BITS} bits")
            if len(key) != 80:
                raise MickeyKeyIvError("key must be 80 bits")
        except MickeyKeyIvError as exc:
            raise MickeyKeyIvError(f"lane {lane}: {exc}") from exc
        keys[lane] = np.packbits(np.asarray(key, np.uint8))
        if iv:
            packed = np.packbits(np.asarray(iv, np.uint8))
            ivs[lane, : len(packed)] = packed
        nbits[lane] = len(iv)
    n = len(materials)
    uniform = len(set(nbits[:n].tolist())) == 1
    if uniform:
        nbits[n:] = nbits[0]
    else:
        nbits[n:] = MK2_IV_UNUSED
    return keys, ivs, nbits, uniform


class MickeySliced:
    """W parallel MICKEY 2.0 instances, column-major, resident on the GPU.

    Mirrors pkg/src/slicerng/mickey.py:236-375.  `rregs` / `sregs` are read
    back from the device on access; `keystream_words` is resumable and a
    zero-length request leaves the state untouched (tests/test_mickey.py:167).
    """

    def __init__(self, rregs, sregs, width: int, device: int = 0):
        if width not in LANE_WIDTHS:
            raise ValueError(f"lane width must be one of {LANE_WIDTHS}")
        rregs, sregs = list(rregs), list(sregs)
        if len(rregs) != STATE_BITS or len(sregs) != STATE_BITS:
            raise ValueError("sliced state needs 100 R words and 100 S words")
        self.width = width
        self.mask = (1 << width) - 1
        self._gen = hostmem.acquire_context(MickeyGenerator, device)
        self._gen.import_state(self._words_to_rs(rregs, sregs), width)

    def __del__(self):
        # the context goes back to this thread's pool of idle contexts (hostmem.py) instead of being destroyed:
        # the reference's callers build one engine per 64-lane batch (cli.py:219-231)
        gen, self._gen = getattr(self, "_gen", None), None
        if gen is not None:
            try:
                hostmem.release_context(gen)
            except Exception:  # interpreter shutdown
                pass

    @classmethod
    def _adopt(cls, gen: MickeyGenerator, width: int) -> "MickeySliced":
        self = object.__new__(cls)
        self.width = width
        self.mask = (1 << width) - 1
        self._gen = gen
        return self

    def _words_to_rs(self, rregs, sregs) -> np.ndarray:
        G = self.width // 32
        rs = np.zeros((200, G), np.uint32)
        for i in range(STATE_BITS):
            for g in range(G):
                rs[i, g] = (int(rregs[i]) >> (32 * g)) & 0xFFFFFFFF
                rs[100 + i, g] = (int(sregs[i]) >> (32 * g)) & 0xFFFFFFFF
        return rs

    @classmethod
    def from_key_ivs(cls, materials: Sequence[MickeyKeyIv], width: int = 64, device: int = 0) -> "MickeySliced":
        """Per-lane key/IV load + pre-clock on the GPU (mickey.py:258-304)."""
        if width not in LANE_WIDTHS:
            raise ValueError(f"lane width must be one of {LANE_WIDTHS}")
        keys, ivs, nbits, uniform = pack_materials(materials, width)
        gen = hostmem.acquire_context(MickeyGenerator, device)
        try:
            if uniform:
                gen.init_material(keys, ivs, int(nbits[0]))
            else:
                gen.init_ragged(keys, ivs, nbits)
        except BaseException:
            gen.close()
            raise
        return cls._adopt(gen, width)

    # -- state views ------------------------------------------------------
    def _state_words(self):
        rs = self._gen.export_state().astype(np.uint64)
        G = rs.shape[1]
        words = rs[:, 0].copy()
        if G == 2:
            words |= rs[:, 1] << np.uint64(32)
        return [int(w) for w in words[:100]], [int(w) for w in words[100:]]

    @property
    def rregs(self) -> list:
        return self._state_words()[0]

    @property
    def sregs(self) -> list:
        return self._state_words()[1]

    def extract_lane(self, j: int) -> LaneState:
        r, s = self._state_words()
        return LaneState([(w >> j) & 1 for w in r], [(w >> j) & 1 for w in s])

    # -- clocking ---------------------------------------------------------
    def clock_kg(self, mixing: bool, input_word: int) -> None:
        G = self.width // 32
        w = np.array([[(int(input_word) >> (32 * g)) & 0xFFFFFFFF for g in range(G)]], np.uint32)
        self._gen.clock(mixing, w, 1)

    def keystream_words(self, nclocks: int) -> list:
        """One output word per clock: bit j = lane j's keystream bit (mickey.py:362-368)."""
        if nclocks == 0:
            return []
        out = self._gen.generate_colmajor(nclocks)
        return [int(w) for w in _as_u64(out)]

    def keystream_lane_bits(self, nbits: int) -> list:
        words = np.array(self.keystream_words(nbits), np.uint64)
        return [((words >> np.uint64(j)) & np.uint64(1)).astype(np.uint8).tolist() for j in range(self.width)]


def _as_u64(out: np.ndarray) -> np.ndarray:
    """uint32 [T][G] (G = 1 or 2) -> the reference's uint64 [T] word array."""
    if out.shape[1] == 2:
        return np.ascontiguousarray(out).view("<u8").reshape(-1)
    return out[:, 0].astype(np.uint64)


class MickeyScalar:
    """Single-instance engine with the reference's interface (mickey.py:101-161).

    The reference's bit-serial class is its CPU oracle; here the one instance is
    lane 0 of a GPU-resident 32-lane group, so every clock still runs in the
    CUDA kernels (there is no CPU cipher code in this package).  `r` / `s` are
    0/1 lists read back from the device.
    """

    def __init__(self, r=None, s=None, device: int = 0):
        r = [0] * STATE_BITS if r is None else list(r)
        s = [0] * STATE_BITS if s is None else list(s)
        if len(r) != STATE_BITS or len(s) != STATE_BITS:
            raise ValueError("R and S must be 100 bits each")
        self._eng = MickeySliced([int(b) & 1 for b in r], [int(b) & 1 for b in s], 32, device=device)

    @classmethod
    def from_key_iv(cls, material: MickeyKeyIv, device: int = 0) -> "MickeyScalar":
        """Load IV bits, then key bits, then preclock, all with mixing (mickey.py:141-151)."""
        self = object.__new__(cls)
        self._eng = MickeySliced.from_key_ivs([material], width=32, device=device)
        return self

    @property
    def r(self) -> list:
        return self._eng.extract_lane(0).r

    @property
    def s(self) -> list:
        return self._eng.extract_lane(0).s

    def clock_kg(self, mixing: bool, input_bit: int) -> None:
        self._eng.clock_kg(mixing, int(input_bit) & 1)

    def keystream_bits(self, nbits: int) -> list:
        return [int(w) & 1 for w in self._eng.keystream_words(nbits)]

    def keystream_bytes(self, nbytes: int, bit_order: str = "msb") -> bytes:
        if bit_order not in ("msb", "lsb"):
            raise ValueError(f"unknown bit order {bit_order!r}")
        bits = np.array(self.keystream_bits(8 * nbytes), np.uint8)
        return np.packbits(bits, bitorder="big" if bit_order == "msb" else "little").tobytes()


class MickeyScalarPacked(MickeyScalar):
    """Same engine with each register exposed as one int (mickey.py:173-227): bit i = register bit i."""

    def __init__(self, r: int = 0, s: int = 0, device: int = 0):
        super().__init__([(r >> i) & 1 for i in range(STATE_BITS)], [(s >> i) & 1 for i in range(STATE_BITS)], device)

    @property
    def r(self) -> int:  # type: ignore[override]
        return sum(b << i for i, b in enumerate(self._eng.extract_lane(0).r))

    @property
    def s(self) -> int:  # type: ignore[override]
        return sum(b << i for i, b in enumerate(self._eng.extract_lane(0).s))


def scalar_keystream(material: MickeyKeyIv, nbits: int, device: int = 0) -> list:
    """Convenience: initialise and emit nbits (mickey.py:378-380)."""
    return MickeyScalar.from_key_iv(material, device).keystream_bits(nbits)
