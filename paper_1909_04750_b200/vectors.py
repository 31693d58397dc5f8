"""Host mirror of the reference's MICKEY test-vector module (pkg/src/slicerng/vectors.py).

The three records are the cipher's published eSTREAM vectors (vectors.py:41-60);
`verify_vectors("mickey")` checks every lane of the GPU engine at both lane
widths, the way the reference checks its sliced engine (vectors.py:154-198).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import mickey

LANE_CHECK_WIDTHS = (32, 64)


@dataclass(frozen=True)
class VectorRecord:
    algo: str
    key: bytes
    iv: bytes
    ks: bytes
    bit_order: str = "msb"
    kind: str = "keystream"

    def format_line(self) -> str:
        return f"key={self.key.hex()} iv={self.iv.hex()} ks={self.ks.hex()}"


_K = bytes.fromhex("123456789abcdef01234")
MICKEY_VECTORS = (
    VectorRecord("mickey", _K, bytes.fromhex("21436587"), bytes.fromhex("9821e10c5ed28d32bbc3d1fb15e93a15")),
    VectorRecord("mickey", _K, b"", bytes.fromhex("92f1b8779b47da74075e7a8ccc23c80c")),
    VectorRecord("mickey", _K, bytes.fromhex("21436587a9cbed0f2143"), bytes.fromhex("804c60856af63516c8f21827bd81f6be")),
)
GRAIN_VECTORS = (  # published Grain v1 vectors, LSB-first convention (vectors.py:62-77)
    VectorRecord("grain", bytes(10), bytes(8), bytes.fromhex("dee931cf1662a72f77d02b6b6188a8f6"), bit_order="lsb"),
    VectorRecord("grain", bytes.fromhex("0123456789abcdef1234"), bytes.fromhex("0123456789abcdef"),
                 bytes.fromhex("7f362bd3f7abae2036642fe0bd2aafad"), bit_order="lsb"),
)
ALL_VECTORS = {"mickey": MICKEY_VECTORS, "grain": GRAIN_VECTORS}


class VectorMismatch(AssertionError):
    """The engine failed to reproduce an embedded or file vector."""


def parse_vector_file(text: str, algo: str = "mickey", bit_order: str = "msb"):
    """`key=<hex> iv=<hex> ks=<hex>` lines; '#' starts a comment (docs/conventions.md:66-74)."""
    records = []
    for lineno, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        fields = dict(part.split("=", 1) for part in line.split() if "=" in part)
        if not {"key", "ks"} <= set(fields):
            raise ValueError(f"line {lineno}: expected key=<hex> iv=<hex> ks=<hex>")
        try:   # a missing iv= means the empty IV (vectors.py:120)
            records.append(VectorRecord(algo, bytes.fromhex(fields["key"]), bytes.fromhex(fields.get("iv", "")),
                                        bytes.fromhex(fields["ks"]), bit_order))
        except ValueError as exc:
            raise ValueError(f"line {lineno}: {exc}") from exc
    return records


def verify_vectors(algo: str = "mickey", records=None, device: int = 0):
    """(records checked, failure descriptions): every lane at W = 32 and 64 on the GPU."""
    if algo not in ALL_VECTORS:
        raise ValueError(f"algorithm {algo!r} is not on the GPU path of this package")
    from . import grain

    records = ALL_VECTORS[algo] if records is None else records
    failures = []
    for rec in records:
        for width in LANE_CHECK_WIDTHS:
            if algo == "mickey":
                eng = mickey.MickeySliced.from_key_ivs([mickey.MickeyKeyIv(rec.key, rec.iv)] * width, width=width,
                                                       device=device)
            else:
                eng = grain.GrainSliced.from_key_ivs([grain.GrainKeyIv(rec.key, rec.iv)] * width, width=width,
                                                     device=device)
            words = np.array(eng.keystream_words(8 * len(rec.ks)), np.uint64)
            for j in range(width):
                bits = ((words >> np.uint64(j)) & np.uint64(1)).astype(np.uint8)
                got = np.packbits(bits, bitorder="big" if rec.bit_order == "msb" else "little").tobytes()
                if got != rec.ks:
                    failures.append(f"{algo} width {width} lane {j}: {rec.format_line()} got {got.hex()}")
                    break
    return len(records), failures
