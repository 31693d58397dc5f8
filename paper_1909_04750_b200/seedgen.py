"""Host mirror of the reference's seed derivation (pkg/src/slicerng/seedgen.py).

Same names and validation as the reference (`MasterSeed`, `SeedError`,
`derive_lane_material`, `derive_all`), but the AES-128 counter construction
runs in csrc/mk2_seedgen.cuh, one GPU thread per lane, and the reference's
64-lane cap (seedgen.py:22) is lifted to the 2^32 lanes the derivation block's
lane field can address.  Only the MICKEY tag is served here (the other
ciphers are outside this repo's path).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import hostmem
from .generator import MickeyGenerator
from .mickey import MickeyKeyIv

SEED_BYTES = 32
MAX_LANES = 1 << 32          # reference: 64 (seedgen.py:22)
REFERENCE_MAX_LANES = 64
_ALGO_TAGS = {"aes-ctr": 1, "grain": 2, "mickey": 3}  # sorted names, seedgen.py:31


class SeedError(ValueError):
    """Invalid master seed or lane request (seedgen.py:34-35)."""


@dataclass(frozen=True)
class MasterSeed:
    """256-bit master entropy value with its target algorithm and lane count (seedgen.py:38-54)."""

    seed: bytes
    algo: str = "mickey"
    lanes: int = REFERENCE_MAX_LANES

    def __post_init__(self):
        if len(self.seed) != SEED_BYTES:
            raise SeedError(f"master seed must be {SEED_BYTES} bytes")
        if self.seed == bytes(SEED_BYTES):
            raise SeedError("all-zero master seed rejected")
        if self.algo not in _ALGO_TAGS:
            raise SeedError(f"unknown algorithm {self.algo!r}")
        if self.algo != "mickey":
            raise SeedError(f"algorithm {self.algo!r} is not on the GPU path of this package")
        if not 1 <= self.lanes <= MAX_LANES:
            raise SeedError(f"lane count must be in [1, {MAX_LANES}]")


def derive_arrays(master: MasterSeed, first_lane: int = 0, n: int | None = None, device: int = 0):
    """keys u8[n,10], ivs u8[n,10] for lanes first_lane .. first_lane+n-1 (computed on the GPU)."""
    n = master.lanes - first_lane if n is None else n
    if first_lane < 0 or n < 1 or first_lane + n > master.lanes:
        raise IndexError(f"lanes [{first_lane}, {first_lane + n}) out of range [0, {master.lanes})")
    with hostmem.borrow_context(MickeyGenerator, device) as gen:
        return gen.derive_material(master.seed, first_lane, n)


def derive_lane_material(master: MasterSeed, lane: int, device: int = 0) -> MickeyKeyIv:
    """Key/IV material for one lane (seedgen.py:63-86)."""
    if not 0 <= lane < master.lanes:
        raise IndexError(f"lane {lane} out of range [0, {master.lanes})")
    keys, ivs = derive_arrays(master, lane, 1, device)
    return MickeyKeyIv(keys[0].tobytes(), ivs[0].tobytes())


def derive_all(master: MasterSeed, device: int = 0) -> list:
    """Material for every lane of the master seed (seedgen.py:89-91)."""
    keys, ivs = derive_arrays(master, 0, master.lanes, device)
    return [MickeyKeyIv(keys[j].tobytes(), ivs[j].tobytes()) for j in range(master.lanes)]
