"""ctypes front-end of oracle/mickey_oracle.c -- TEST INFRASTRUCTURE ONLY.

The C file restates the reference's algorithm (citations inside it); this
module only marshals numpy arrays.  It is the *checker* for the CUDA path and
the CPU arm bench.py times beside it.  Nothing under paper_1909_04750_b200/
imports it.

Parity status: pinned by tests/test_oracle.py against the reference's eSTREAM
vectors (pkg/src/slicerng/vectors.py:41-60) and tests/golden/mickey_golden.json
(generated from the reference itself by oracle/gen_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libmickey_oracle.so"
_lib = None

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


def build(force: bool = False) -> Path:
    """Compile the C oracle with the committed Makefile (gcc only)."""
    src = _HERE / "mickey_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(_HERE), "-B", "libmickey_oracle.so"], check=True,
                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    return _LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(_LIB_PATH))
        L.mk2o_tables.argtypes = [u8p]
        L.mk2o_scalar_init.argtypes = [C.c_void_p, u8p, u8p, C.c_int]
        L.mk2o_scalar_clock.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.mk2o_scalar_keystream_bytes.argtypes = [C.c_void_p, C.c_uint64, u8p]
        L.mk2o_scalar_keystream_bits.argtypes = [C.c_void_p, C.c_uint64, u8p]
        L.mk2o_sliced_init.argtypes = [C.c_void_p, u8p, u8p, C.c_int, u8p, C.c_int]
        L.mk2o_sliced_init.restype = C.c_int
        L.mk2o_sliced_clock.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
        L.mk2o_sliced_keystream_words.argtypes = [C.c_void_p, C.c_uint64, u64p]
        L.mk2o_sliced_loop.argtypes = [u64p, u64p, u64p, C.c_uint64]
        for name, outp in (("mk2o_bulk_colmajor", u32p), ("mk2o_bulk_rowmajor", u8p)):
            f = getattr(L, name)
            f.argtypes = [u8p, u8p, C.c_int, u8p, C.c_int, C.c_uint64, C.c_uint64, outp, C.c_int]
            f.restype = C.c_int
        L.mk2o_timed_loops.argtypes = [u64p, u64p, u64p, C.c_uint64, C.c_int, C.c_int]
        L.mk2o_timed_loops.restype = C.c_uint64
        L.mk2o_checksum_colmajor.argtypes = [u32p, C.c_uint64, C.c_uint64, C.c_uint64]
        L.mk2o_checksum_colmajor.restype = C.c_uint64
        L.mk2o_checksum_job.argtypes = [u8p, u8p, C.c_int, u8p, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_uint64, C.c_int, C.POINTER(C.c_int)]
        L.mk2o_checksum_job.restype = C.c_uint64
        L.mk2o_max_threads.restype = C.c_int
        L.mk2o_aes128_encrypt.argtypes = [u8p, u8p, u8p]
        L.mk2o_grain_init.argtypes = [C.c_void_p, u8p, u8p, C.c_int]
        L.mk2o_grain_init.restype = C.c_int
        L.mk2o_grain_keystream_words.argtypes = [C.c_void_p, C.c_uint64, u64p]
        L.mk2o_grain_bulk.argtypes = [u8p, u8p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.mk2o_grain_bulk.restype = C.c_int
        L.mk2o_derive_material.argtypes = [u8p, C.c_uint32, C.c_uint64, C.c_uint64, u8p, u8p]
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def tables() -> dict:
    out = np.zeros((5, 100), np.uint8)
    lib().mk2o_tables(_p(out, u8p))
    return dict(zip(("RTAPS", "COMP0", "COMP1", "FB0", "FB1"), (row.tolist() for row in out)))


def _iv_arrays(iv, iv_nbits=None):
    """Accept bytes (MSB-first) or a 0/1 sequence; return (bytes10, nbits)."""
    if isinstance(iv, (bytes, bytearray)):
        n = 8 * len(iv) if iv_nbits is None else iv_nbits
        buf = bytes(iv) + bytes(10 - len(iv))
    else:
        bits = list(iv)
        n = len(bits)
        bits = bits + [0] * (80 - n)
        buf = np.packbits(np.array(bits, np.uint8)).tobytes()
    if n > 80:
        raise ValueError("IV must be at most 80 bits")
    return np.frombuffer(buf, np.uint8).copy(), n


class Scalar:
    """Bit-serial engine (restates MickeyScalar, mickey.py:101-161)."""

    def __init__(self):
        self._st = np.zeros(200, np.uint8)

    @classmethod
    def from_key_iv(cls, key: bytes, iv=b"") -> "Scalar":
        if len(key) != 10:
            raise ValueError("key must be 10 bytes")
        st = cls()
        ivb, n = _iv_arrays(iv)
        k = np.frombuffer(bytes(key), np.uint8).copy()
        lib().mk2o_scalar_init(st._st.ctypes.data, _p(k, u8p), _p(ivb, u8p), n)
        return st

    @property
    def r(self):
        return self._st[:100].tolist()

    @property
    def s(self):
        return self._st[100:].tolist()

    def clock_kg(self, mixing: bool, bit: int):
        lib().mk2o_scalar_clock(self._st.ctypes.data, int(bool(mixing)), int(bit))

    def keystream_bytes(self, nbytes: int) -> bytes:
        out = np.zeros(nbytes, np.uint8)
        lib().mk2o_scalar_keystream_bytes(self._st.ctypes.data, nbytes, _p(out, u8p))
        return out.tobytes()

    def keystream_bits(self, nbits: int):
        out = np.zeros(nbits, np.uint8)
        lib().mk2o_scalar_keystream_bits(self._st.ctypes.data, nbits, _p(out, u8p))
        return out.tolist()


def pack_materials(materials):
    """[(key, iv)] -> keys u8[n,10], ivs u8[n,10], nbits u8[n]."""
    n = len(materials)
    keys = np.zeros((n, 10), np.uint8)
    ivs = np.zeros((n, 10), np.uint8)
    nb = np.zeros(n, np.uint8)
    for j, (key, iv) in enumerate(materials):
        if len(key) != 10:
            raise ValueError(f"lane {j}: key must be 10 bytes")
        keys[j] = np.frombuffer(bytes(key), np.uint8)
        ivs[j], nb[j] = _iv_arrays(iv)
    return keys, ivs, nb


class Sliced:
    """64-lane column-major engine (restates MickeySliced, mickey.py:236-375)."""

    def __init__(self):
        self._st = np.zeros(200, np.uint64)

    @classmethod
    def from_key_ivs(cls, materials) -> "Sliced":
        keys, ivs, nb = pack_materials(materials)
        st = cls()
        rc = lib().mk2o_sliced_init(st._st.ctypes.data, _p(keys, u8p), _p(ivs, u8p), 10, _p(nb, u8p), len(materials))
        if rc:
            raise ValueError(f"sliced init failed rc={rc}")
        return st

    @property
    def rregs(self):
        return [int(x) for x in self._st[:100]]

    @property
    def sregs(self):
        return [int(x) for x in self._st[100:]]

    def clock_kg(self, mixing: bool, word: int):
        lib().mk2o_sliced_clock(self._st.ctypes.data, int(bool(mixing)), C.c_uint64(word))

    def keystream_words(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        lib().mk2o_sliced_keystream_words(self._st.ctypes.data, n, _p(out, u64p))
        return out


def sliced_words(materials, nclocks: int, width: int = 64) -> np.ndarray:
    """Restates kernels.mickey_sliced_words (kernels.py:189-200)."""
    eng = Sliced.from_key_ivs(materials)
    r = eng._st[:100].copy()
    s = eng._st[100:].copy()
    out = np.zeros(nclocks + nclocks % 2, np.uint64)
    lib().mk2o_sliced_loop(_p(r, u64p), _p(s, u64p), _p(out, u64p), len(out))
    if width < 64:
        out &= np.uint64((1 << width) - 1)
    return out[:nclocks]


def _bulk_args(keys, ivs, iv_bits):
    keys = np.ascontiguousarray(keys, np.uint8).reshape(-1, 10)
    N = keys.shape[0]
    ivs = np.ascontiguousarray(ivs, np.uint8).reshape(N, -1) if np.size(ivs) else np.zeros((N, 1), np.uint8)
    if np.isscalar(iv_bits):
        uniform, nb = int(iv_bits), np.zeros(1, np.uint8)
    else:
        uniform, nb = -1, np.ascontiguousarray(iv_bits, np.uint8)
    if ivs.shape[1] < 10:  # C side may read up to ceil(nbits/8) bytes per row
        ivs = np.ascontiguousarray(np.pad(ivs, ((0, 0), (0, 10 - ivs.shape[1]))))
    return keys, ivs, uniform, nb, N


def bulk_colmajor(keys, ivs, iv_bits, T: int, nthreads: int = 0) -> np.ndarray:
    """uint32 out[T][ceil(N/32)] for N instances (SURVEY.md 8(b) layout)."""
    keys, ivs, uniform, nb, N = _bulk_args(keys, ivs, iv_bits)
    out = np.zeros((T, (N + 31) // 32), np.uint32)
    rc = lib().mk2o_bulk_colmajor(_p(keys, u8p), _p(ivs, u8p), ivs.shape[1], _p(nb, u8p), uniform, N, T,
                                  _p(out, u32p), nthreads)
    if rc:
        raise RuntimeError(f"oracle bulk_colmajor rc={rc}")
    return out


def bulk_rowmajor(keys, ivs, iv_bits, T: int, nthreads: int = 0) -> np.ndarray:
    """uint8 out[N][T/8], MSB-first rows (kernels.py:604-621)."""
    keys, ivs, uniform, nb, N = _bulk_args(keys, ivs, iv_bits)
    if T % 8:
        raise ValueError("bit count must be a multiple of 8")
    out = np.zeros((N, T // 8), np.uint8)
    rc = lib().mk2o_bulk_rowmajor(_p(keys, u8p), _p(ivs, u8p), ivs.shape[1], _p(nb, u8p), uniform, N, T,
                                  _p(out, u8p), nthreads)
    if rc:
        raise RuntimeError(f"oracle bulk_rowmajor rc={rc}")
    return out


def checksum_colmajor(out: np.ndarray, g_offset: int = 0) -> int:
    out = np.ascontiguousarray(out, np.uint32)
    T, G = out.shape
    return int(lib().mk2o_checksum_colmajor(_p(out, u32p), T, G, g_offset))


def checksum_counter(key: bytes, first: int, n: int, T: int, g_offset: int | None = None, nthreads: int = 0) -> int:
    """Checksum of the whole counter-IV job (SURVEY.md 8(d) set: one key, IV_k = 80-bit big-endian k for
    k = first .. first+n-1, T bits each) computed batch by batch without materialising the keystream:
    equals checksum_colmajor(bulk_colmajor(*counter_material(key, first, n), 80, T), first // 32)."""
    if first % 64:
        raise ValueError("first must be a multiple of 64")
    k = np.frombuffer(bytes(key), np.uint8).copy()
    rc = C.c_int(0)
    v = lib().mk2o_checksum_job(_p(k, u8p), None, 10, None, 80, 1, first, n, T,
                                first // 32 if g_offset is None else g_offset, nthreads, C.byref(rc))
    if rc.value:
        raise RuntimeError(f"oracle checksum_counter rc={rc.value}")
    return int(v)


def checksum_material(keys, ivs, iv_bits, T: int, g_offset: int = 0, nthreads: int = 0) -> int:
    """Checksum of bulk_colmajor(keys, ivs, iv_bits, T) without materialising it (every instance, every bit)."""
    keys, ivs, uniform, nb, N = _bulk_args(keys, ivs, iv_bits)
    rc = C.c_int(0)
    v = lib().mk2o_checksum_job(_p(keys, u8p), _p(ivs, u8p), ivs.shape[1], _p(nb, u8p), uniform, 0, 0, N, T, g_offset,
                                nthreads, C.byref(rc))
    if rc.value:
        raise RuntimeError(f"oracle checksum_material rc={rc.value}")
    return int(v)


def counter_material(key: bytes, first: int, n: int):
    """Synthetic set of SURVEY.md 8(d): one key, IV_k = 80-bit big-endian k."""
    keys = np.tile(np.frombuffer(bytes(key), np.uint8), (n, 1))
    ivs = np.zeros((n, 10), np.uint8)
    for j in range(n):
        ivs[j] = np.frombuffer((first + j).to_bytes(10, "big"), np.uint8)
    return keys, ivs


def timed_loops(nclocks: int, nworkers: int, ncalls: int = 1, states: np.ndarray | None = None):
    """Run `nworkers` independent 64-lane keystream loops, each `ncalls` calls of
    `nclocks` clocks (the region the reference's bench times,
    bench.py:169-183, repeated like its `repeats`).  Returns seconds elapsed."""
    import time

    if states is None:
        rng = np.random.default_rng(1)
        states = rng.integers(0, 2**63, size=(nworkers, 200), dtype=np.uint64)
    r = np.ascontiguousarray(states[:, :100])
    s = np.ascontiguousarray(states[:, 100:])
    nclocks += nclocks % 2
    scratch = np.zeros((nworkers, nclocks), np.uint64)
    scratch[:] = 1  # touch pages outside the timed region
    t0 = time.perf_counter()
    lib().mk2o_timed_loops(_p(r, u64p), _p(s, u64p), _p(scratch, u64p), nclocks, ncalls, nworkers)
    return time.perf_counter() - t0


def max_threads() -> int:
    return int(lib().mk2o_max_threads())


ALGO_TAG_MICKEY = 3  # sorted(("aes-ctr", "grain", "mickey")).index("mickey") + 1, seedgen.py:31


def aes128_encrypt(key: bytes, block: bytes) -> bytes:
    k = np.frombuffer(bytes(key), np.uint8).copy()
    b = np.frombuffer(bytes(block), np.uint8).copy()
    out = np.zeros(16, np.uint8)
    lib().mk2o_aes128_encrypt(_p(k, u8p), _p(b, u8p), _p(out, u8p))
    return out.tobytes()


def derive_material(seed: bytes, first_lane: int, n: int, tag: int = ALGO_TAG_MICKEY):
    """Restates seedgen.derive_lane_material (seedgen.py:63-86) for lanes first_lane .. first_lane+n-1."""
    if len(seed) != 32:
        raise ValueError("master seed must be 32 bytes")
    sd = np.frombuffer(bytes(seed), np.uint8).copy()
    keys = np.zeros((n, 10), np.uint8)
    ivs = np.zeros((n, 10), np.uint8)
    lib().mk2o_derive_material(_p(sd, u8p), tag, first_lane, n, _p(keys, u8p), _p(ivs, u8p))
    return keys, ivs


def suite_streams(seed: bytes, nstreams: int, stream_bits: int) -> np.ndarray:
    """Restates cli._suite_streams (cli.py:212-231): batches of 64 lanes, batch b keyed by the master seed with its
    first byte XORed with b, lane material from derive_lane_material, MSB-first packed keystream per lane (a last
    partial byte zero-padded, as np.packbits does).  uint8[nstreams][ceil(stream_bits / 8)]."""
    keys = np.zeros((nstreams, 10), np.uint8)
    ivs = np.zeros((nstreams, 10), np.uint8)
    for b in range((nstreams + 63) // 64):
        lanes = min(64, nstreams - 64 * b)
        k, v = derive_material(bytes([seed[0] ^ b]) + seed[1:], 0, lanes)
        keys[64 * b: 64 * b + lanes], ivs[64 * b: 64 * b + lanes] = k, v
    nbytes = (stream_bits + 7) // 8
    rows = bulk_rowmajor(keys, ivs, 80, 8 * nbytes)
    if stream_bits % 8:
        rows[:, -1] &= np.uint8((0xFF << (8 - stream_bits % 8)) & 0xFF)
    return rows


# ---------------------------------------------------------------- Grain v1 (grain.py)

def _grain_arrays(materials):
    n = len(materials)
    keys = np.zeros((n, 10), np.uint8)
    ivs = np.zeros((n, 8), np.uint8)
    for j, (key, iv) in enumerate(materials):
        if len(key) != 10 or len(iv) != 8:
            raise ValueError(f"lane {j}: key must be 10 bytes and IV 8 bytes")
        keys[j] = np.frombuffer(bytes(key), np.uint8)
        ivs[j] = np.frombuffer(bytes(iv), np.uint8)
    return keys, ivs


class GrainSliced:
    """Up to 64 lanes (restates GrainSliced, grain.py:232-308; 1 lane = GrainScalar :136-173)."""

    def __init__(self):
        self._st = np.zeros(160, np.uint64)

    @classmethod
    def from_key_ivs(cls, materials) -> "GrainSliced":
        keys, ivs = _grain_arrays(materials)
        st = cls()
        rc = lib().mk2o_grain_init(st._st.ctypes.data, _p(keys, u8p), _p(ivs, u8p), len(materials))
        if rc:
            raise ValueError(f"grain init failed rc={rc}")
        return st

    @property
    def b(self):
        return [int(x) for x in self._st[:80]]

    @property
    def s(self):
        return [int(x) for x in self._st[80:]]

    def keystream_words(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        lib().mk2o_grain_keystream_words(self._st.ctypes.data, n, _p(out, u64p))
        return out


def grain_scalar_bytes(key: bytes, iv: bytes, nbytes: int, bit_order: str = "msb") -> bytes:
    words = GrainSliced.from_key_ivs([(key, iv)]).keystream_words(8 * nbytes)
    bits = (words & np.uint64(1)).astype(np.uint8)
    return np.packbits(bits, bitorder="big" if bit_order == "msb" else "little").tobytes()


def grain_bulk_colmajor(keys, ivs, T: int, nthreads: int = 0) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint8).reshape(-1, 10)
    ivs = np.ascontiguousarray(ivs, np.uint8).reshape(-1, 8)
    N = keys.shape[0]
    out = np.zeros((T, (N + 31) // 32), np.uint32)
    rc = lib().mk2o_grain_bulk(_p(keys, u8p), _p(ivs, u8p), N, T, out.ctypes.data, 0, 0, nthreads)
    if rc:
        raise RuntimeError(f"oracle grain bulk rc={rc}")
    return out


def grain_bulk_rowmajor(keys, ivs, T: int, bit_order: str = "msb", nthreads: int = 0) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint8).reshape(-1, 10)
    ivs = np.ascontiguousarray(ivs, np.uint8).reshape(-1, 8)
    N = keys.shape[0]
    if T % 8:
        raise ValueError("bit count must be a multiple of 8")
    out = np.zeros((N, T // 8), np.uint8)
    rc = lib().mk2o_grain_bulk(_p(keys, u8p), _p(ivs, u8p), N, T, out.ctypes.data, 1, int(bit_order == "lsb"), nthreads)
    if rc:
        raise RuntimeError(f"oracle grain bulk rc={rc}")
    return out
