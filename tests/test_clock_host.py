"""clock_block<K> (csrc/mk2_clock.cuh: K clocks with R's feedback reduction deferred) checked on the
CPU: the header is compiled as host C++ (tests/host_clock_check.cpp, truth tables in software) and
compared with the one-clock form and with the oracle's sliced engine (mickey.py:329-360) on random
states -- every block length, with and without mixing / input words.  The GPU parity tests cover the
same code as SASS; this one needs no GPU."""
import ctypes as C
import random
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import mickey_oracle as orc

HERE = Path(__file__).resolve().parent
pytestmark = pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
u32p = C.POINTER(C.c_uint32)


@pytest.fixture(scope="module")
def hc(tmp_path_factory):
    so = tmp_path_factory.mktemp("hc") / "libhostclock.so"
    subprocess.run(["g++", "-std=c++17", "-O1", "-shared", "-fPIC", "-o", str(so), str(HERE / "host_clock_check.cpp")],
                   check=True)
    lib = C.CDLL(str(so))
    lib.hc_plain.argtypes = [u32p, u32p, C.c_int, C.c_int, u32p, C.c_int, u32p]
    lib.hc_block.argtypes = [C.c_int, u32p, u32p, C.c_int, C.c_int, u32p, u32p]
    lib.hc_block_masked.argtypes = [C.c_int, u32p, u32p, u32p, u32p]
    lib.hc_transpose32.argtypes = [u32p]
    lib.hc_ragged_group.argtypes = [u32p, u32p, C.c_int, u32p, u32p]
    return lib


def _p(a):
    return a.ctypes.data_as(u32p)


def _oracle_steps(r, s, mixing, words):
    """The oracle's 64-lane engine on the same 32 lanes (upper lanes zero)."""
    eng = orc.Sliced()
    eng._st[:100] = r.astype(np.uint64)
    eng._st[100:] = s.astype(np.uint64)
    z = []
    for w in words:
        z.append((int(eng._st[0]) ^ int(eng._st[100])) & 0xFFFFFFFF)
        eng.clock_kg(mixing, int(w))
    low = eng._st & np.uint64(0xFFFFFFFF)
    return low[:100].astype(np.uint32), low[100:].astype(np.uint32), np.array(z, np.uint32)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("mixing,has_in", [(False, False), (True, False), (True, True), (False, True)])
def test_block_equals_plain_clock_and_oracle(hc, K, mixing, has_in):
    rng = random.Random(1000 * K + 10 * mixing + has_in)
    for trial in range(8):
        r0 = np.array([rng.getrandbits(32) for _ in range(100)], np.uint32)
        s0 = np.array([rng.getrandbits(32) for _ in range(100)], np.uint32)
        if trial == 0:                       # lock-step lanes: every word 0 or all-ones (tests/test_mickey.py:111-117)
            r0 = np.where(r0 & 1, 0xFFFFFFFF, 0).astype(np.uint32)
            s0 = np.where(s0 & 1, 0xFFFFFFFF, 0).astype(np.uint32)
        nblocks = 3
        words = np.array([rng.getrandbits(32) if has_in else 0 for _ in range(K * nblocks)], np.uint32)
        rp, sp, zp = r0.copy(), s0.copy(), np.zeros(K * nblocks, np.uint32)
        hc.hc_plain(_p(rp), _p(sp), mixing, has_in, _p(words), K * nblocks, _p(zp))
        rb, sb, zb = r0.copy(), s0.copy(), np.zeros(K * nblocks, np.uint32)
        for b in range(nblocks):             # reduced state in, reduced state out: blocks chain
            win, zout = words[b * K:(b + 1) * K].copy(), np.zeros(K, np.uint32)
            assert hc.hc_block(K, _p(rb), _p(sb), mixing, has_in, _p(win), _p(zout)) == 0
            zb[b * K:(b + 1) * K] = zout
        ro, so, zo = _oracle_steps(r0, s0, mixing, words)
        assert np.array_equal(rp, ro) and np.array_equal(sp, so) and np.array_equal(zp, zo), "one-clock form vs oracle"
        assert np.array_equal(rb, ro) and np.array_equal(sb, so) and np.array_equal(zb, zo), "block form vs oracle"


def test_overflow_patterns_are_powers_of_x_mod_p(hc):
    """Q_j = x^(100+j) mod (x^100 + RTAPS): the compile-time table the reduction is generated from."""
    taps = [i for i, b in enumerate(orc.tables()["RTAPS"]) if b]
    q = sum(1 << i for i in taps)            # x^100 = T(x)
    for j in range(6):
        assert [hc.hc_q_bit(j, i) for i in range(100)] == [(q >> i) & 1 for i in range(100)], j
        q <<= 1
        if (q >> 100) & 1:
            q = (q & ((1 << 100) - 1)) ^ sum(1 << i for i in taps)


def test_block_costs_fewer_lop3_than_plain_clocks(hc):
    counts = {K: hc.hc_block_lop3_count(K) for K in range(1, 7)}
    assert counts[1] in (327, 328)           # degenerate block = the plain clock (+1: r0 handled separately)
    for K in range(2, 7):
        assert counts[K] / K < counts[K - 1] / (K - 1)
    assert counts[4] == 1213 and counts[5] == 1503 and counts[6] == 1794


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_masked_block_holds_late_lanes_in_the_zero_state(hc, K):
    """clock_block_masked<K> (ragged IV lengths: a lane with a shorter IV joins later) against the plain
    semantics -- clock every lane, then force the lanes that have not started back to zero -- and, lane by lane,
    against the oracle's engine started at the lane's own first clock (mickey.py:287-289: per-lane init)."""
    rng = random.Random(77 + K)
    nclocks = 3 * K
    for trial in range(6):
        start = [rng.randrange(0, nclocks + 1) for _ in range(32)]        # lane j's first active clock
        act = np.array([sum((c >= start[j]) << j for j in range(32)) for c in range(nclocks)], np.uint32)
        words = np.array([rng.getrandbits(32) for _ in range(nclocks)], np.uint32) & act   # idle lanes carry zero input
        r = np.zeros(100, np.uint32)
        s = np.zeros(100, np.uint32)
        rp, sp = r.copy(), s.copy()
        z = np.zeros(1, np.uint32)
        for c in range(nclocks):                                          # reference semantics, one clock at a time
            hc.hc_plain(_p(rp), _p(sp), 1, 1, _p(words[c:c + 1].copy()), 1, _p(z))
            rp &= act[c]
            sp &= act[c]
        for b in range(nclocks // K):
            assert hc.hc_block_masked(K, _p(r), _p(s), _p(words[b * K:(b + 1) * K].copy()), _p(act[b * K:(b + 1) * K].copy())) == 0
        assert np.array_equal(r, rp) and np.array_equal(s, sp)
        for j in (0, 7, 31):                                              # per-lane: the oracle started at clock start[j]
            eng = orc.Sliced()
            for c in range(start[j], nclocks):
                eng.clock_kg(True, (int(words[c]) >> j) & 1)
            assert [(int(x) >> j) & 1 for x in r] == [int(x) & 1 for x in eng._st[:100]]
            assert [(int(x) >> j) & 1 for x in s] == [int(x) & 1 for x in eng._st[100:]]
    assert hc.hc_zero_leak_extra_ops() == 5


def test_transpose32_and_ragged_group_packing(hc):
    """The bit-matrix helpers of pack_ragged_kernel's fast path (csrc/mk2_bits.cuh) against plain Python: lane j
    with L_j IV bits idles for lmax - L_j clocks and then feeds its IV bits MSB-first (bitops.py:33-36)."""
    rng = random.Random(5)
    a = np.array([rng.getrandbits(32) for _ in range(32)], np.uint32)
    t = a.copy()
    hc.hc_transpose32(_p(t))
    assert all(((int(t[b]) >> j) & 1) == ((int(a[j]) >> b) & 1) for b in range(32) for j in range(32))
    for trial in range(20):
        ivs = np.array([[rng.getrandbits(8) for _ in range(10)] for _ in range(32)], np.uint8)
        lens = [rng.choice([0, 1, 7, 8, 31, 32, 33, 63, 64, 65, 79, 80, 0xFF, rng.randrange(81)]) for _ in range(32)]
        real = [l for l in lens if l <= 80]
        lmax = max(real) if real and trial % 5 else 80
        inw = np.zeros(96, np.uint32)
        act = np.zeros(96, np.uint32)
        hc.hc_ragged_group(_p(ivs.reshape(-1).view("<u4").copy()), _p(np.array(lens, np.uint8).view("<u4").copy()), lmax,
                           _p(inw), _p(act))
        for c in range(96):
            want_in = want_act = 0
            for j, L in enumerate(lens):
                if L > 80 or c >= lmax or c < lmax - L:
                    continue
                want_act |= 1 << j
                cc = c - (lmax - L)
                want_in |= ((int(ivs[j, cc >> 3]) >> (7 - (cc & 7))) & 1) << j
            assert int(inw[c]) == want_in and int(act[c]) == want_act, (trial, c)
