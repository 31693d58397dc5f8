"""GPU parity: the CUDA path (through the C ABI) vs the oracle and the goldens.

Bit-exact is the bar (integer / bit work).  Mirrors the reference's test
strategy for this path: KATs on every lane, the
sliced<->scalar differential, lock-step symmetry, ragged / odd-length edges,
resumability, and -- at BASELINE.json's instance counts -- sampled groups plus
layout-independent checksums.
"""
import hashlib

import numpy as np
import pytest

from conftest import golden_material

pytestmark = pytest.mark.gpu


def sha(b):
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def pkg():
    import paper_1909_04750_b200 as p

    assert p._native.lib().mk2_device_count() >= 1, "no CUDA device: GPU tests cannot run"
    return p


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    assert torch.cuda.is_available()
    return torch


@pytest.fixture(autouse=True, params=["small-batch-kernels", "throughput-kernels"])
def kernel_family(request, monkeypatch):
    """Every test of this file runs twice: with new contexts using the warp-per-group kernels for small batches
    (the default, csrc/mk2_coop.cuh) and with the thread-per-group throughput kernels at every size -- most cases
    here are small, and the tails, tile boundaries and staging modes of BOTH families must stay covered."""
    from paper_1909_04750_b200 import generator, hostmem

    monkeypatch.setattr(generator, "DEFAULT_SMALL_BATCH", request.param == "small-batch-kernels")
    monkeypatch.setenv("MK2_SMALL_BATCH", "1" if request.param == "small-batch-kernels" else "0")   # child processes
    hostmem.drop_idle_contexts()      # pooled contexts were created under the other setting
    yield request.param
    hostmem.drop_idle_contexts()


def mats_of(pkg, recs):
    return [pkg.MickeyKeyIv(*golden_material(r)) for r in recs]


def random_arrays(seed, n, iv_bytes=10):
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 256, (n, 10), dtype=np.uint8), rng.integers(0, 256, (n, iv_bytes), dtype=np.uint8))


# ---------------------------------------------------------------- reference-shaped API

@pytest.mark.parametrize("width", [32, 64])
def test_estream_vectors_every_lane(pkg, golden, width):
    # tests/test_mickey.py:44-47 -> vectors.verify_vectors (vectors.py:189-197)
    for rec in golden["kats"]:
        m = pkg.MickeyKeyIv(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"]))
        eng = pkg.MickeySliced.from_key_ivs([m] * width, width=width)
        st = eng.extract_lane(width - 1)
        assert f"{sum(b << i for i, b in enumerate(st.r)):x}" == rec["post_init_r"]
        assert f"{sum(b << i for i, b in enumerate(st.s)):x}" == rec["post_init_s"]
        lanes = eng.keystream_lane_bits(128)
        for j in range(width):
            assert np.packbits(np.array(lanes[j], np.uint8)).tobytes() == bytes.fromhex(rec["ks"]), (rec["iv"], j)


def test_golden_sliced_cases(pkg, golden):
    # kernels.mickey_sliced_words + MickeySliced init state, uniform / ragged / short / bit-length IVs
    for case in golden["sliced_cases"]:
        mats = mats_of(pkg, case["materials"])
        width = case["width"]
        eng = pkg.MickeySliced.from_key_ivs(mats, width=width)
        assert [f"{w:x}" for w in eng.rregs] == case["init_state"]["r"], case["name"]
        assert [f"{w:x}" for w in eng.sregs] == case["init_state"]["s"], case["name"]
        words = pkg.mickey_sliced_words(mats, case["nclocks"], width)
        assert words.dtype == np.uint64 and words.shape == (case["nclocks"],)
        assert sha(words.astype("<u8").tobytes()) == case["words_sha256"], case["name"]
        if width == 32:
            assert int(words.max()) < (1 << 32)  # tests/test_kernels.py:85-88


def test_sliced_words_match_oracle_odd_count(pkg, oracle):
    # tests/test_kernels.py:20-25 (501 clocks: odd count)
    import random

    rng = random.Random(0xFA57)
    raw = [(rng.randbytes(10), rng.randbytes(4)) for _ in range(64)]
    for width, count in ((32, 32), (64, 64)):
        got = pkg.mickey_sliced_words([pkg.MickeyKeyIv(k, iv) for k, iv in raw[:count]], 501, width)
        want = oracle.sliced_words(raw[:count], 501, width)
        assert np.array_equal(got, want)


def test_lockstep_words_uniform(pkg, golden, oracle):
    # tests/test_mickey.py:148-154
    rec = golden["kats"][0]
    m = pkg.MickeyKeyIv(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"]))
    eng = pkg.MickeySliced.from_key_ivs([m] * 32, width=32)
    bits = oracle.Scalar.from_key_iv(m.key, m.iv).keystream_bits(128)
    for word, bit in zip(eng.keystream_words(128), bits):
        assert word == (0xFFFFFFFF if bit else 0)


def test_zero_length_request_keeps_state_and_resume(pkg, golden):
    # tests/test_mickey.py:167-171 + resumability of keystream_words (mickey.py:362-368)
    mats = mats_of(pkg, golden["sliced_cases"][1]["materials"])
    eng = pkg.MickeySliced.from_key_ivs(mats, width=64)
    before = (eng.rregs, eng.sregs)
    assert eng.keystream_words(0) == []
    assert (eng.rregs, eng.sregs) == before
    a = eng.keystream_words(100) + eng.keystream_words(157)
    whole = pkg.MickeySliced.from_key_ivs(mats, width=64).keystream_words(257)
    assert a == whole


def test_clock_kg_and_state_constructor(pkg, oracle):
    # MickeySliced(rregs, sregs, width) + clock_kg(mixing, word) (mickey.py:245-253, 329-360)
    rng = np.random.default_rng(3)
    r = [int(x) for x in rng.integers(0, 2**63, 100, dtype=np.uint64)]
    s = [int(x) for x in rng.integers(0, 2**63, 100, dtype=np.uint64)]
    eng = pkg.MickeySliced(r, s, 64)
    ref = oracle.Sliced()
    ref._st[:100] = r
    ref._st[100:] = s
    for mixing, word in ((True, 0x0123456789ABCDEF), (False, 0), (True, 0), (False, 0xFFFFFFFF00000000)):
        eng.clock_kg(mixing, word)
        ref.clock_kg(mixing, word)
        assert eng.rregs == ref.rregs and eng.sregs == ref.sregs
    assert eng.keystream_words(33) == [int(w) for w in ref.keystream_words(33)]
    with pytest.raises(ValueError):
        pkg.MickeySliced(r[:99], s, 64)


def test_c1_config_million_bits(pkg, golden):
    # BASELINE config 1: 32 lock-step instances, test-vector key/IV, 1 Mbit each
    for rec in golden["kats"]:
        m = pkg.MickeyKeyIv(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"]))
        words = pkg.mickey_sliced_words([m] * 32, 1_000_000, 32)
        assert sha(words.astype("<u4").tobytes()) == rec["c1_words_u4_sha256"]
        lane0 = pkg.words_to_lane_bytes(words, 0)
        assert sha(lane0) == rec["c1_lane0_sha256"] and lane0[-16:].hex() == rec["c1_lane0_tail16"]


def test_bench_seed_lanes_both_layouts(pkg, golden):
    b = golden["bench_seed"]
    mats = mats_of(pkg, b["materials"])
    words = pkg.mickey_sliced_words(mats, b["nclocks"], 64)
    assert sha(words.astype("<u8").tobytes()) == b["words_u8_sha256"]
    keys, ivs, nbits, _ = pkg.mickey.pack_materials(mats, 64)
    with pkg.MickeyGenerator(0) as gen:
        gen.init_material(keys, ivs, 80)
        row = gen.generate_rowmajor(b["nclocks"])
        assert sha(row.tobytes()) == b["lane_major_sha256"]
        assert f"{gen.checksum():x}" == b["u64_wrap_sum"]


# ---------------------------------------------------------------- bulk C-ABI paths

@pytest.mark.parametrize("iv_bits", [0, 1, 13, 32, 77, 80])
def test_bulk_colmajor_uniform_vs_oracle(pkg, oracle, iv_bits):
    N, T = 2048 + 96, 301
    keys, ivs = random_arrays(100 + iv_bits, N)
    got = pkg.bulk_colmajor(keys, ivs, iv_bits, T)
    want = oracle.bulk_colmajor(keys, ivs, iv_bits, T)
    assert got.shape == want.shape == (T, N // 32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("N,T", [(1000, 1408), (32, 8), (4099, 136), (64, 1024 + 120)])
def test_bulk_rowmajor_vs_oracle_ragged_shapes(pkg, oracle, N, T):
    # N not a multiple of 32, T with a tail past the 128-clock tiles
    keys, ivs = random_arrays(N + T, N)
    got = pkg.bulk_rowmajor(keys, ivs, 80, T)
    want = oracle.bulk_rowmajor(keys, ivs, 80, T)
    assert got.shape == (N, T // 8)
    assert np.array_equal(got, want)


def test_bulk_ragged_iv_lengths_with_unused_lanes(pkg, oracle):
    N, T = 777, 264
    rng = np.random.default_rng(42)
    keys, ivs = random_arrays(9, N)
    nbits = rng.integers(0, 81, N, dtype=np.uint8)
    got_c = pkg.bulk_colmajor(keys, ivs, nbits, T)
    got_r = pkg.bulk_rowmajor(keys, ivs, nbits, T)
    assert np.array_equal(got_r, oracle.bulk_rowmajor(keys, ivs, nbits, T))
    want_c = oracle.bulk_colmajor(keys, ivs, nbits, T)
    # the oracle pads a ragged 64-lane batch with zero-state lanes; so does MK2_IV_UNUSED
    assert np.array_equal(got_c, want_c)
    # explicit unused lanes in the middle behave as zero-state lanes
    nb2 = nbits.copy()
    nb2[5] = nb2[700] = pkg._native.MK2_IV_UNUSED
    with pkg.MickeyGenerator(0) as gen:
        gen.init_ragged(keys, ivs, nb2)
        rs = gen.export_state()
        assert not ((rs[:, 5 // 32] >> np.uint32(5 % 32)) & 1).any()
        assert not ((rs[:, 700 // 32] >> np.uint32(700 % 32)) & 1).any()
        col = gen.generate_colmajor(64)
    keep = np.ones(N, bool)
    keep[[5, 700]] = False
    bits_got = (col[:, np.arange(N) // 32] >> (np.arange(N) % 32).astype(np.uint32)) & 1
    bits_want = (want_c[:64, np.arange(N) // 32] >> (np.arange(N) % 32).astype(np.uint32)) & 1
    assert np.array_equal(bits_got[:, keep], bits_want[:, keep])


def test_counter_iv_sets_golden_and_oracle(pkg, golden, oracle):
    for c in golden["counter_iv"]:
        key = bytes.fromhex(c["key"])
        with pkg.MickeyGenerator(0) as gen:
            gen.init_counter(key, c["first"], c["n"])
            col = gen.generate_colmajor(c["nclocks"])
            assert sha(col.tobytes()) == c["colmajor_sha256"]
            assert f"{gen.checksum():x}" == c["u64_wrap_sum"]
            gen.init_counter(key, c["first"], c["n"])
            row = gen.generate_rowmajor(c["nclocks"])
            assert sha(row.tobytes()) == c["rowmajor_sha256"]
            assert f"{gen.checksum():x}" == c["u64_wrap_sum"]  # layout independent
    # explicit material == synthesised material
    keys, ivs = oracle.counter_material(key, 1 << 33, 160)
    with pkg.MickeyGenerator(0) as gen:
        a = gen.init_counter(key, 1 << 33, 160).generate_colmajor(96)
        b = gen.init_material(keys, ivs, 80).generate_colmajor(96)
    assert np.array_equal(a, b)
    with pytest.raises(ValueError):
        pkg.MickeyGenerator(0).init_counter(key, 7, 64)


def test_state_export_import_resume(pkg, oracle):
    keys, ivs = random_arrays(77, 320)
    with pkg.MickeyGenerator(0) as gen:
        gen.init_material(keys, ivs, 80)
        first = gen.generate_colmajor(200)
        rs = gen.export_state()
        rest = gen.generate_colmajor(123)
        with pkg.MickeyGenerator(0) as gen2:
            gen2.import_state(rs, 320)
            assert np.array_equal(gen2.generate_colmajor(123), rest)
        assert gen.clocks == 323 and gen.instances == 320 and gen.groups == 10
    want = oracle.bulk_colmajor(keys, ivs, 80, 323)
    assert np.array_equal(np.vstack([first, rest]), want)


def test_device_buffers_strides_and_chunked_rows(pkg, oracle, torch_cuda):
    torch = torch_cuda
    N, T = 4096, 512
    keys, ivs = random_arrays(5, N)
    want_c = oracle.bulk_colmajor(keys, ivs, 80, T)
    want_r = oracle.bulk_rowmajor(keys, ivs, 80, T)
    dk, di = torch.from_numpy(keys).cuda(), torch.from_numpy(ivs).cuda()
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        # device material, device output with a wider stride (a shard inside a bigger array)
        gen.init_material(dk, di, 80)
        out = torch.zeros((T, 200), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, out[:, 40:].data_ptr(), stride_words=200)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint32)
        assert np.array_equal(got[:, 40:40 + N // 32], want_c) and not got[:, :40].any() and not got[:, 168:].any()
        # row-major into a device tensor, filled in three calls (256 + 128 + 128 clocks)
        gen.init_material(dk, di, 80)
        rows = torch.zeros((N, T // 8), dtype=torch.uint8, device="cuda")
        gen.generate_rowmajor(256, rows, byte_offset=0)
        gen.generate_rowmajor(128, rows, byte_offset=32)
        gen.generate_rowmajor(128, rows, byte_offset=48)
        torch.cuda.synchronize()
        assert np.array_equal(rows.cpu().numpy(), want_r)
        # unaligned pitch takes the byte-store path
        gen.init_material(dk, di, 80)
        rows2 = torch.zeros((N, 67), dtype=torch.uint8, device="cuda")
        gen.generate_rowmajor(T, rows2.data_ptr() + 3, pitch_bytes=67)
        torch.cuda.synchronize()
        assert np.array_equal(rows2.cpu().numpy()[:, 3:3 + 64], want_r)
        gen.set_stream(None)
    # host output with a stride (staged path)
    with pkg.MickeyGenerator(0) as gen:
        gen.init_material(keys, ivs, 80)
        host = np.zeros((T, 150), np.uint32)
        gen.generate_colmajor(T, host, stride_words=150)
        assert np.array_equal(host[:, :128], want_c) and not host[:, 128:].any()


def test_trim_keeps_state(pkg, oracle):
    keys, ivs = random_arrays(8, 2048)
    with pkg.MickeyGenerator(0) as gen:
        gen.init_material(keys, ivs, 80)
        a = gen.generate_rowmajor(256)
        gen.trim()
        b = gen.generate_rowmajor(256)
    assert np.array_equal(np.hstack([a, b]), oracle.bulk_rowmajor(keys, ivs, 80, 512))


def test_error_paths(pkg):
    gen = pkg.MickeyGenerator(0)
    with pytest.raises(pkg.Mk2Error, match="mk2_init"):
        gen.generate_colmajor(8)
    keys, ivs = random_arrays(1, 64)
    gen.init_material(keys, ivs, 80)
    with pytest.raises(ValueError):
        gen.generate_rowmajor(12)
    with pytest.raises(ValueError):
        gen.generate_colmajor(8, np.zeros((8, 1), np.uint32), stride_words=1)
    with pytest.raises(ValueError):
        gen.init_material(keys, ivs[:, :4], 80)
    with pytest.raises(ValueError):
        gen.init_material(keys[:, :9], ivs, 80)
    with pytest.raises(ValueError, match="lane 3"):
        nb = np.full(64, 8, np.uint8)
        nb[3] = 81
        gen.init_ragged(keys, ivs, nb)
    gen.close()


def test_sharded_checksum_is_invariant(pkg, golden):
    # the checksum over disjoint instance ranges is the same at D = 1, 2, 4
    key = bytes.fromhex(golden["counter_iv"][0]["key"])
    n, T = 4096 + 64, 256
    sums = {}
    for world in (1, 2, 4):
        total = 0
        for rank in range(world):
            gen, sh = pkg.sharding.counter_generator(key, n, world, rank)
            with gen:
                gen.generate_colmajor(T)
                total = (total + gen.checksum()) % (1 << 64)
        sums[world] = total
    assert sums[1] == sums[2] == sums[4]


# ---------------------------------------------------------------- BASELINE-size properties

def _sample_groups_vs_oracle(oracle, key, first, col_t, groups, T):
    """col_t: torch int32 [T][G] on device; compare sampled 64-lane pairs of groups with the oracle."""
    for g in groups:
        g &= ~1
        keys, ivs = oracle.counter_material(key, first + 32 * g, 64)
        want = oracle.bulk_colmajor(keys, ivs, 80, T)
        got = col_t[:, g:g + 2].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want), f"group {g}"


def test_c2_instance_count_sampled_and_checksummed(pkg, golden, oracle, torch_cuda):
    """BASELINE config 2 geometry (2^20 instances, column-major): a 4096-clock slice of the
    stream, sampled groups bit-exact vs the oracle, and the in-kernel checksum equal to a
    checksum recomputed from the emitted buffer; then the same instances row-major give the
    same checksum (layout independence) and equal bits on sampled rows."""
    torch = torch_cuda
    key = bytes.fromhex(golden["kats"][0]["key"])
    N, T = 1 << 20, 4096
    G = N // 32
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        gen.init_counter(key, 0, N)
        col = torch.empty((T, G), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, col)
        torch.cuda.synchronize()
        rng = np.random.default_rng(0)
        _sample_groups_vs_oracle(oracle, key, 0, col, [0, G - 2] + rng.integers(0, G, 6).tolist(), T)
        # checksum recomputed from the buffer: sum of the [T][G] buffer read as u64 words
        as_u64 = col.view(torch.int64)
        assert (int(as_u64.sum().item()) % (1 << 64)) == gen.checksum()
        # two half-length calls == one call (resume at scale)
        gen.init_counter(key, 0, N)
        col2 = torch.empty_like(col)
        gen.generate_colmajor(T // 2, col2[: T // 2])
        gen.generate_colmajor(T // 2, col2[T // 2:])
        torch.cuda.synchronize()
        assert torch.equal(col, col2)
        csum = gen.checksum()
        # row-major of the same instances
        gen.init_counter(key, 0, N)
        rows = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
        gen.generate_rowmajor(T, rows)
        torch.cuda.synchronize()
        assert gen.checksum() == csum
        for n in (0, 31, 32, 12345, N - 1):
            keys, ivs = oracle.counter_material(key, n, 1)
            assert rows[n].cpu().numpy().tobytes() == oracle.bulk_rowmajor(keys, ivs, 80, T)[0].tobytes()
        # the transposed device buffer equals the row-major one on a sampled block of 64 rows
        blk = col[:, 100:102].cpu().numpy().view(np.uint32)
        bits = (blk[:, np.arange(64) // 32] >> (np.arange(64) % 32).astype(np.uint32)) & 1
        assert np.array_equal(np.packbits(bits.T.astype(np.uint8), axis=1), rows[3200:3264].cpu().numpy())
        gen.set_stream(None)


def _rowmajor_buffer_checksum(torch, rows, g_offset=0):
    """The checksum (sum of the column-major stream as u64 words) recomputed from a ROW-major device buffer:
    sum_n popcount(row n) << ((n + 32 g_offset) % 64), mod 2^64."""
    lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=rows.device)
    N = rows.shape[0]
    total = 0
    step = max(1, (1 << 25) // max(1, rows.shape[1]))
    for n0 in range(0, N, step):
        blk = rows[n0:n0 + step]
        pc = lut[blk.long()].sum(dim=1)
        sh = (torch.arange(n0, n0 + blk.shape[0], device=rows.device, dtype=torch.int64) + 32 * (g_offset & 1)) % 64
        total = (total + int(torch.bitwise_left_shift(pc, sh).sum().item())) % (1 << 64)
    return total


def test_full_coverage_checksum_c2_geometry(pkg, golden, oracle, torch_cuda):
    """EVERY instance and chain of the BASELINE config 2 geometry (2^20 instances = 1024 chains) against the oracle:
    the oracle computes the checksum of the whole 2^20 x 4096-bit job batch by batch (mk2o_checksum_job, pinned to the
    reference's own wrap-sums in tests/test_oracle.py); the GPU's in-kernel checksum must equal it in both layouts,
    and must equal the sum of the buffer it emitted (so the emitted bits, not just the accumulators, are covered).
    Mirrors tests/test_acceptance.py:103-135 (all instances compared, not a sample)."""
    torch = torch_cuda
    key = bytes.fromhex(golden["kats"][0]["key"])
    N, T = 1 << 20, 4096
    G = N // 32
    first = 3 << 20
    want = oracle.checksum_counter(key, first, N, T)
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        gen.set_group_offset(first // 32)
        gen.init_counter(key, first, N)
        col = torch.empty((T, G), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, col)
        torch.cuda.synchronize()
        assert gen.checksum() == want
        assert int(col.view(torch.int64).sum().item()) % (1 << 64) == want
        del col
        gen.init_counter(key, first, N)
        rows = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
        gen.generate_rowmajor(T, rows)
        torch.cuda.synchronize()
        assert gen.checksum() == want
        assert _rowmajor_buffer_checksum(torch, rows, first // 32) == want
        gen.set_stream(None)
    del rows
    torch.cuda.empty_cache()


def test_full_coverage_checksum_c3_clock_count(pkg, golden, oracle, torch_cuda):
    """BASELINE config 3's clock count (65 536 bits per instance, 16 scheduling chunks with state parking in
    between) for every one of 2^18 instances, row-major through tensor memory and column-major, against the
    oracle's whole-job checksum."""
    torch = torch_cuda
    key = bytes.fromhex(golden["kats"][0]["key"])
    N, T = 1 << 18, 65536
    first = 1 << 33
    want = oracle.checksum_counter(key, first, N, T)
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        gen.set_group_offset(first // 32)
        buf = torch.empty(N * T // 8, dtype=torch.uint8, device="cuda")
        gen.init_counter(key, first, N)
        gen.generate_rowmajor(T, buf.view(N, T // 8))
        torch.cuda.synchronize()
        assert gen.checksum() == want
        assert _rowmajor_buffer_checksum(torch, buf.view(N, T // 8), first // 32) == want
        gen.init_counter(key, first, N)
        col = buf.view(torch.int32).view(T, N // 32)
        gen.generate_colmajor(T, col)
        torch.cuda.synchronize()
        assert gen.checksum() == want
        assert int(col.view(torch.int64).sum().item()) % (1 << 64) == want
        gen.set_stream(None)
    del buf, col
    torch.cuda.empty_cache()


def test_full_coverage_checksum_c5_explicit_material(pkg, oracle, torch_cuda):
    """BASELINE config 5's shape (fresh random key/IV pairs x 1 Kbit) for every one of 2^20 pairs: explicit host
    material through mk2_init_from_material + generate and through the one-shot mk2_bulk_rowmajor (several
    pipeline blocks), both against the oracle's whole-job checksum."""
    N, T = 1 << 20, 1024
    rng = np.random.default_rng(0x1909)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    want = oracle.checksum_material(keys, ivs, 80, T)
    with pkg.MickeyGenerator(0) as gen:
        col = gen.init_material(keys, ivs, 80).generate_colmajor(T)
        assert gen.checksum() == want
        assert int(col.view("<u8").sum(dtype=np.uint64)) == want
        rows, csum = gen.bulk_rowmajor(keys, ivs, 80, T)
        assert csum == want
        # the same batch resident on the device: the one-kernel path (csrc/mk2_fused.cuh), every pair
        dk, di = torch_cuda.from_numpy(keys).cuda(), torch_cuda.from_numpy(ivs).cuda()
        drows = torch_cuda.empty((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        _, dsum = gen.bulk_rowmajor(dk, di, 80, T, drows)
        assert gen.last_kernel_launches == 1 and dsum == want
        assert np.array_equal(drows.cpu().numpy(), rows)
        bits = np.unpackbits(rows[4096:4160], axis=1)              # rows -> column words of one 64-lane batch
        words = (bits.T.astype(np.uint64) << np.arange(64, dtype=np.uint64)).sum(axis=1, dtype=np.uint64)
        assert np.array_equal(words, col[:, 128:130].copy().view("<u8").reshape(-1))


def test_full_length_chains_every_group(pkg, golden, oracle, torch_cuda):
    """The full 10^6-clock length of BASELINE config 2 (15 scheduling chunks, state parked and reloaded between
    them) for EVERY group of 32 chains (2^15 instances), against the oracle's whole-job checksum."""
    torch = torch_cuda
    key = bytes.fromhex(golden["kats"][0]["key"])
    N, T = 1 << 15, 1_000_000
    want = oracle.checksum_counter(key, 0, N, T)
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        gen.set_chunk_clocks(66688)                                # the chunk length the planner picks at 2^20 instances
        gen.init_counter(key, 0, N)
        col = torch.empty((T, N // 32), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, col)
        torch.cuda.synchronize()
        assert gen.checksum() == want
        assert int(col.view(torch.int64).sum().item()) % (1 << 64) == want
        gen.set_stream(None)
    del col
    torch.cuda.empty_cache()


def _free_gib(torch):
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0] / 2**30


def test_c2_full_size_million_bits(pkg, golden, oracle, torch_cuda):
    """BASELINE config 2 at its FULL size -- 2^20 instances x 10^6 bits, 131 GB of column-major keystream resident
    in HBM: the in-kernel checksum equals the sum of the emitted buffer, two half-length calls resume to the same
    checksum (chunked = unchunked), and sampled 64-instance groups are bit-exact against the oracle over the
    whole 1 Mbit."""
    torch = torch_cuda
    N, T = 1 << 20, 1_000_000
    G = N // 32
    if _free_gib(torch) < T * G * 4 / 2**30 + 6:
        pytest.skip("needs 131 GB of free HBM")
    key = bytes.fromhex(golden["kats"][0]["key"])
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        gen.init_counter(key, 0, N)
        col = torch.empty((T, G), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, col)
        torch.cuda.synchronize()
        csum = gen.checksum()
        total = 0
        for part in col.view(torch.int64).split(1 << 14):        # exact mod 2^64: int64 sums wrap
            total = (total + int(part.sum().item())) % (1 << 64)
        assert total == csum
        rng = np.random.default_rng(2)
        _sample_groups_vs_oracle(oracle, key, 0, col, [0, G - 2] + rng.integers(0, G, 2).tolist(), T)
        keep = col[:, 4242].clone()
        col.zero_()
        gen.init_counter(key, 0, N)
        gen.generate_colmajor(T // 2, col[: T // 2])
        gen.generate_colmajor(T - T // 2, col[T // 2:])
        torch.cuda.synchronize()
        assert gen.checksum() == csum and torch.equal(col[:, 4242], keep)
        gen.set_stream(None)
    del col
    torch.cuda.empty_cache()


def test_c3_full_size_rowmajor(pkg, golden, oracle, torch_cuda):
    """BASELINE config 3 at its FULL size -- 2^24 instances x 64 Kbit, 137 GB of row-major keystream: checksum equal
    to the column-major run of the same instances (layout independence), sampled rows bit-exact vs the oracle."""
    torch = torch_cuda
    N, T = 1 << 24, 65536
    if _free_gib(torch) < N * T / 8 / 2**30 + 20:
        pytest.skip("needs 137 GB of free HBM")
    key = bytes.fromhex(golden["kats"][0]["key"])
    first = 1 << 33
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        buf = torch.empty(N * T // 8, dtype=torch.uint8, device="cuda")
        rows = buf.view(N, T // 8)
        gen.init_counter(key, first, N)
        gen.generate_rowmajor(T, rows)
        torch.cuda.synchronize()
        c_row = gen.checksum()
        rng = np.random.default_rng(3)
        for n in [0, 1023, 1024, N - 1] + rng.integers(0, N, 8).tolist():
            keys, ivs = oracle.counter_material(key, first + int(n), 1)
            assert rows[n].cpu().numpy().tobytes() == oracle.bulk_rowmajor(keys, ivs, 80, T)[0].tobytes(), n
        gen.init_counter(key, first, N)
        gen.generate_colmajor(T, buf.view(torch.int32).view(T, N // 32))   # same bytes, reused as [T][G]
        torch.cuda.synchronize()
        assert gen.checksum() == c_row
        gen.set_stream(None)
    del rows, buf
    torch.cuda.empty_cache()


def test_c5_full_size_fresh_material(pkg, oracle, torch_cuda):
    """BASELINE config 5 at its FULL size -- 2^26 fresh (key, IV) pairs x 1 Kbit, explicit material arrays on the
    device, 8.6 GB of row-major keystream: init + generate, the one-shot bulk call as ONE fused kernel
    (csrc/mk2_fused.cuh) and the same call as pack / init / keystream kernels over the whole batch agree on every
    byte and on the checksum; sampled rows bit-exact vs the oracle."""
    torch = torch_cuda
    N, T = 1 << 26, 1024
    if _free_gib(torch) < 2 * N * T / 8 / 2**30 + 12:
        pytest.skip("needs 30 GB of free HBM")
    g = torch.Generator(device="cuda").manual_seed(0x190904750)
    keys = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
    ivs = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        rows = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
        gen.init_material(keys, ivs, 80)
        gen.generate_rowmajor(T, rows)
        torch.cuda.synchronize()
        csum = gen.checksum()
        rng = np.random.default_rng(5)
        idx = torch.from_numpy(np.unique(np.concatenate([[0, 31, 32, N - 1], rng.integers(0, N, 300)]))).cuda()
        want = oracle.bulk_rowmajor(keys[idx].cpu().numpy(), ivs[idx].cpu().numpy(), 80, T)
        assert np.array_equal(rows[idx].cpu().numpy(), want)
        rows2 = torch.empty_like(rows)
        _, csum2 = gen.bulk_rowmajor(keys, ivs, 80, T, rows2)
        torch.cuda.synchronize()
        assert gen.last_kernel_launches == 1 and csum2 == csum and torch.equal(rows, rows2)
        rows2.zero_()
        gen.set_bulk_fused(False)
        _, csum3 = gen.bulk_rowmajor(keys, ivs, 80, T, rows2)
        torch.cuda.synchronize()
        assert gen.last_kernel_launches > 1 and csum3 == csum and torch.equal(rows, rows2)
        gen.set_stream(None)
    del rows, rows2, keys, ivs
    torch.cuda.empty_cache()


def test_rowmajor_host_output_tiles(pkg, oracle):
    """Host row-major output crosses several [chain block] x [time chunk] staging tiles."""
    N, T = 32 * 32 * 2400 + 40, 4096 + 256          # > 2 x 8 x 148 chains -> two chain blocks
    key = bytes.fromhex("0123456789abcdef0123")
    with pkg.MickeyGenerator(0) as gen:
        gen.init_counter(key, 0, N)
        rows = np.zeros((N, T // 8 + 5), np.uint8)   # pitch wider than the row
        gen.generate_rowmajor(T, rows, pitch_bytes=rows.shape[1])
        csum = gen.checksum()
        gen.init_counter(key, 0, N)
        gen.generate_colmajor(T)
        assert gen.checksum() == csum
    assert not rows[:, T // 8:].any()
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([[0, 1023, 1024, 1184 * 1024 - 1, 1184 * 1024, 2368 * 1024 - 1, 2368 * 1024, N - 1],
                                    rng.integers(0, N, 60)]))
    for n in idx:
        keys, ivs = oracle.counter_material(key, int(n), 1)
        assert rows[n, : T // 8].tobytes() == oracle.bulk_rowmajor(keys, ivs, 80, T)[0].tobytes(), n


@pytest.mark.parametrize("stage_mib", [1, 3])
def test_host_outputs_with_small_staging_tiles(pkg, oracle, stage_mib):
    """mk2_set_stage_bytes: host outputs cut into many staging tiles (column-major: time chunks; row-major:
    [chain block] x [time chunk] 2-D copies) are the same bits as the oracle's."""
    N, T = 32 * 32 * 9 + 7, 8192 + 264
    rng = np.random.default_rng(stage_mib)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stage_bytes(stage_mib << 20)
        gen.init_material(keys, ivs, 80)
        cols = gen.generate_colmajor(T)
        c1 = gen.checksum()
        gen.init_material(keys, ivs, 80)
        rows = np.zeros((N, T // 8 + 3), np.uint8)
        gen.generate_rowmajor(T, rows, pitch_bytes=rows.shape[1])
        assert gen.checksum() == c1
    cols = np.asarray(cols)
    want_cols = oracle.bulk_colmajor(keys, ivs, 80, T)
    assert cols.shape == want_cols.shape and np.array_equal(cols, want_cols)
    assert np.array_equal(rows[:, : T // 8], oracle.bulk_rowmajor(keys, ivs, 80, T)) and not rows[:, T // 8:].any()


def test_c5_init_dominated_explicit_material(pkg, oracle, torch_cuda):
    """BASELINE config 5 shape (fresh key/IV pairs x 1 Kbit) at 2^20 pairs: explicit random
    material from host arrays, row-major output to the host, sampled rows vs the oracle."""
    N, T = 1 << 20, 1024
    keys, ivs = random_arrays(0x1909_0475, N)
    rows = pkg.bulk_rowmajor(keys, ivs, 80, T)
    rng = np.random.default_rng(1)
    idx = np.unique(np.concatenate([[0, 1, 31, 32, N - 1], rng.integers(0, N, 200)]))
    want = oracle.bulk_rowmajor(keys[idx], ivs[idx], 80, T)
    assert np.array_equal(rows[idx], want)


# ---------------------------------------------------------------- persistent scheduler

@pytest.mark.parametrize("block,chunk", [(0, 0), (32, 128), (64, 384), (128, 1000), (256, 128), (256, 1 << 30)])
def test_schedule_knobs_do_not_change_bits(pkg, oracle, block, chunk):
    """Any worker-warp count / chunk length must give the same keystream (column- and row-major),
    including a partial last chain (G % 32 != 0), a partial last group (N % 32 != 0) and chunk tails."""
    N, T = 32 * 75 + 9, 1160
    keys, ivs = random_arrays(31337, N)
    want_c = oracle.bulk_colmajor(keys, ivs, 80, T)
    want_r = oracle.bulk_rowmajor(keys, ivs, 80, T)
    with pkg.MickeyGenerator(0) as gen:
        gen.set_block_threads(block)
        gen.set_chunk_clocks(chunk)
        got_c = gen.init_material(keys, ivs, 80).generate_colmajor(T)
        plan = gen.last_plan()
        assert plan[0] in (32, 64, 128, 256) and plan[1] >= 1
        c1 = gen.checksum()
        got_r = gen.init_material(keys, ivs, 80).generate_rowmajor(T)
        assert gen.checksum() == c1
    assert np.array_equal(got_c, want_c)
    assert np.array_equal(got_r, want_r)


def test_many_chains_many_chunks_and_trace(pkg, oracle, torch_cuda):
    """More chains than worker warps, tiny chunks: every chain migrates between SMs many times."""
    torch = torch_cuda
    N, T = 32 * 32 * 700, 640          # 700 chains
    key = bytes.fromhex("00112233445566778899")
    with pkg.MickeyGenerator(0) as gen:
        gen.set_chunk_clocks(128)
        gen.set_trace(1 << 14)
        gen.init_counter(key, 64, N)
        col = torch.empty((T, N // 32), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, col.data_ptr())
        tr = gen.read_trace()
        assert len(tr) == 700 * 5                       # one record per (chain, chunk)
        assert set(zip(tr["chain"].tolist(), tr["k"].tolist())) == {(c, k) for c in range(700) for k in range(5)}
        order = np.lexsort((tr["k"], tr["chain"]))
        t = tr[order]
        same = t["chain"][1:] == t["chain"][:-1]
        assert np.all(t["t_start"][1:][same] >= t["t_end"][:-1][same])   # chunks of a chain never overlap
        assert len(np.unique(tr["smid"])) > 100         # work really spread over the SMs
        gen.set_trace(0)
        gen.set_chunk_clocks(0)
        gen.init_counter(key, 64, N)
        col2 = torch.empty_like(col)
        gen.generate_colmajor(T, col2.data_ptr())
        assert torch.equal(col, col2)
    for g in (0, 1023, 22398):
        g &= ~1
        keys, ivs = oracle.counter_material(key, 64 + 32 * g, 64)
        assert np.array_equal(col[:, g:g + 2].cpu().numpy().view(np.uint32), oracle.bulk_colmajor(keys, ivs, 80, T))


def test_knob_validation(pkg):
    gen = pkg.MickeyGenerator(0)
    with pytest.raises(ValueError):
        gen.set_block_threads(48)
    with pytest.raises(ValueError):
        gen.set_chunk_clocks(64)
    with pytest.raises((ValueError, pkg.Mk2Error)):
        gen.set_stage_bytes(4096)
    gen.set_stage_bytes(0)
    gen.close()


# ---------------------------------------------------------------- seed derivation

def test_seed_derivation_matches_reference_and_oracle(pkg, golden, oracle, torch_cuda):
    from paper_1909_04750_b200 import seedgen

    for rec in golden["seedgen"]:
        seed = bytes.fromhex(rec["seed"])
        master = seedgen.MasterSeed(seed, "mickey", 64)
        mats = seedgen.derive_all(master)
        blob = b"".join(m.key + bytes(m.iv) for m in mats)
        assert sha(blob) == rec["all64_sha256"]
        for lane, m in rec["lanes"].items():
            got = seedgen.derive_lane_material(master, int(lane))
            assert got.key.hex() == m["key"] and bytes(got.iv).hex() == m["iv"]
    # past the reference's 64-lane cap: the oracle defines the continuation
    seed = bytes.fromhex(golden["seedgen"][1]["seed"])
    first, n = (1 << 32) - 100_000, 100_000
    with pkg.MickeyGenerator(0) as gen:
        keys, ivs = gen.derive_material(seed, first, n)
        wk, wi = oracle.derive_material(seed, first, n)
        assert np.array_equal(keys, wk) and np.array_equal(ivs, wi)
        # device buffers
        dk = torch_cuda.empty((n, 10), dtype=torch_cuda.uint8, device="cuda")
        di = torch_cuda.empty((n, 10), dtype=torch_cuda.uint8, device="cuda")
        gen.derive_material(seed, first, n, dk, di)
        torch_cuda.cuda.synchronize()
        assert np.array_equal(dk.cpu().numpy(), wk) and np.array_equal(di.cpu().numpy(), wi)
        with pytest.raises(ValueError):
            gen.derive_material(seed, (1 << 32) - 5, 10)
        with pytest.raises(ValueError):
            gen.derive_material(bytes(32), 0, 10)
        # init_seed == derive + init_material, and the bench-seed golden keystream
        a = gen.init_seed(seed, 1000, 5000).generate_colmajor(200)
        k5, i5 = oracle.derive_material(seed, 1000, 5000)
        b = gen.init_material(k5, i5, 80).generate_colmajor(200)
        assert np.array_equal(a, b)
        assert np.array_equal(a, oracle.bulk_colmajor(k5, i5, 80, 200))
        bs = golden["bench_seed"]
        row = gen.init_seed(bytes.fromhex(golden["seedgen"][0]["seed"]), 0, 64).generate_rowmajor(bs["nclocks"])
        assert sha(row.tobytes()) == bs["lane_major_sha256"]


# ---------------------------------------------------------------- CLI

def test_cli_gen_matches_reference_cli(pkg, golden, tmp_path):
    from paper_1909_04750_b200 import cli

    for case in golden["cli_gen"]:
        out = tmp_path / "o.hex"
        assert cli.main(["gen", "--out", str(out), *case["argv"]]) == 0
        assert out.read_text() == case["hex"], case["argv"]
    # raw format == hex format, more lanes than the reference engine is wide
    raw, hx = tmp_path / "o.bin", tmp_path / "o2.hex"
    argv = ["--bits", str(200 * 64), "--lanes", "200", "--seed", "ab" * 32]
    cli.main(["gen", "--format", "raw", "--out", str(raw), *argv])
    cli.main(["gen", "--out", str(hx), *argv])
    assert raw.read_bytes().hex() == hx.read_text()
    first4 = [c for c in golden["cli_gen"] if c["argv"][:4] == ["--bits", "8192", "--lanes", "4"]][0]["hex"]
    assert raw.read_bytes()[:8].hex() == first4[:16]      # lane 0 of the same seed starts the same way
    with pytest.raises(SystemExit):
        cli.main(["gen", "--bits", "12"])
    with pytest.raises(SystemExit):
        cli.main(["gen", "--bits", "24", "--lanes", "2"])


def test_cli_vectors_and_bench(pkg, tmp_path, capsys):
    from paper_1909_04750_b200 import cli, vectors

    assert vectors.verify_vectors("mickey") == (3, [])
    assert cli.main(["vectors"]) == 0
    f = tmp_path / "v.txt"
    f.write_text("# comment\nkey=123456789abcdef01234 iv=21436587 ks=9821e10c5ed28d32bbc3d1fb15e93a15\n"
                 "key=123456789abcdef01234 iv= ks=00f1b8779b47da74075e7a8ccc23c80c\n")
    assert cli.main(["vectors", "--file", str(f)]) == cli.EXIT_VECTOR_MISMATCH
    js = tmp_path / "b.json"
    assert cli.main(["bench", "--mib", "64", "--repeats", "3", "--lanes-log2", "16", "--json-out", str(js)]) == 0
    import json as _json

    rec = _json.loads(js.read_text())["results"][0]
    assert {"algorithm", "impl", "width", "nbytes", "seconds", "gbit_per_s", "runs", "speedup_vs_naive"} <= set(rec)
    assert rec["impl"] == "cuda" and rec["gbit_per_s"] > 10 and len(rec["runs"]) == 3


def test_two_threads_two_contexts(pkg, oracle):
    """One context per worker thread, as the reference's ThreadPoolExecutor bench does (bench.py:265-282)."""
    from concurrent.futures import ThreadPoolExecutor

    def work(seed):
        keys, ivs = random_arrays(seed, 3000)
        with pkg.MickeyGenerator(0) as gen:
            col = gen.init_material(keys, ivs, 80).generate_colmajor(700)
            row = gen.init_material(keys, ivs, 80).generate_rowmajor(512)
        return seed, col, row

    with ThreadPoolExecutor(max_workers=4) as pool:
        results = list(pool.map(work, [11, 22, 33, 44]))
    for seed, col, row in results:
        keys, ivs = random_arrays(seed, 3000)
        assert np.array_equal(col, oracle.bulk_colmajor(keys, ivs, 80, 700))
        assert np.array_equal(row, oracle.bulk_rowmajor(keys, ivs, 80, 512))


# ---------------------------------------------------------------- Grain v1

def test_grain_vectors_and_golden_cases(pkg, golden):
    from paper_1909_04750_b200 import grain, vectors

    assert vectors.verify_vectors("grain") == (2, [])
    g = golden["grain"]
    for c in g["sliced_cases"]:
        mats = [grain.GrainKeyIv(bytes.fromhex(m["key"]), bytes.fromhex(m["iv"])) for m in c["materials"]]
        eng = grain.GrainSliced.from_key_ivs(mats, width=c["width"])
        assert [f"{x:x}" for x in eng.b] == c["init_state"]["b"], c["name"]
        assert [f"{x:x}" for x in eng.s] == c["init_state"]["s"], c["name"]
        words = grain.grain_sliced_words(mats, c["nclocks"], c["width"])
        assert words.astype("<u8").tobytes().hex() == c["words_hex"], c["name"]
        a = eng.keystream_words(100) + eng.keystream_words(c["nclocks"] - 100) if c["nclocks"] > 100 else eng.keystream_words(c["nclocks"])
        assert a == [int(w) for w in words]                       # resumable, odd split across windows
    for c in g["scalar_cases"]:
        m = grain.GrainKeyIv(bytes.fromhex(c["key"]), bytes.fromhex(c["iv"]))
        eng = grain.GrainSliced.from_key_ivs([m], width=32)
        lane = eng.extract_lane(0)
        assert f"{sum(b << i for i, b in enumerate(lane.r)):x}" == c["post_init_b"]
        assert f"{sum(b << i for i, b in enumerate(lane.s)):x}" == c["post_init_s"]
        bits = np.array(eng.keystream_lane_bits(1024)[0], np.uint8)
        assert np.packbits(bits).tobytes().hex() == c["ks128_msb"]
    mats = [grain.GrainKeyIv(bytes.fromhex(m["key"]), bytes.fromhex(m["iv"])) for m in g["sliced_cases"][1]["materials"]]
    keys, ivs = grain.pack_materials(mats, 64)
    T = g["long"]["nclocks"]
    with grain.GrainGenerator(0) as gen:
        assert sha(gen.init_material(keys, ivs).generate_colmajor(T).tobytes()) == g["long"]["words_u8_sha256"]
        c1 = gen.checksum()
        assert sha(gen.init_material(keys, ivs).generate_rowmajor(T).tobytes()) == g["long"]["lane_major_msb_sha256"]
        assert gen.checksum() == c1
        assert sha(gen.init_material(keys, ivs).generate_rowmajor(T, bit_order="lsb").tobytes()) == g["long"]["lane_major_lsb_sha256"]
        with pytest.raises(pkg.Mk2Error, match="Grain state"):
            pkg.MickeyGenerator.generate_colmajor(gen, 8)


@pytest.mark.parametrize("block,chunk", [(0, 0), (64, 128), (256, 1 << 30), (128, 400)])
def test_grain_bulk_vs_oracle(pkg, oracle, block, chunk, torch_cuda):
    from paper_1909_04750_b200 import grain

    rng = np.random.default_rng(77)
    N, T = 32 * 70 + 11, 1000
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 8), dtype=np.uint8)
    with grain.GrainGenerator(0) as gen:
        gen.set_block_threads(block)
        gen.set_chunk_clocks(chunk)
        col = gen.init_material(keys, ivs).generate_colmajor(T)
        row = gen.init_material(keys, ivs).generate_rowmajor(T)
        # device buffers, resumed in two calls
        dk, di = torch_cuda.from_numpy(keys).cuda(), torch_cuda.from_numpy(ivs).cuda()
        gen.init_material(dk, di)
        dev = torch_cuda.zeros((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        gen.generate_rowmajor(512, dev, byte_offset=0, bit_order="lsb")
        gen.generate_rowmajor(T - 512, dev, byte_offset=64, bit_order="lsb")
        torch_cuda.cuda.synchronize()
    assert np.array_equal(col, oracle.grain_bulk_colmajor(keys, ivs, T))
    assert np.array_equal(row, oracle.grain_bulk_rowmajor(keys, ivs, T))
    assert np.array_equal(dev.cpu().numpy(), oracle.grain_bulk_rowmajor(keys, ivs, T, "lsb"))


@pytest.mark.parametrize("staging", [2, 3])
@pytest.mark.parametrize("N,T,chunk", [(32 * 70 + 11, 1000, 0), (1 << 15, 4096 + 520, 1024), (64, 8, 0), (4099, 136, 0)])
def test_grain_rowmajor_512_clock_tiles(pkg, oracle, N, T, chunk, staging, torch_cuda):
    """The opt-in Grain row-major kernels with 512-clock tiles (csrc/mk2_grain_row64.cuh): split between tensor
    and shared memory (mk2_set_row_staging(ctx, 2)) or in L2-resident global scratch (3): whole tiles, short
    tails, partial last groups, both byte orders, unaligned rows -- same bytes as the oracle and as the default
    kernel."""
    from paper_1909_04750_b200 import grain

    rng = np.random.default_rng(N + T)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 8), dtype=np.uint8)
    want = oracle.grain_bulk_rowmajor(keys, ivs, T)
    with grain.GrainGenerator(0) as gen:
        gen.set_row_staging(staging)
        gen.set_chunk_clocks(chunk)
        row = gen.init_material(keys, ivs).generate_rowmajor(T)
        csum = gen.checksum()
        lsb = gen.init_material(keys, ivs).generate_rowmajor(T, bit_order="lsb")
        dev = torch_cuda.zeros((N, T // 8 + 3), dtype=torch_cuda.uint8, device="cuda")   # pitch not a multiple of 16
        gen.init_material(keys, ivs).generate_rowmajor(T, dev)
        torch_cuda.cuda.synchronize()
        assert gen.last_plan()[0] == 256
        gen.set_row_staging(0)
        ref = gen.init_material(keys, ivs).generate_rowmajor(T)
        assert gen.checksum() == csum
    assert np.array_equal(row, want) and np.array_equal(ref, want)
    assert np.array_equal(lsb, oracle.grain_bulk_rowmajor(keys, ivs, T, "lsb"))
    assert np.array_equal(dev.cpu().numpy()[:, : T // 8], want)


@pytest.mark.parametrize("N,T,chunk", [(32 * 70, 256, 0), (1 << 15, 4096 + 512, 1024), (32 * 1500, 2048, 256), (64, 768, 0),
                                       (4099, 512, 0), (2048, 1000, 0)])
def test_grain_rowmajor_ring_kernel(pkg, oracle, N, T, chunk, torch_cuda):
    """Grain row-major for lone warps (csrc/mk2_grain_ring.cuh, mk2_set_row_staging(ctx, 4)): four warps per SM,
    in-register bit transposes, the drain of tile i riding on the first eight windows of tile i + 1 through a
    three-block ring.  One tile, many tiles, chunks of one tile (every tile is a chunk's last), both byte orders,
    resumed calls; shapes it does not take (partial groups, T not a multiple of 256, unaligned rows) fall back to
    the default kernel.  Same bytes as the oracle, same checksum as the default kernel."""
    from paper_1909_04750_b200 import grain

    rng = np.random.default_rng(N + T)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 8), dtype=np.uint8)
    want = oracle.grain_bulk_rowmajor(keys, ivs, T)
    takes = N % 32 == 0 and T % 256 == 0
    with grain.GrainGenerator(0) as gen:
        gen.set_row_staging(4)
        gen.set_chunk_clocks(chunk)
        dev = torch_cuda.zeros((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        gen.init_material(keys, ivs).generate_rowmajor(T, dev)
        torch_cuda.cuda.synchronize()
        csum = gen.checksum()
        lsb = torch_cuda.zeros((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        gen.init_material(keys, ivs).generate_rowmajor(T, lsb, bit_order="lsb")
        two = torch_cuda.zeros((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        if T >= 512 and takes:   # resumed: 256 clocks, then the rest
            gen.init_material(keys, ivs)
            gen.generate_rowmajor(256, two, byte_offset=0)
            gen.generate_rowmajor(T - 256, two, byte_offset=32)
        odd = torch_cuda.zeros((N, T // 8 + 3), dtype=torch_cuda.uint8, device="cuda")   # pitch not a multiple of 32
        gen.init_material(keys, ivs).generate_rowmajor(T, odd)
        torch_cuda.cuda.synchronize()
        gen.set_row_staging(0)
        gen.init_material(keys, ivs).generate_rowmajor(T)
        assert gen.checksum() == csum
    assert np.array_equal(dev.cpu().numpy(), want)
    assert np.array_equal(lsb.cpu().numpy(), oracle.grain_bulk_rowmajor(keys, ivs, T, "lsb"))
    if T >= 512 and takes:
        assert np.array_equal(two.cpu().numpy(), want)
    assert np.array_equal(odd.cpu().numpy()[:, : T // 8], want)


@pytest.mark.parametrize("N,T,chunk", [(1024, 256, 0), (1 << 15, 4096 + 512, 1024), (1024 * 37, 2048, 256), (2048, 768, 0),
                                       (4099, 512, 0), (2048, 1000, 0)])
def test_grain_rowmajor_eight_warp_kernel(pkg, oracle, N, T, chunk, torch_cuda):
    """Grain row-major with eight warps per SM (csrc/mk2_grain_row8.cuh, mk2_set_row_staging(ctx, 5)): 28 groups of
    every 256-clock tile in shared memory, four in tensor memory.  One tile, many tiles, one-tile chunks, both byte
    orders, resumed calls; shapes it does not take (partial chains, T not a multiple of 256, unaligned rows) fall
    back to the default kernel.  Same bytes as the oracle, same checksum as the default kernel."""
    from paper_1909_04750_b200 import grain

    rng = np.random.default_rng(N + T + 1)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 8), dtype=np.uint8)
    want = oracle.grain_bulk_rowmajor(keys, ivs, T)
    takes = N % 1024 == 0 and T % 256 == 0
    with grain.GrainGenerator(0) as gen:
        gen.set_row_staging(5)
        gen.set_chunk_clocks(chunk)
        dev = torch_cuda.zeros((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        gen.init_material(keys, ivs).generate_rowmajor(T, dev)
        torch_cuda.cuda.synchronize()
        if takes:
            assert gen.last_plan()[0] == 256
        csum = gen.checksum()
        lsb = torch_cuda.zeros((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        gen.init_material(keys, ivs).generate_rowmajor(T, lsb, bit_order="lsb")
        two = torch_cuda.zeros((N, T // 8), dtype=torch_cuda.uint8, device="cuda")
        if T >= 512 and takes:   # resumed: 256 clocks, then the rest
            gen.init_material(keys, ivs)
            gen.generate_rowmajor(256, two, byte_offset=0)
            gen.generate_rowmajor(T - 256, two, byte_offset=32)
        odd = torch_cuda.zeros((N, T // 8 + 3), dtype=torch_cuda.uint8, device="cuda")   # pitch not a multiple of 32
        gen.init_material(keys, ivs).generate_rowmajor(T, odd)
        torch_cuda.cuda.synchronize()
        gen.set_row_staging(0)
        gen.init_material(keys, ivs).generate_rowmajor(T)
        assert gen.checksum() == csum
    assert np.array_equal(dev.cpu().numpy(), want)
    assert np.array_equal(lsb.cpu().numpy(), oracle.grain_bulk_rowmajor(keys, ivs, T, "lsb"))
    if T >= 512 and takes:
        assert np.array_equal(two.cpu().numpy(), want)
    assert np.array_equal(odd.cpu().numpy()[:, : T // 8], want)


def test_grain_large_sampled(pkg, oracle, torch_cuda):
    """2^20 Grain instances x 4096 bits: sampled groups vs the oracle, layout-independent checksum."""
    from paper_1909_04750_b200 import grain

    torch = torch_cuda
    N, T = 1 << 20, 4096
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 8), dtype=np.uint8)
    dk, di = torch.from_numpy(keys).cuda(), torch.from_numpy(ivs).cuda()
    with grain.GrainGenerator(0) as gen:
        gen.init_material(dk, di)
        col = torch.empty((T, N // 32), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, col)
        torch.cuda.synchronize()
        assert (int(col.view(torch.int64).sum().item()) % (1 << 64)) == gen.checksum()
        csum = gen.checksum()
        gen.init_material(dk, di)
        rows = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
        gen.generate_rowmajor(T, rows)
        torch.cuda.synchronize()
        assert gen.checksum() == csum
    for g in (0, 777, N // 32 - 2):
        g &= ~1
        sl = slice(32 * g, 32 * g + 64)
        assert np.array_equal(col[:, g:g + 2].cpu().numpy().view(np.uint32), oracle.grain_bulk_colmajor(keys[sl], ivs[sl], T))
        assert np.array_equal(rows[sl].cpu().numpy(), oracle.grain_bulk_rowmajor(keys[sl], ivs[sl], T))


def test_scalar_engine_interface(pkg, golden):
    """MickeyScalar / MickeyScalarPacked / naive-bytes entry points (mickey.py:101-227, kernels.py:203-229):
    the reference's test_mickey.py scalar tests, served by lane 0 of a GPU group."""
    for rec in golden["kats"]:                                           # tests/test_mickey.py:38-41
        st = pkg.MickeyScalar.from_key_iv(pkg.MickeyKeyIv(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"])))
        assert st.keystream_bytes(16).hex() == rec["ks"]
    for rec in golden["scalar_cases"][:4] + golden["scalar_cases"][-2:]:
        m = pkg.MickeyKeyIv(*golden_material(rec))
        a, b = pkg.MickeyScalar.from_key_iv(m), pkg.MickeyScalarPacked.from_key_iv(m)
        assert f"{sum(x << i for i, x in enumerate(a.r)):x}" == rec["post_init_r"] and f"{b.s:x}" == rec["post_init_s"]
        assert a.keystream_bytes(64).hex() == rec["ks256"][:128]
        assert pkg.kernels.mickey_naive_bitwise_bytes(m, 32).hex() == rec["ks256"][:64]
        assert pkg.kernels.mickey_packed_bytes(m, 32).hex() == rec["ks256"][:64]
        assert pkg.scalar_keystream(m, 16) == np.unpackbits(np.frombuffer(bytes.fromhex(rec["ks256"][:4]), np.uint8)).tolist()
    z = pkg.MickeyScalarPacked()                                          # tests/test_mickey.py:59-66
    z.clock_kg(False, 0)
    assert f"{z.r:x}" == golden["zero_state_one_clock"]["r"] and f"{z.s:x}" == golden["zero_state_one_clock"]["s"]
    k = golden["kats"][0]                                                 # tests/test_mickey.py:76-83
    st = pkg.MickeyScalarPacked.from_key_iv(pkg.MickeyKeyIv(bytes.fromhex(k["key"]), bytes.fromhex(k["iv"])))
    for r_hex, s_hex in golden["kat0_state_trace_100"][:12]:
        st.clock_kg(False, 0)
        assert f"{st.r:x}" == r_hex and f"{st.s:x}" == s_hex
    by_bytes = pkg.MickeyScalar.from_key_iv(pkg.MickeyKeyIv(bytes(range(10)), b"\xa5"))   # tests/test_mickey.py:102-108
    by_bits = pkg.MickeyScalar.from_key_iv(pkg.MickeyKeyIv(bytes(range(10)), [1, 0, 1, 0, 0, 1, 0, 1]))
    assert by_bytes.r == by_bits.r and by_bytes.s == by_bits.s
    with pytest.raises(ValueError):
        pkg.MickeyScalar([0] * 99, [0] * 100)


def test_c3_instance_count_rowmajor_sampled(pkg, golden, oracle, torch_cuda):
    """BASELINE config 3 geometry: 2^24 instances, row-major through the warp/register bit transpose,
    a 2048-clock slice; sampled rows bit-exact vs the oracle, checksum equal to the column-major run's,
    seed-derived and counter material."""
    torch = torch_cuda
    key = bytes.fromhex(golden["kats"][0]["key"])
    N, T = 1 << 24, 2048
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stream(torch.cuda.current_stream().cuda_stream)
        gen.init_counter(key, 1 << 30, N)
        rows = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
        gen.generate_rowmajor(T, rows)
        torch.cuda.synchronize()
        c_row = gen.checksum()
        assert gen.last_plan()[0] == 256                       # eight worker warps: staging tiles in tensor memory
        rng = np.random.default_rng(24)
        for n in [0, 31, 32, 1023, 1024, N - 1] + rng.integers(0, N, 10).tolist():
            keys, ivs = oracle.counter_material(key, (1 << 30) + int(n), 1)
            assert rows[n].cpu().numpy().tobytes() == oracle.bulk_rowmajor(keys, ivs, 80, T)[0].tobytes(), n
        del rows
        gen.init_counter(key, 1 << 30, N)
        col = torch.empty((T, N // 32), dtype=torch.int32, device="cuda")
        gen.generate_colmajor(T, col)
        torch.cuda.synchronize()
        assert gen.checksum() == c_row
        assert (int(col.view(torch.int64).sum().item()) % (1 << 64)) == c_row
        gen.set_stream(None)


def test_cli_gen_grain_matches_reference_cli(pkg, golden, tmp_path):
    from paper_1909_04750_b200 import cli

    for case in golden["cli_gen_grain"]:
        out = tmp_path / "g.hex"
        assert cli.main(["gen", "--algo", "grain", "--out", str(out), *case["argv"]]) == 0
        assert out.read_text() == case["hex"], case["argv"]
    assert cli.main(["vectors", "--algo", "grain"]) == 0


@pytest.mark.parametrize("N,T,block,chunk", [(1000, 1408, 0, 0), (32, 8, 0, 0), (4099, 136, 64, 256), (64, 1024 + 120, 256, 512),
                                             (32 * 32 * 20 + 5, 2048 + 264, 256, 768), (32 * 32 * 9, 512, 96, 256)])
def test_rowmajor_tensor_memory_staging(pkg, oracle, N, T, block, chunk):
    """mk2_set_row_staging(2): the 256-word staging tile lives in tensor memory (tcgen05.st / tcgen05.ld) instead
    of shared memory; same bits for aligned and ragged shapes, partial last chains, every worker-warp count."""
    rng = np.random.default_rng(N * 7 + T)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    want = oracle.bulk_rowmajor(keys, ivs, 80, T)
    with pkg.MickeyGenerator(0) as gen:
        gen.set_row_staging(2)
        gen.set_block_threads(block)
        gen.set_chunk_clocks(chunk)
        gen.init_material(keys, ivs, 80)
        got = gen.generate_rowmajor(T)
        c_tmem = gen.checksum()
        half = (T // 16) * 8
        gen.init_material(keys, ivs, 80)
        a = np.zeros((N, T // 8 + 1), np.uint8)                       # odd pitch: the unaligned drain
        gen.generate_rowmajor(half, a, pitch_bytes=a.shape[1])
        gen.generate_rowmajor(T - half, a, pitch_bytes=a.shape[1], byte_offset=half // 8)
        gen.set_row_staging(1)
        gen.init_material(keys, ivs, 80)
        gen.generate_rowmajor(T)
        assert gen.checksum() == c_tmem
    assert np.array_equal(got, want)
    assert np.array_equal(a[:, : T // 8], want)


@pytest.mark.parametrize("N,T,iv_bits", [(1, 8, 0), (32, 1000, 32), (64, 4096 + 37, 80), (1000, 333, 13), (5000, 2048, 80),
                                         (65536, 96, 80)])
def test_small_batch_warp_per_group_kernels(pkg, oracle, N, T, iv_bits):
    """Small batches (up to 2048 groups; the reference's own unit is 64 lanes, kernels.py:189-200) are initialised
    and clocked by warp-per-group kernels (csrc/mk2_coop.cuh: state spread over the lanes, taps and neighbours by
    shuffle).  Same words, state and checksum as the thread-per-group kernels (mk2_set_small_batch(0)) and as the
    oracle; a context initialised by one kind and clocked, resumed or exported by the other agrees too."""
    rng = np.random.default_rng(N * 7 + T)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    want = oracle.bulk_colmajor(keys, ivs, iv_bits, T + 40)
    with pkg.MickeyGenerator(0) as a, pkg.MickeyGenerator(0) as b:
        a.set_small_batch(True)
        b.set_small_batch(False)
        wa = a.init_material(keys, ivs, iv_bits).generate_colmajor(T)
        wb = b.init_material(keys, ivs, iv_bits).generate_colmajor(T)
        assert a.last_plan()[0] == 128 and np.array_equal(wa, wb) and np.array_equal(wa, want[:T])
        assert a.checksum() == b.checksum() and np.array_equal(a.export_state(), b.export_state())
        # cross over: the state the warp-per-group kernels left is continued by the throughput kernels and back
        a.set_small_batch(False)
        b.set_small_batch(True)
        ma, mb = a.generate_colmajor(40), b.generate_colmajor(40)
        assert np.array_equal(ma, want[T:]) and np.array_equal(mb, want[T:]) and a.checksum() == b.checksum()
        # row-major: the warp-per-group row kernel (32 x 32 bit transpose across the lanes), both byte orders, rows
        # that are not 4-byte aligned, a resumed second piece; the throughput row kernel on the same state; and the
        # one-shot bulk call, which takes the same small-batch route
        if T % 8 == 0:
            rows = oracle.bulk_rowmajor(keys, ivs, iv_bits, T + 40)
            assert np.array_equal(b.init_material(keys, ivs, iv_bits).generate_rowmajor(T), rows[:, : T // 8])
            assert b.last_plan()[0] == 128
            assert np.array_equal(b.generate_rowmajor(40), rows[:, T // 8:])
            assert np.array_equal(a.init_material(keys, ivs, iv_bits).generate_rowmajor(T), rows[:, : T // 8])
            odd = np.zeros((N, T // 8 + 3), np.uint8)
            b.init_material(keys, ivs, iv_bits).generate_rowmajor(T, odd, pitch_bytes=odd.shape[1])
            assert np.array_equal(odd[:, : T // 8], rows[:, : T // 8]) and not odd[:, T // 8:].any()
            lsb = b.init_material(keys, ivs, iv_bits).generate_rowmajor(T, bit_order="lsb")
            assert np.array_equal(lsb, np.packbits(np.unpackbits(rows[:, : T // 8], axis=1), axis=1, bitorder="little"))
            got, csum = b.bulk_rowmajor(keys, ivs, iv_bits, T)
            assert np.array_equal(got, rows[:, : T // 8]) and csum == oracle.checksum_material(keys, ivs, iv_bits, T)


def test_c_abi_from_plain_c(c_abi_consumer):
    """The drop-in boundary used from plain C (tests/c/abi_consumer.c: include/mk2.h + libmk2.so, malloc'ed host
    buffers): the eSTREAM vector on 70 instances through init + generate and through the one-shot bulk call."""
    import subprocess

    res = subprocess.run([str(c_abi_consumer)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, (res.returncode, res.stdout, res.stderr)
    assert res.stdout.startswith("ok: 70 instances x 128 bits")


@pytest.mark.parametrize("N,T,iv_bits,pad", [(1024, 1024, 80, 0), (32 * 70 + 11, 1000, 80, 0), (5, 8, 0, 0), (4099, 264, 32, 3),
                                             (1 << 15, 4096 + 520, 80, 0), (2 * 8 * 148 * 1024 + 4096 + 7, 128, 16, 0),
                                             (1 << 16, 256, 0, 16)])
def test_bulk_rowmajor_fused_kernel(pkg, oracle, N, T, iv_bits, pad, torch_cuda):
    """mk2_bulk_rowmajor with key/IV arrays and output on the device = ONE kernel (csrc/mk2_fused.cuh: records ->
    input words in tensor memory -> load clocks -> pre-clocks -> keystream -> rows): the same bytes and checksum
    as the pack / init / keystream kernels (mk2_set_bulk_fused(0)) and as the oracle; partial last group and
    chain, IV lengths 0 / 16 / 32 / 80 bits, short tails, unaligned rows, more than one pipeline block, and the
    state it leaves for a resuming call (mickey_sliced_words + words_lane_major_bytes, kernels.py:189-200, :615-621)."""
    torch = torch_cuda
    rng = np.random.default_rng(N + T)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    dk, di = torch.from_numpy(keys).cuda(), torch.from_numpy(ivs).cuda()
    sample = np.unique(np.concatenate([np.arange(min(N, 96)), np.arange(max(0, N - 96), N), rng.integers(0, N, 64)]))
    want = oracle.bulk_rowmajor(keys[sample], ivs[sample], iv_bits, T)
    resumable = N <= 2 * 8 * torch.cuda.get_device_properties(0).multi_processor_count * 1024
    with pkg.MickeyGenerator(0) as gen:
        gen.set_small_batch(False)                                 # batches of <= 2048 groups would take the warp-per-group kernels
        gen.set_bulk_fused(2)                                      # also for T > 1024, where the default is pack + init + keystream
        a = torch.zeros((N, T // 8 + pad), dtype=torch.uint8, device="cuda")
        _, ca = gen.bulk_rowmajor(dk, di, iv_bits, T, a)
        assert gen.last_kernel_launches == 1                       # the fused path ran
        if resumable:
            more = gen.generate_rowmajor(64)
            resumed = gen.checksum()
        else:
            with pytest.raises(pkg.Mk2Error):
                gen.generate_rowmajor(8)
        gen.set_bulk_fused(False)
        b = torch.zeros((N, T // 8 + pad), dtype=torch.uint8, device="cuda")
        _, cb = gen.bulk_rowmajor(dk, di, iv_bits, T, b)
        assert gen.last_kernel_launches > 1
        if resumable:
            assert np.array_equal(more, gen.generate_rowmajor(64)) and resumed == gen.checksum()
    torch.cuda.synchronize()
    assert ca == cb and bool((a == b).all().item())
    assert np.array_equal(a.cpu().numpy()[sample][:, : T // 8], want)
    if pad:
        assert not bool(a[:, T // 8:].any().item())


def test_bulk_rowmajor_one_shot_pipelined_blocks(pkg, oracle, torch_cuda):
    """mk2_bulk_rowmajor: N spans three pipeline blocks (2 x 8 x SMs x 1024 instances each); host and device
    buffers, IV lengths 80 / 13 / 0; rows and the whole-call checksum equal init + generate and the oracle."""
    torch = torch_cuda
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    block = 2 * 8 * sms * 1024
    N, T = 2 * block + 32 * 1000 + 9, 256
    rng = np.random.default_rng(99)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    sample = np.unique(np.concatenate([[0, block - 1, block, 2 * block - 1, 2 * block, N - 1], rng.integers(0, N, 40)]))
    with pkg.MickeyGenerator(0) as gen:
        for iv_bits in (80, 13, 0):
            rows, csum = gen.bulk_rowmajor(keys, ivs, iv_bits, T)
            want = oracle.bulk_rowmajor(keys[sample], ivs[sample], iv_bits, T)
            assert np.array_equal(rows[sample], want), iv_bits
            gen.init_material(keys, ivs if iv_bits else None, iv_bits)
            ref_rows = gen.generate_rowmajor(T)
            assert gen.checksum() == csum and np.array_equal(rows, ref_rows), iv_bits
            gen.bulk_rowmajor(keys, ivs, iv_bits, 8)
            with pytest.raises(pkg.Mk2Error):                   # a multi-block bulk call leaves no resumable state
                gen.generate_rowmajor(8)
        # device buffers in, device buffer out, pitch wider than the row
        dk, di = torch.from_numpy(keys).cuda(), torch.from_numpy(ivs).cuda()
        dout = torch.zeros((N, T // 8 + 16), dtype=torch.uint8, device="cuda")
        _, csum_dev = gen.bulk_rowmajor(dk, di, 80, T, dout)
        rows80, csum80 = gen.bulk_rowmajor(keys, ivs, 80, T)
        assert csum_dev == csum80 and np.array_equal(dout[:, : T // 8].cpu().numpy(), rows80)
        # one block only: the context stays resumable
        small, _ = gen.bulk_rowmajor(keys[:5000], ivs[:5000], 80, 64)
        more = gen.generate_rowmajor(64)
        both = oracle.bulk_rowmajor(keys[:5000], ivs[:5000], 80, 128)
        assert np.array_equal(np.hstack([small, more]), both)


def test_every_block_tail_length(pkg, oracle):
    """The keystream loops run clock_block<K> (K = 6 column-major, 5 row-major) plus a one-clock tail, the init
    kernel blocks of 4 over L_iv + 80 load clocks: every remainder of every block length, in one call and resumed."""
    rng = np.random.default_rng(66)
    N = 77
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    for iv_bits in (0, 1, 2, 3, 80):                                   # load clocks 80..83, 160: all remainders mod 4
        want = oracle.bulk_colmajor(keys, ivs, iv_bits, 64)
        with pkg.MickeyGenerator(0) as gen:
            for T in range(1, 15):
                gen.init_material(keys, ivs, iv_bits)
                assert np.array_equal(gen.generate_colmajor(T), want[:T]), (iv_bits, T)
            gen.init_material(keys, ivs, iv_bits)
            got = np.vstack([gen.generate_colmajor(n) for n in (1, 5, 6, 7, 11, 13, 21)])   # resume at every phase
            assert np.array_equal(got, want), iv_bits
    want_rows = oracle.bulk_rowmajor(keys, ivs, 80, 320)
    with pkg.MickeyGenerator(0) as gen:
        for T in (8, 16, 24, 32, 40, 48, 248, 256, 264, 320):
            gen.init_material(keys, ivs, 80)
            assert np.array_equal(gen.generate_rowmajor(T), want_rows[:, : T // 8]), T


def test_randomized_differential(pkg, oracle):
    """Seeded random sweep over instance counts, clock counts, IV lengths (uniform and ragged), layouts and
    scheduling knobs: every combination must equal the oracle bit for bit (the reference uses hypothesis for
    its layout round trips, tests/test_bitslab.py:68-74; this is the same idea for the whole path)."""
    rng = np.random.default_rng(20260101)
    for case in range(40):
        N = int(rng.integers(1, 6000))
        keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
        ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
        ragged = bool(rng.integers(0, 2))
        iv_bits = rng.integers(0, 81, N, dtype=np.uint8) if ragged else int(rng.integers(0, 81))
        row = bool(rng.integers(0, 2))
        T = int(rng.integers(1, 400)) * 8 if row else int(rng.integers(1, 2500))
        block = int(rng.choice([0, 32, 96, 128, 224, 256]))
        chunk = int(rng.choice([0, 128, 256, 777, 4096]))
        split = int(rng.integers(0, T // 8 + 1)) * 8 if row else int(rng.integers(0, T + 1))
        with pkg.MickeyGenerator(0) as gen:
            gen.set_block_threads(block)
            gen.set_chunk_clocks(chunk)
            if ragged:
                gen.init_ragged(keys, ivs, iv_bits)
            else:
                gen.init_material(keys, ivs, iv_bits)
            if row:
                got = np.zeros((N, T // 8), np.uint8)
                gen.generate_rowmajor(split, got, byte_offset=0)                 # two calls: resume mid-stream
                gen.generate_rowmajor(T - split, got, byte_offset=split // 8)
                want = oracle.bulk_rowmajor(keys, ivs, iv_bits, T)
            else:
                a = gen.generate_colmajor(split) if split else np.zeros((0, (N + 31) // 32), np.uint32)
                b = gen.generate_colmajor(T - split) if T - split else np.zeros((0, (N + 31) // 32), np.uint32)
                got = np.vstack([a, b])
                want = oracle.bulk_colmajor(keys, ivs, iv_bits, T)
                assert gen.checksum() == oracle.checksum_colmajor(want)
        assert np.array_equal(got, want), (case, N, T, ragged, row, block, chunk, split)


def test_acceptance_thousand_random_instances(pkg, oracle):
    """The reference's acceptance criterion (tests/test_acceptance.py:103-135): 1000 random MICKEY instances
    x 10 000 bits, IV length random 0..10 bytes, sliced engine == per-instance scalar streams."""
    import random

    rng = random.Random(0xACCE)
    N, T = 1000, 10_000
    keys = np.frombuffer(rng.randbytes(10 * N), np.uint8).reshape(N, 10).copy()
    ivs = np.zeros((N, 10), np.uint8)
    nbits = np.zeros(N, np.uint8)
    for n in range(N):
        ln = rng.randrange(0, 11)
        ivs[n, :ln] = np.frombuffer(rng.randbytes(ln), np.uint8) if ln else 0
        nbits[n] = 8 * ln
    got = pkg.bulk_rowmajor(keys, ivs, nbits, T)
    assert np.array_equal(got, oracle.bulk_rowmajor(keys, ivs, nbits, T))
    for n in (0, 499, 999):                      # and the bit-serial engine agrees on single instances
        st = oracle.Scalar.from_key_iv(keys[n].tobytes(), ivs[n, : nbits[n] // 8].tobytes())
        assert st.keystream_bytes(T // 8) == got[n].tobytes()


# ---------------------------------------------------------------- round 2: host buffers, ragged at scale, LSB rows, faults

def test_pageable_host_outputs_go_through_bounce_tiles(pkg, oracle):
    """Caller-owned PAGEABLE numpy arrays (what kernels.py:194-200 returns) large enough for the pinned bounce
    pipeline: several staging tiles per call, column-major (contiguous and strided), row-major (pitched) and the
    one-shot bulk call -- all bit-exact against the oracle; the pool-backed default arrays agree."""
    N, T = (1 << 17) + 96, 4096                                        # 64 MiB per layout: the copy lanes' threshold
    keys, ivs = random_arrays(77, N)
    want_c = oracle.bulk_colmajor(keys, ivs, 80, T)
    want_r = oracle.bulk_rowmajor(keys, ivs, 80, T)
    G = (N + 31) // 32
    with pkg.MickeyGenerator(0) as gen:
        gen.set_stage_bytes(5 << 20)                                   # 13 column tiles, several row tiles
        gen.set_host_threads(3)
        out = np.empty((T, G), np.uint32)                              # pageable, first touched by the copy workers
        gen.init_material(keys, ivs, 80).generate_colmajor(T, out)
        assert np.array_equal(out, want_c)
        wide = np.zeros((T, G + 5), np.uint32)
        gen.init_material(keys, ivs, 80).generate_colmajor(T, wide, stride_words=G + 5)
        assert np.array_equal(wide[:, :G], want_c) and not wide[:, G:].any()
        rows = np.zeros((N, T // 8 + 24), np.uint8)
        gen.init_material(keys, ivs, 80).generate_rowmajor(T, rows)
        assert np.array_equal(rows[:, : T // 8], want_r) and not rows[:, T // 8:].any()
        rows2 = np.empty((N, T // 8), np.uint8)
        _, csum = gen.bulk_rowmajor(keys, ivs, 80, T, rows2)
        assert np.array_equal(rows2, want_r) and csum == oracle.checksum_colmajor(want_c)
        gen.set_host_threads(1)                                        # the calling thread alone
        out[:] = 0
        gen.init_material(keys, ivs, 80).generate_colmajor(T, out)
        assert np.array_equal(out, want_c)
        # default result arrays: page-locked blocks from the pool (direct D2H), owned by the caller
        a = gen.init_material(keys, ivs, 80).generate_colmajor(T)
        b = gen.init_material(keys, ivs, 80).generate_rowmajor(T)
        assert np.array_equal(a, want_c) and np.array_equal(b, want_r)
    from paper_1909_04750_b200 import hostmem
    allocs = hostmem.pool.allocs
    del a, b                                                           # blocks go back to the cache ...
    with pkg.MickeyGenerator(0) as gen:
        c = gen.init_material(keys, ivs, 80).generate_colmajor(T)      # ... and are reused without a new allocation
        assert np.array_equal(c, want_c) and hostmem.pool.allocs == allocs


def test_pageable_outputs_with_rows_wider_than_a_lane_slot(pkg, oracle, monkeypatch):
    """Copy lanes when one row of the staging tile is wider than a lane's page-locked slot (column-major output of
    more than 16 M instances with the default 8 MiB sub-chunks): sub-chunks are then pieces of rows.  Forced here
    at 2^19 instances by shrinking the sub-chunk size (MK2_LANE_BYTES, read when a context creates its lanes)."""
    monkeypatch.setenv("MK2_LANE_BYTES", "65536")
    N, T = (1 << 19) + 64, 1024                                        # 65 544-byte rows, 64 MiB of output
    key = bytes.fromhex("123456789abcdef01234")
    G = N // 32
    with pkg.MickeyGenerator(0) as gen:
        out = np.empty((T, G), np.uint32)
        gen.init_counter(key, 0, N).generate_colmajor(T, out)
        csum = gen.checksum()
        wide = np.zeros((T, G + 3), np.uint32)
        gen.init_counter(key, 0, N).generate_colmajor(T, wide, stride_words=G + 3)
    assert int(out.view("<u8").sum(dtype=np.uint64)) == csum == oracle.checksum_counter(key, 0, N, T)
    assert np.array_equal(wide[:, :G], out) and not wide[:, G:].any()
    keys, ivs = oracle.counter_material(key, 64 * 4000, 64)
    assert np.array_equal(out[:, 8000:8002], oracle.bulk_colmajor(keys, ivs, 80, T))


def test_rowmajor_lsb_bit_order(pkg, oracle):
    """bit_order="lsb" of words_to_lane_bytes / words_lane_major_bytes (kernels.py:604-621) straight from the GPU:
    the tensor-memory kernel, the shared-memory kernel, ragged tails and the host mirror's helpers agree."""
    N, T = 2048 + 40, 1024 + 136
    keys, ivs = random_arrays(31, N)
    msb = oracle.bulk_rowmajor(keys, ivs, 80, T)
    want = np.packbits(np.unpackbits(msb, axis=1), axis=1, bitorder="little")
    for staging in (0, 1):
        with pkg.MickeyGenerator(0) as gen:
            gen.set_row_staging(staging)
            got = gen.init_material(keys, ivs, 80).generate_rowmajor(T, bit_order="lsb")
            assert np.array_equal(got, want), staging
            assert np.array_equal(gen.init_material(keys, ivs, 80).generate_rowmajor(T), msb)
    assert np.array_equal(pkg.bulk_rowmajor(keys, ivs, 80, T, bit_order="lsb"), want)
    words = pkg.mickey_sliced_words([pkg.MickeyKeyIv(keys[j].tobytes(), ivs[j].tobytes()) for j in range(64)], T)
    assert pkg.words_lane_major_bytes(words, 64, "lsb") == want[:64].tobytes()
    with pytest.raises(ValueError):
        pkg.bulk_rowmajor(keys, ivs, 80, T, bit_order="big")


def test_ragged_iv_lengths_at_scale(pkg, oracle, torch_cuda):
    """The reference's acceptance workload shape (random IV length of 0..10 bytes per instance,
    tests/test_acceptance.py:103-135) at 2^17 instances, plus bit-granular lengths and unused lanes: the
    vectorised packing + masked-block init against the oracle's per-lane scalar init, every instance
    (whole-job checksum) and sampled rows; device-resident inputs take the same path."""
    torch = torch_cuda
    N, T = 1 << 17, 256
    rng = np.random.default_rng(2024)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    for name, nbits in (("bytes", (8 * rng.integers(0, 11, N)).astype(np.uint8)),
                        ("bits", rng.integers(0, 81, N).astype(np.uint8)),
                        ("short", rng.integers(0, 24, N).astype(np.uint8))):
        want = oracle.checksum_material(keys, ivs, nbits, T)
        with pkg.MickeyGenerator(0) as gen:
            gen.init_ragged(keys, ivs, nbits)
            col = gen.generate_colmajor(T)
            assert gen.checksum() == want, name
            assert int(col.view("<u8").sum(dtype=np.uint64)) == want, name
            idx = np.unique(np.concatenate([[0, 31, 32, N - 1], rng.integers(0, N, 200)]))
            gen.init_ragged(torch.from_numpy(keys).cuda(), torch.from_numpy(ivs).cuda(), torch.from_numpy(nbits).cuda())
            rows = gen.generate_rowmajor(T)
            assert gen.checksum() == want, name
            for n in idx:
                lane = oracle.bulk_rowmajor(keys[n:n + 1], ivs[n:n + 1], nbits[n:n + 1], T)[0]
                assert np.array_equal(rows[n], lane), (name, n)
    # int64 lengths (numpy's default) are converted, not read as raw bytes; out-of-range values are rejected
    with pkg.MickeyGenerator(0) as gen:
        a = gen.init_ragged(keys[:96], ivs[:96], nbits[:96].astype(np.int64)).generate_colmajor(64)
        b = gen.init_ragged(keys[:96], ivs[:96], nbits[:96].tolist()).generate_colmajor(64)
        c = gen.init_ragged(keys[:96], ivs[:96], nbits[:96]).generate_colmajor(64)
        assert np.array_equal(a, c) and np.array_equal(b, c)
        with pytest.raises(ValueError, match="lane 7"):
            bad = nbits[:96].astype(np.int64)
            bad[7] = 300
            gen.init_ragged(keys[:96], ivs[:96], bad)


def test_failures_leave_the_context_usable(pkg, oracle, torch_cuda):
    """Fault injection through the C ABI: an init that cannot get its state arrays (NOMEM), a host-output call
    that cannot get its staging tiles, bad arguments in the middle of a session.  Afterwards the same context
    must report 'no material' (not launch on freed buffers) and then work normally."""
    torch = torch_cuda
    keys, ivs = random_arrays(5, 4096)
    want = oracle.bulk_colmajor(keys, ivs, 80, 128)
    gen = pkg.MickeyGenerator(0)
    gen.init_material(keys, ivs, 80)
    with pytest.raises(pkg.Mk2Error, match="code -5"):                 # 2^35 instances = 860 GB of state
        gen.init_counter(bytes(10), 0, 1 << 35)
    with pytest.raises(pkg.Mk2Error, match="no key/IV material"):      # the old state is gone, and known to be gone
        gen.generate_colmajor(8)
    with pytest.raises(pkg.Mk2Error, match="no key/IV material"):
        gen.checksum()
    assert np.array_equal(gen.init_material(keys, ivs, 80).generate_colmajor(128), want)
    # staging tiles that do not fit: fill the device, ask for a host output that needs 2 x 1 GiB of staging
    big_n = 1 << 21
    gen.init_counter(bytes(10), 0, big_n)
    gen.set_stage_bytes(1 << 30)
    free = torch.cuda.mem_get_info()[0]
    hog = torch.empty(max(0, free - (768 << 20)), dtype=torch.uint8, device="cuda")
    host = np.empty((8192, big_n // 32), np.uint32)
    with pytest.raises(pkg.Mk2Error, match="code -5"):
        gen.generate_colmajor(8192, host)
    del hog
    torch.cuda.empty_cache()
    gen.set_stage_bytes(0)
    ref = pkg.MickeyGenerator(0)
    a = gen.init_counter(bytes(10), 0, 4096).generate_colmajor(256)
    b = ref.init_counter(bytes(10), 0, 4096).generate_colmajor(256)
    assert np.array_equal(a, b)
    # bulk call failing on its arguments does not clobber the live state
    gen.init_material(keys, ivs, 80)
    with pytest.raises(ValueError):
        gen.bulk_rowmajor(keys, ivs, 80, 12)                            # not a multiple of 8 (Python-side check)
    with pytest.raises(ValueError):
        gen._ck(gen._lib.mk2_bulk_rowmajor(gen._ctx, keys.ctypes.data, ivs.ctypes.data, 10, 80, 4096, 64, 0, 8, None),
                "mk2_bulk_rowmajor")                                    # NULL out
    assert np.array_equal(gen.generate_colmajor(128), want)
    # derivation tags (seedgen.py:24-31): aes-ctr and unknown tags are rejected before anything is allocated
    for tag in (0, 1, 4):
        with pytest.raises(ValueError):
            gen.derive_material(bytes(range(32)), 0, 8, algo_tag=tag)
    kg, ig = gen.derive_material(bytes(range(32)), 0, 8, algo_tag=2)
    assert kg.shape == (8, 10) and ig.shape == (8, 8)
    wk, wi = oracle.derive_material(bytes(range(32)), 0, 8, tag=2)
    assert np.array_equal(kg, wk) and np.array_equal(ig, wi[:, :8])
    gen.close()
    ref.close()


def test_entry_points_restore_the_callers_device(pkg, torch_cuda):
    """Every C-ABI entry point runs under a device guard: the caller's current device is unchanged."""
    torch = torch_cuda
    before = torch.cuda.current_device()
    with pkg.MickeyGenerator(0) as gen:
        gen.init_counter(bytes(10), 0, 64).generate_colmajor(8)
        gen.checksum()
    assert torch.cuda.current_device() == before
    x = torch.ones(4, device="cuda")
    assert x.device.index == before and float(x.sum()) == 4.0


def test_reference_shaped_calls_reuse_idle_contexts(pkg, golden):
    """mickey_sliced_words / MickeySliced.from_key_ivs in the reference's 64-lane batching pattern
    (cli.py:219-231) take an idle context of the thread instead of creating and destroying one per call."""
    from paper_1909_04750_b200 import hostmem
    from paper_1909_04750_b200.generator import MickeyGenerator
    import gc
    gc.collect()                          # engines of earlier tests still waiting for the collector release theirs now
    hostmem.drop_idle_contexts()
    rec = golden["kats"][0]
    mats = [pkg.MickeyKeyIv(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"]))] * 64
    w1 = pkg.mickey_sliced_words(mats, 128)
    idle = hostmem._idle((MickeyGenerator, 0))
    assert len(idle) == 1
    ctx = idle[0]._ctx.value
    for _ in range(3):
        assert np.array_equal(pkg.mickey_sliced_words(mats, 128), w1)
    assert len(idle) == 1 and idle[0]._ctx.value == ctx              # the same context served every call
    eng = pkg.MickeySliced.from_key_ivs(mats, 64)
    assert len(idle) == 0 and eng._gen._ctx.value == ctx
    eng2 = pkg.MickeySliced.from_key_ivs(mats, 64)                     # a second live engine gets its own
    assert eng2._gen._ctx.value != ctx
    assert eng.keystream_words(16) == eng2.keystream_words(16) == [int(w) for w in w1[:16]]
    del eng, eng2
    assert len(idle) == 2
    assert pkg.words_to_lane_bytes(w1, 5)[:16].hex() == rec["ks"]
    hostmem.drop_idle_contexts()


def test_nist_rows_from_the_gpu_match_the_rows_the_suite_judged(pkg):
    """Closes the chain of tests/test_nist_quality.py: the 100 x 1 Mbit streams of the reference's acceptance
    criterion 4 (test_acceptance.py:188-223), on which the reference's NIST SP 800-22 subset passes, are, by
    SHA-256, exactly what the B200 emits for them (cli.suite_streams: seed-derived material, one row-major run)."""
    import json
    from pathlib import Path
    from paper_1909_04750_b200 import cli
    fx = json.loads((Path(__file__).resolve().parent / "golden" / "nist_rows_sha256.json").read_text())
    rows = cli.suite_streams(bytes.fromhex(fx["seed"]), fx["rows"], fx["nbits"])
    assert [hashlib.sha256(r.tobytes()).hexdigest() for r in rows] == fx["sha256"]


def _gpu_rank_worker(rank, world, port, n, T, key_hex, q):
    """One rank of the multi-GPU path on the one GPU there is: its own context and stream on cuda:0, its shard of
    the key/IV range, and the checksum all-reduce -- through a world_size-2 gloo group (NCCL needs one GPU per
    rank; the collective's arithmetic, the sharding and the group-offset weighting are the same code)."""
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1909_04750_b200 as p
        from paper_1909_04750_b200 import sharding
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        gen, sh = sharding.counter_generator(bytes.fromhex(key_hex), n, world, rank, device=0)
        gen.set_stream(stream.cuda_stream)
        out = torch.empty((T, sh.groups), dtype=torch.int32, device="cuda")
        dist.barrier()                                   # both ranks generate at the same time on the same device
        gen.generate_colmajor(T, out)
        stream.synchronize()
        local = gen.checksum()
        buf = int(out.view(torch.int64).sum().item()) % (1 << 64) if sh.groups % 2 == 0 and sh.group_offset % 2 == 0 else None
        total = sharding.allreduce_checksum(local)       # the path's only collective
        gen.set_stream(None)
        gen.close()
        q.put((rank, sh.first, sh.count, local, total, buf))
    finally:
        dist.destroy_process_group()


def test_two_ranks_drive_the_gpu_and_allreduce_their_checksums(pkg, golden, oracle):
    """bench.py --gpus 2's data path with the real kernels: two processes, each with its own context on the GPU and a
    disjoint key/IV range, generate concurrently and combine their checksums with one all-reduce; the sum must equal
    the single-context run and the oracle's whole-job checksum."""
    import socket
    import torch.multiprocessing as mp
    key_hex = golden["counter_iv"][0]["key"]
    n, T, world = (1 << 17) + 64, 2048, 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_rank_worker, args=(r, world, port, n, T, key_hex, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][1] == 0 and res[1][1] == res[0][2] and res[0][2] + res[1][2] == n
    want = oracle.checksum_counter(bytes.fromhex(key_hex), 0, n, T)
    assert res[0][4] == res[1][4] == want                              # all-reduced sum, on both ranks
    assert (res[0][3] + res[1][3]) % (1 << 64) == want
    for r in res:
        if r[5] is not None:
            assert r[5] == r[3]                                        # each rank's emitted buffer carries its checksum
    with pkg.MickeyGenerator(0) as gen:                                # the same job on one context
        gen.init_counter(bytes.fromhex(key_hex), 0, n).generate_colmajor(T)
        assert gen.checksum() == want


def test_suite_streams_match_the_reference_cli(pkg, oracle, tmp_path):
    """`cli streams` / cli.suite_streams: the streams the reference's `slicerng test` would judge (cli.py:212-231),
    all batches from one init + row-major generation on the GPU; digests made by the reference itself."""
    import json
    from pathlib import Path
    from paper_1909_04750_b200 import cli
    fx = json.loads((Path(__file__).resolve().parent / "golden" / "suite_streams_sha256.json").read_text())
    for c in fx["cases"]:
        rows = cli.suite_streams(bytes.fromhex(c["seed"]), c["streams"], c["stream_bits"])
        assert rows.shape == (c["streams"], (c["stream_bits"] + 7) // 8)
        assert [sha(r.tobytes()) for r in rows] == c["sha256"], c["seed"]
    big = cli.suite_streams(bytes.fromhex("11" * 32), 1000, 8192)          # 16 batches, one GPU call
    assert np.array_equal(big, oracle.suite_streams(bytes.fromhex("11" * 32), 1000, 8192))
    out = tmp_path / "s.npy"
    assert cli.main(["streams", "--streams", "5", "--stream-bits", "4096", "--out", str(out)]) == 0
    assert np.array_equal(np.load(out), big[:5, :512])
    d = tmp_path / "raw"
    assert cli.main(["streams", "--streams", "3", "--stream-bits", "77", "--seed", "a7" + "00" * 31, "--out", str(d)]) == 0
    assert sha((d / "stream_00002.bin").read_bytes()) == fx["cases"][3]["sha256"][2]
    with pytest.raises(SystemExit):
        cli.main(["streams", "--streams", "20000", "--stream-bits", "8", "--out", str(out)])   # > 256 batches


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_multi_rank_code_path_on_one_gpu(scaling):
    """bench.py launched the way the driver launches it for N > 1 (torch.distributed.run, one process per rank),
    with the gloo debug backend so that two ranks can share the one GPU: disjoint key/IV ranges per rank, per-rank
    records, the all-reduced checksum and its in-run cross-check, weak and strong (fixed total job) scaling."""
    import json
    import socket
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(root / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--dist-backend", "gloo", "--clocks", "16384", "--no-e2e", "--no-curand", "--no-cpu-baseline", "--no-latency"]
    cmd += ["--instances-log2", "16"] if scaling == "weak" else ["--scaling", "strong", "--total-bits", str(16384 * (3 * 32768 + 64))]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=str(root))
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]                          # rank 0 prints the one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0 and d["gpu_launches"] > 0
    r0, r1 = d["ranks"]
    assert (r0["rank"], r1["rank"]) == (0, 1) and r0["first"] == 0 and r1["first"] == r0["count"]
    total = r0["count"] + r1["count"]
    assert total == d["config"]["total_instances"] == (2 << 16 if scaling == "weak" else 3 * 32768 + 64)
    assert d["checksum_check"]["equal"] is True and "gloo" in d["checksum_check"]["collective"]
    csum = (int(r0["checksum"], 16) + int(r1["checksum"], 16)) % (1 << 64)
    assert int(d["checksum_u64_sum"], 16) == csum
    # the same job on one context gives the same checksum (the last timed step's key/IV ranges)
    import paper_1909_04750_b200 as p
    step = (2 + 3 - 1) % 4                                              # bench rotates 4 starting indices over its steps
    with p.MickeyGenerator(0) as gen:
        gen.init_counter(bytes.fromhex("123456789abcdef01234"), step * total, total).generate_colmajor(16384)
        assert gen.checksum() == csum
