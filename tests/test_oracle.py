"""Pins the CPU oracle (oracle/mickey_oracle.c) to the reference.

Every expected value comes from tests/golden/mickey_golden.json, which
oracle/gen_golden.py produced by running the reference package itself, or
from the eSTREAM vectors the reference embeds (vectors.py:41-60).  CPU only.
"""
import hashlib

import numpy as np
import pytest

from conftest import golden_material


def sha(b):
    return hashlib.sha256(b).hexdigest()


def bits_int(bits):
    return sum(int(b) << i for i, b in enumerate(bits))


def test_tables_match_reference(oracle, golden):
    t = oracle.tables()
    g = golden["tables"]
    assert [i for i, b in enumerate(t["RTAPS"]) if b] == g["RTAPS"]
    assert len(g["RTAPS"]) == 50  # tests/test_mickey.py:28-35
    for name in ("COMP0", "COMP1", "FB0", "FB1"):
        assert t[name] == g[name]
    assert t["COMP0"][0] == t["COMP0"][99] == t["COMP1"][0] == t["COMP1"][99] == 0


def test_estream_vectors_scalar(oracle, golden):
    for rec in golden["kats"]:
        st = oracle.Scalar.from_key_iv(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"]))
        assert f"{bits_int(st.r):x}" == rec["post_init_r"]
        assert f"{bits_int(st.s):x}" == rec["post_init_s"]
        assert st.keystream_bytes(16).hex() == rec["ks"]


@pytest.mark.parametrize("width", [32, 64])
def test_estream_vectors_every_lane(oracle, golden, width):
    # vectors.verify_vectors: every lane of the sliced engine (vectors.py:189-197)
    for rec in golden["kats"]:
        mats = [(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"]))] * width
        words = oracle.sliced_words(mats, 128, width)
        full = (1 << width) - 1
        assert set(int(w) for w in words) <= {0, full}
        lane_bits = ((words >> np.uint64(width - 1)) & np.uint64(1)).astype(np.uint8)
        assert np.packbits(lane_bits).tobytes() == bytes.fromhex(rec["ks"])


def test_scalar_cases(oracle, golden):
    for rec in golden["scalar_cases"]:
        key, iv = golden_material(rec)
        st = oracle.Scalar.from_key_iv(key, iv)
        assert f"{bits_int(st.r):x}" == rec["post_init_r"]
        assert f"{bits_int(st.s):x}" == rec["post_init_s"]
        assert st.keystream_bytes(256).hex() == rec["ks256"]


def test_zero_state_clock_and_trace(oracle, golden):
    st = oracle.Scalar()
    st.clock_kg(False, 0)
    assert f"{bits_int(st.r):x}" == golden["zero_state_one_clock"]["r"]
    assert f"{bits_int(st.s):x}" == golden["zero_state_one_clock"]["s"]
    k = golden["kats"][0]
    st = oracle.Scalar.from_key_iv(bytes.fromhex(k["key"]), bytes.fromhex(k["iv"]))
    for r_hex, s_hex in golden["kat0_state_trace_100"]:
        st.clock_kg(False, 0)
        assert f"{bits_int(st.r):x}" == r_hex and f"{bits_int(st.s):x}" == s_hex


def test_sliced_cases(oracle, golden):
    for case in golden["sliced_cases"]:
        mats = [golden_material(m) for m in case["materials"]]
        eng = oracle.Sliced.from_key_ivs(mats)
        width = case["width"]
        mask = (1 << width) - 1
        # lanes >= width of the 64-lane oracle hold padding; compare the low `width` lanes
        assert [f"{w & mask:x}" for w in eng.rregs] == [f"{int(x, 16) & mask:x}" for x in case["init_state"]["r"]], case["name"]
        assert [f"{w & mask:x}" for w in eng.sregs] == [f"{int(x, 16) & mask:x}" for x in case["init_state"]["s"]], case["name"]
        words = oracle.sliced_words(mats, case["nclocks"], width)
        assert sha(words.astype("<u8").tobytes()) == case["words_sha256"], case["name"]
        if case["words_hex"]:
            assert words.astype("<u8").tobytes().hex() == case["words_hex"]
        # resumable engine agrees with the restart-only loop (mickey.py:362 vs kernels.py:46)
        stepped = eng.keystream_words(case["nclocks"]) & np.uint64(mask)
        assert np.array_equal(stepped, words)


def test_c1_lockstep_million(oracle, golden):
    rec = golden["kats"][0]
    mats = [(bytes.fromhex(rec["key"]), bytes.fromhex(rec["iv"]))] * 32
    words = oracle.sliced_words(mats, 1_000_000, 32)
    assert sha(words.astype("<u4").tobytes()) == rec["c1_words_u4_sha256"]
    lane0 = np.packbits((words & np.uint64(1)).astype(np.uint8)).tobytes()
    assert sha(lane0) == rec["c1_lane0_sha256"]
    assert lane0[-16:].hex() == rec["c1_lane0_tail16"]


def test_bench_seed_lanes(oracle, golden):
    b = golden["bench_seed"]
    mats = [golden_material(m) for m in b["materials"]]
    keys, ivs, nb = oracle.pack_materials(mats)
    col = oracle.bulk_colmajor(keys, ivs, 80, b["nclocks"])
    assert sha(col.tobytes()) == b["words_u8_sha256"]
    assert f"{oracle.checksum_colmajor(col):x}" == b["u64_wrap_sum"]
    row = oracle.bulk_rowmajor(keys, ivs, 80, b["nclocks"] // 8 * 8)
    assert sha(row.tobytes()) == b["lane_major_sha256"]
    assert row[0, :16].tobytes().hex() == b["lane0_first16"]


def test_counter_iv_sets(oracle, golden):
    for c in golden["counter_iv"]:
        keys, ivs = oracle.counter_material(bytes.fromhex(c["key"]), c["first"], c["n"])
        col = oracle.bulk_colmajor(keys, ivs, 80, c["nclocks"])
        row = oracle.bulk_rowmajor(keys, ivs, 80, c["nclocks"])
        assert sha(col.tobytes()) == c["colmajor_sha256"]
        assert sha(row.tobytes()) == c["rowmajor_sha256"]
        assert row[0, :16].tobytes().hex() == c["lane0_first16"]
        assert row[-1, :16].tobytes().hex() == c["lane_last_first16"]
        assert f"{oracle.checksum_colmajor(col):x}" == c["u64_wrap_sum"]
        assert f"{int(np.bitwise_xor.reduce(np.ascontiguousarray(col).view('<u8').ravel())):x}" == c["xor_fold"]


def test_bulk_ragged_and_partial_batches(oracle):
    # bulk layouts agree with per-lane scalar streams, incl. N not a multiple of 32/64
    rng = np.random.default_rng(7)
    N, T = 150, 264
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    nbits = rng.integers(0, 81, N, dtype=np.uint8)
    row = oracle.bulk_rowmajor(keys, ivs, nbits, T)
    col = oracle.bulk_colmajor(keys, ivs, nbits, T)
    assert col.shape == (T, 5)
    for n in (0, 31, 32, 63, 64, 100, 149):
        bits = np.unpackbits(ivs[n])[: nbits[n]].tolist()
        ks = oracle.Scalar.from_key_iv(keys[n].tobytes(), bits).keystream_bytes(T // 8)
        assert row[n].tobytes() == ks
        lane = ((col[:, n // 32] >> np.uint32(n % 32)) & 1).astype(np.uint8)
        assert np.packbits(lane).tobytes() == ks


def test_aes_blocks_and_seed_derivation(oracle, golden):
    # vectors.py:78-93 (FIPS-197 examples) and seedgen.py:57-86 as run by the reference
    for b in golden["aes_blocks"]:
        assert oracle.aes128_encrypt(bytes.fromhex(b["key"]), bytes.fromhex(b["pt"])).hex() == b["ct"]
    for rec in golden["seedgen"]:
        keys, ivs = oracle.derive_material(bytes.fromhex(rec["seed"]), 0, 64)
        for lane, m in rec["lanes"].items():
            assert keys[int(lane)].tobytes().hex() == m["key"] and ivs[int(lane)].tobytes().hex() == m["iv"]
        blob = b"".join(keys[j].tobytes() + ivs[j].tobytes() for j in range(64))
        assert sha(blob) == rec["all64_sha256"]
    # the bench-seed lanes of bench.py:43-45 are the same derivation
    mats = golden["bench_seed"]["materials"]
    keys, ivs = oracle.derive_material(bytes.fromhex(golden["seedgen"][0]["seed"]), 0, 64)
    assert [keys[j].tobytes().hex() for j in range(64)] == [m["key"] for m in mats]
    assert [ivs[j].tobytes().hex() for j in range(64)] == [m["iv"] for m in mats]
    # windows agree with the whole
    k2, i2 = oracle.derive_material(bytes.fromhex(golden["seedgen"][1]["seed"]), 40, 10)
    kall, iall = oracle.derive_material(bytes.fromhex(golden["seedgen"][1]["seed"]), 0, 64)
    assert np.array_equal(k2, kall[40:50]) and np.array_equal(i2, iall[40:50])


def test_grain_oracle_matches_reference(oracle, golden):
    g = golden["grain"]
    for v in g["vectors"]:
        assert oracle.grain_scalar_bytes(bytes.fromhex(v["key"]), bytes.fromhex(v["iv"]), 16, v["bit_order"]).hex() == v["ks"]
    for c in g["scalar_cases"]:
        eng = oracle.GrainSliced.from_key_ivs([(bytes.fromhex(c["key"]), bytes.fromhex(c["iv"]))])
        assert f"{sum((w & 1) << i for i, w in enumerate(eng.b)):x}" == c["post_init_b"]
        assert f"{sum((w & 1) << i for i, w in enumerate(eng.s)):x}" == c["post_init_s"]
        assert oracle.grain_scalar_bytes(bytes.fromhex(c["key"]), bytes.fromhex(c["iv"]), 128).hex() == c["ks128_msb"]
        assert oracle.grain_scalar_bytes(bytes.fromhex(c["key"]), bytes.fromhex(c["iv"]), 64, "lsb").hex() == c["ks64_lsb"]
    for c in g["sliced_cases"]:
        mats = [(bytes.fromhex(m["key"]), bytes.fromhex(m["iv"])) for m in c["materials"]]
        eng = oracle.GrainSliced.from_key_ivs(mats)
        assert [f"{x:x}" for x in eng.b] == c["init_state"]["b"] and [f"{x:x}" for x in eng.s] == c["init_state"]["s"]
        assert eng.keystream_words(c["nclocks"]).astype("<u8").tobytes().hex() == c["words_hex"], c["name"]
    mats = [(bytes.fromhex(m["key"]), bytes.fromhex(m["iv"])) for m in g["sliced_cases"][1]["materials"]]
    keys, ivs = oracle._grain_arrays(mats)
    T = g["long"]["nclocks"]
    assert sha(oracle.grain_bulk_colmajor(keys, ivs, T).tobytes()) == g["long"]["words_u8_sha256"]
    assert sha(oracle.grain_bulk_rowmajor(keys, ivs, T).tobytes()) == g["long"]["lane_major_msb_sha256"]
    assert sha(oracle.grain_bulk_rowmajor(keys, ivs, T, "lsb").tobytes()) == g["long"]["lane_major_lsb_sha256"]


def test_whole_job_checksum_matches_reference_and_buffer_checksum(oracle, golden):
    """mk2o_checksum_job (the full-coverage checker of the BASELINE-size GPU tests) against the reference's own
    uint64 wrap-sums of the counter-IV sets, and against the checksum of the materialised oracle buffer."""
    for rec in golden["counter_iv"]:
        key = bytes.fromhex(rec["key"])
        assert f"{oracle.checksum_counter(key, rec['first'], rec['n'], rec['nclocks']):016x}" == rec["u64_wrap_sum"].rjust(16, "0")
    key = bytes.fromhex("123456789abcdef01234")
    for first, n, T in ((0, 64, 100), (64, 96, 77), (128, 992, 33), (0, 32, 8)):
        k, v = oracle.counter_material(key, first, n)
        want = oracle.checksum_colmajor(oracle.bulk_colmajor(k, v, 80, T), first // 32)
        assert oracle.checksum_counter(key, first, n, T) == want
        assert oracle.checksum_counter(key, first, n, T, nthreads=1) == want
    rng = np.random.default_rng(3)
    for n, T, ivb, go in ((1000, 65, 80, 0), (64, 12, 13, 1), (33, 9, 0, 3)):
        k = rng.integers(0, 256, (n, 10), dtype=np.uint8)
        v = rng.integers(0, 256, (n, 10), dtype=np.uint8)
        assert oracle.checksum_material(k, v, ivb, T, go) == oracle.checksum_colmajor(oracle.bulk_colmajor(k, v, ivb, T), go)
    nb = rng.integers(0, 81, 1000).astype(np.uint8)   # ragged IV lengths
    k = rng.integers(0, 256, (1000, 10), dtype=np.uint8)
    v = rng.integers(0, 256, (1000, 10), dtype=np.uint8)
    assert oracle.checksum_material(k, v, nb, 40) == oracle.checksum_colmajor(oracle.bulk_colmajor(k, v, nb, 40))


def test_suite_streams_match_the_reference_cli(oracle):
    """The streams `slicerng test` generates for its NIST suite (cli._suite_streams, cli.py:212-231), digests made
    by the reference itself (oracle/gen_suite_streams.py): batch seeds, partial last batch, bit counts that are
    not a multiple of 8."""
    import json
    from pathlib import Path
    fx = json.loads((Path(__file__).resolve().parent / "golden" / "suite_streams_sha256.json").read_text())
    for c in fx["cases"]:
        rows = oracle.suite_streams(bytes.fromhex(c["seed"]), c["streams"], c["stream_bits"])
        assert rows[0, :16].tobytes().hex() == c["first16"]
        assert [sha(r.tobytes()) for r in rows] == c["sha256"], c["seed"]
