#!/usr/bin/env python
"""Generate tests/golden/mickey_golden.json from the REFERENCE itself.

Run in the build container only (the reference tree does not travel):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

Every expected value below is computed by importing the reference package
`slicerng` (pkg/src/slicerng/{mickey,kernels,vectors,bench,seedgen}.py) and
calling its own engines; nothing here comes from this repo's oracle or CUDA
path.  The JSON is the committed fixture that pins oracle/mickey_oracle.c and,
through it and directly, the CUDA kernels.  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

import numpy as np

try:
    from slicerng import bench as ref_bench
    from slicerng import kernels as ref_kernels
    from slicerng import mickey as ref_mickey
    from slicerng import vectors as ref_vectors
except ImportError:  # pragma: no cover
    sys.exit("reference package not importable: set PYTHONPATH=/root/reference/pkg/src")

MickeyKeyIv = ref_mickey.MickeyKeyIv
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "mickey_golden.json"


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def mat_json(m):
    iv = m.iv
    if isinstance(iv, (bytes, bytearray)):
        return {"key": m.key.hex(), "iv": bytes(iv).hex()}
    return {"key": m.key.hex(), "iv_bits": list(iv)}


def bits_int(bits):
    return sum(b << i for i, b in enumerate(bits))


def words_case(name, mats, nclocks, width):
    """kernels.mickey_sliced_words on `mats` + per-lane scalar cross-check."""
    words = ref_kernels.mickey_sliced_words(mats, nclocks, width)
    pure = ref_mickey.MickeySliced.from_key_ivs(mats, width)
    state = {"r": [f"{w:x}" for w in pure.rregs], "s": [f"{w:x}" for w in pure.sregs]}
    assert [int(w) for w in words] == pure.keystream_words(nclocks)
    return {
        "name": name,
        "width": width,
        "nclocks": nclocks,
        "materials": [mat_json(m) for m in mats],
        "init_state": state,
        "words_hex": words.astype("<u8").tobytes().hex() if nclocks <= 1024 else None,
        "words_sha256": sha(words.astype("<u8").tobytes()),
    }


def main():
    g = {"generator": "oracle/gen_golden.py", "reference": "slicerng @ /root/reference/pkg/src"}

    # --- tables (mickey.py:35-58)
    c = ref_mickey.mickey_constants()
    g["tables"] = {
        "RTAPS": list(c["RTAPS"]),
        "COMP0": list(c["COMP0"]),
        "COMP1": list(c["COMP1"]),
        "FB0": list(c["FB0"]),
        "FB1": list(c["FB1"]),
    }

    # --- eSTREAM KATs (vectors.py:41-60) + post-init states + long digests
    kats = []
    for rec in ref_vectors.MICKEY_VECTORS:
        m = MickeyKeyIv(rec.key, rec.iv)
        st = ref_mickey.MickeyScalarPacked.from_key_iv(m)
        sc = ref_mickey.MickeyScalar.from_key_iv(m)
        assert bits_int(sc.r) == st.r and bits_int(sc.s) == st.s
        # C1: 32 lock-step lanes, T = 1e6 (numba engine)
        words = ref_kernels.mickey_sliced_words([m] * 32, 1_000_000, 32)
        assert set(np.unique(words).tolist()) <= {0, 0xFFFFFFFF}
        lane0 = ref_kernels.words_to_lane_bytes(words, 0)
        assert lane0[:16] == rec.ks
        kats.append({
            "key": rec.key.hex(), "iv": rec.iv.hex(), "ks": rec.ks.hex(),
            "post_init_r": f"{st.r:x}", "post_init_s": f"{st.s:x}",
            "c1_lane0_sha256": sha(lane0),
            "c1_words_u4_sha256": sha(words.astype("<u4").tobytes()),
            "c1_lane0_tail16": lane0[-16:].hex(),
        })
    g["kats"] = kats
    assert ref_vectors.verify_vectors("mickey") == (3, [])

    # --- scalar cases: random key, IV length 0..10 bytes (test_mickey.py:24-25)
    rng = random.Random(0x77)
    scal = []
    for _ in range(8):
        m = MickeyKeyIv(rng.randbytes(10), rng.randbytes(rng.randrange(0, 11)))
        a = ref_mickey.MickeyScalar.from_key_iv(m)
        b = ref_mickey.MickeyScalarPacked.from_key_iv(m)
        r0, s0 = bits_int(a.r), bits_int(a.s)
        assert (r0, s0) == (b.r, b.s)
        ks = a.keystream_bytes(256)
        assert ks == b.keystream_bytes(256)
        scal.append({**mat_json(m), "post_init_r": f"{r0:x}", "post_init_s": f"{s0:x}", "ks256": ks.hex()})
    # bit-length IVs (MickeyKeyIv accepts 0/1 lists, mickey.py:93-98)
    for nbits in (1, 5, 13, 37, 79):
        m = MickeyKeyIv(rng.randbytes(10), [rng.randrange(2) for _ in range(nbits)])
        a = ref_mickey.MickeyScalar.from_key_iv(m)
        scal.append({**mat_json(m), "post_init_r": f"{bits_int(a.r):x}", "post_init_s": f"{bits_int(a.s):x}",
                     "ks256": a.keystream_bytes(256).hex()})
    g["scalar_cases"] = scal

    # --- single-clock traces from the zero state and a KAT state (test_mickey.py:59-83)
    z = ref_mickey.MickeyScalarPacked()
    z.clock_kg(False, 0)
    g["zero_state_one_clock"] = {"r": f"{z.r:x}", "s": f"{z.s:x}"}
    tr = []
    v0 = ref_vectors.MICKEY_VECTORS[0]
    b = ref_mickey.MickeyScalarPacked.from_key_iv(MickeyKeyIv(v0.key, v0.iv))
    for _ in range(100):
        b.clock_kg(False, 0)
        tr.append([f"{b.r:x}", f"{b.s:x}"])
    g["kat0_state_trace_100"] = tr

    # --- sliced cases (test_kernels.py:11-25, test_mickey.py:120-164)
    cases = []
    R = random.Random(0xFA57)
    mm = [MickeyKeyIv(R.randbytes(10), R.randbytes(4)) for _ in range(64)]
    cases.append(words_case("kernels_w32_501", mm[:32], 501, 32))
    cases.append(words_case("kernels_w64_501", mm[:64], 501, 64))
    for width in (32, 64):
        rr = random.Random(width)
        mats = [MickeyKeyIv(rr.randbytes(10), rr.randbytes(rr.randrange(0, 11))) for _ in range(width)]
        cases.append(words_case(f"ragged_random_w{width}_1024", mats, 1024, width))
    rr = random.Random(6)
    mats = [MickeyKeyIv(rr.randbytes(10), rr.randbytes(j % 4)) for j in range(12)]
    cases.append(words_case("ragged_12_lanes_w32", mats, 256, 32))
    cases.append(words_case("ragged_12_lanes_w64", mats, 256, 64))
    rr = random.Random(5)
    mats = [MickeyKeyIv(rr.randbytes(10), rr.randbytes(4)) for _ in range(32)]
    cases.append(words_case("uniform_iv32_w32", mats, 256, 32))
    cases.append(words_case("uniform_7_lanes_w32", mats[:7], 255, 32))
    cases.append(words_case("uniform_40_lanes_w64", (mm + mm)[:40], 64, 64))
    rr = random.Random(11)
    for nbits in (0, 3, 17, 80):
        mats = [MickeyKeyIv(rr.randbytes(10), [rr.randrange(2) for _ in range(nbits)]) for _ in range(64)]
        cases.append(words_case(f"uniform_ivbits{nbits}_w64", mats, 128, 64))
    mats = [MickeyKeyIv(rr.randbytes(10), [rr.randrange(2) for _ in range(rr.randrange(0, 81))]) for _ in range(64)]
    cases.append(words_case("ragged_bitlens_w64", mats, 128, 64))
    v0m = MickeyKeyIv(v0.key, v0.iv)
    rr = random.Random(9)
    mats = [MickeyKeyIv(rr.randbytes(10), rr.randbytes(rr.randrange(0, 11))) for _ in range(16)]
    mats[7] = v0m
    cases.append(words_case("kat_lane7_among_random", mats, 128, 32))
    g["sliced_cases"] = cases

    # --- bench-seed lanes (bench.py:43-45, 95-97), T = 1e6, both layouts
    mats = ref_bench._lane_materials("mickey", 64)
    words = ref_kernels.mickey_sliced_words(mats, 1_000_000, 64)
    lm = ref_kernels.words_lane_major_bytes(words, 64)
    g["bench_seed"] = {
        "materials": [mat_json(m) for m in mats], "nclocks": 1_000_000,
        "words_u8_sha256": sha(words.astype("<u8").tobytes()),
        "lane_major_sha256": sha(lm),
        "lane0_first16": lm[:16].hex(),
        "u64_wrap_sum": f"{int(words.sum(dtype=np.uint64)):x}",
    }
    assert ref_mickey.MickeyScalar.from_key_iv(mats[0]).keystream_bytes(64) == lm[:64]

    # --- counter-IV synthetic set: one key, IV_k = 80-bit BE k
    key = v0.key
    ctr = []
    for first, n, T in ((0, 64, 4096), (1 << 20, 64, 512), ((1 << 40) + 64, 64, 512), (0, 256, 1024)):
        blocks = []
        lane_major = b""
        for b0 in range(0, n, 64):
            ms = [MickeyKeyIv(key, (first + b0 + j).to_bytes(10, "big")) for j in range(64)]
            w = ref_kernels.mickey_sliced_words(ms, T, 64)
            blocks.append(w)
            lane_major += ref_kernels.words_lane_major_bytes(w, 64)
        col = np.stack(blocks, axis=1)  # [T][n/64] u64 == [T][n/32] u32 little-endian
        ctr.append({
            "key": key.hex(), "first": first, "n": n, "nclocks": T,
            "colmajor_sha256": sha(col.astype("<u8").tobytes()),
            "rowmajor_sha256": sha(lane_major),
            "lane0_first16": lane_major[:16].hex(),
            "lane_last_first16": lane_major[(n - 1) * (T // 8):(n - 1) * (T // 8) + 16].hex(),
            "u64_wrap_sum": f"{int(col.sum(dtype=np.uint64)):x}",
            "xor_fold": f"{int(np.bitwise_xor.reduce(col.ravel())):x}",
        })
    g["counter_iv"] = ctr

    # --- lane extraction helpers (kernels.py:600-621; test_kernels.py:75-82)
    w = np.array([0b11, 0b01, 0b10, 0b00] * 2, dtype=np.uint64)
    g["lane_helpers"] = {
        "words": [int(x) for x in w],
        "lane0_bits": ref_kernels.words_to_lane_bits(w, 0).tolist(),
        "lane1_bits": ref_kernels.words_to_lane_bits(w, 1).tolist(),
        "lane0_msb": ref_kernels.words_to_lane_bytes(w, 0).hex(),
        "lane0_lsb": ref_kernels.words_to_lane_bytes(w, 0, "lsb").hex(),
        "lane_major_2": ref_kernels.words_lane_major_bytes(w, 2).hex(),
    }

    # --- seed derivation (seedgen.py:39-86) + the AES block vectors it rests on (vectors.py:78-93)
    from slicerng import seedgen as ref_seedgen
    from slicerng.aes_ctr import AesScalarTable

    sg = []
    for seed in (ref_bench.DEFAULT_SEED, bytes(range(32)), bytes([0xFF] * 31 + [0x01])):
        master = ref_seedgen.MasterSeed(seed, "mickey", 64)
        lanes = {}
        for lane in (0, 1, 2, 31, 63):
            m = ref_seedgen.derive_lane_material(master, lane)
            lanes[str(lane)] = {"key": m.key.hex(), "iv": bytes(m.iv).hex()}
        allm = ref_seedgen.derive_all(master)
        blob = b"".join(m.key + bytes(m.iv) for m in allm)
        sg.append({"seed": seed.hex(), "lanes": lanes, "all64_sha256": sha(blob)})
    g["seedgen"] = sg
    g["aes_blocks"] = [{"key": r.key.hex(), "pt": r.iv.hex(), "ct": r.ks.hex()} for r in ref_vectors.AES_BLOCK_VECTORS]
    for r in ref_vectors.AES_BLOCK_VECTORS:
        assert AesScalarTable(r.key).encrypt_block(r.iv) == r.ks

    # --- CLI outputs (cli.py:102-152): `slicerng gen --algo mickey`, hex format
    import tempfile
    from slicerng import cli as ref_cli

    cli_cases = []
    for argv in (
        ["--bits", "1024"],
        ["--bits", "8192", "--lanes", "4", "--seed", "ab" * 32],
        ["--bits", str(64 * 256), "--lanes", "64", "--seed", ref_bench.DEFAULT_SEED.hex()],
        ["--bits", "128", "--key", "123456789abcdef01234", "--iv", "21436587"],
        ["--bits", "1536", "--key", "123456789abcdef01234", "--lanes", "3"],
        ["--bits", "2048", "--lanes", "7", "--interleave", "bit", "--seed", "cd" * 32],
        ["--bits", "4096", "--lanes", "64", "--interleave", "bit"],
        ["--bits", "1000", "--lanes", "5", "--interleave", "bit", "--key", "00112233445566778899", "--iv", "0102"],
    ):
        with tempfile.NamedTemporaryFile("r", suffix=".hex") as fh:
            assert ref_cli.main(["gen", "--algo", "mickey", "--impl", "sliced", "--out", fh.name, *argv]) == 0
            out = fh.read()
        if "--interleave" not in argv:   # naive == sliced (cli.py:9-11)
            with tempfile.NamedTemporaryFile("r", suffix=".hex") as fh2:
                ref_cli.main(["gen", "--algo", "mickey", "--impl", "naive", "--out", fh2.name, *argv])
                assert fh2.read() == out
        cli_cases.append({"argv": argv, "hex": out})
    g["cli_gen"] = cli_cases
    gcli = []
    for argv in (
        ["--bits", "1024"],
        ["--bits", "4096", "--lanes", "4", "--seed", "ab" * 32],
        ["--bits", "128", "--key", "0123456789abcdef1234", "--iv", "0123456789abcdef"],
        ["--bits", "768", "--key", "00000000000000000000", "--lanes", "3"],
        ["--bits", "2048", "--lanes", "7", "--interleave", "bit", "--seed", "cd" * 32],
        ["--bits", "4096", "--lanes", "64", "--interleave", "bit"],
    ):
        with tempfile.NamedTemporaryFile("r", suffix=".hex") as fh:
            assert ref_cli.main(["gen", "--algo", "grain", "--impl", "sliced", "--out", fh.name, *argv]) == 0
            gcli.append({"argv": argv, "hex": fh.read()})
    g["cli_gen_grain"] = gcli

    # --- Grain v1 (grain.py, kernels.py:268-355): vectors, scalar states, sliced words
    from slicerng import grain as ref_grain

    gg = {"constants": {k: [list(t) if isinstance(t, tuple) else t for t in v] for k, v in ref_grain.grain_constants().items()
                        if k != "H_NFSR_TAP"} | {"H_NFSR_TAP": ref_grain.H_NFSR_TAP}}
    gg["vectors"] = [{"key": r.key.hex(), "iv": r.iv.hex(), "ks": r.ks.hex(), "bit_order": r.bit_order}
                     for r in ref_vectors.GRAIN_VECTORS]
    assert ref_vectors.verify_vectors("grain") == (len(ref_vectors.GRAIN_VECTORS), [])
    R = random.Random(0x6A)
    sc = []
    for _ in range(6):
        m = ref_grain.GrainKeyIv(R.randbytes(10), R.randbytes(8))
        a = ref_grain.GrainScalar.from_key_iv(m)
        p = ref_grain.GrainScalarPacked.from_key_iv(m)
        assert bits_int(a.b) == p.b and bits_int(a.s) == p.s
        b0, s0 = p.b, p.s                                             # post-init state, before any keystream
        ks = a.keystream_bytes(128)
        assert ks == p.keystream_bytes(128)
        sc.append({"key": m.key.hex(), "iv": m.iv.hex(), "post_init_b": f"{b0:x}", "post_init_s": f"{s0:x}",
                   "ks128_msb": ks.hex(), "ks64_lsb": ref_grain.GrainScalar.from_key_iv(m).keystream_bytes(64, "lsb").hex()})
    gg["scalar_cases"] = sc
    R = random.Random(0xFA57)
    _ = [R.randbytes(14) for _ in range(64)]                      # skip what test_kernels.py draws for MICKEY
    gm = [ref_grain.GrainKeyIv(R.randbytes(10), R.randbytes(8)) for _ in range(64)]
    gcases = []
    for name, mats, nclk, width in (("w32_7lanes_443", gm[:7], 443, 32), ("w64_64lanes_443", gm, 443, 64),
                                    ("w32_32lanes_200", gm[:32], 200, 32), ("w64_40lanes_97", gm[:40], 97, 64)):
        words = ref_kernels.grain_sliced_words(mats, nclk, width)
        pure = ref_grain.GrainSliced.from_key_ivs(mats, width)
        st = {"b": [f"{w:x}" for w in pure.b], "s": [f"{w:x}" for w in pure.s]}
        assert [int(w) for w in words] == pure.keystream_words(nclk)
        gcases.append({"name": name, "width": width, "nclocks": nclk, "init_state": st,
                       "materials": [{"key": m.key.hex(), "iv": m.iv.hex()} for m in mats],
                       "words_hex": words.astype("<u8").tobytes().hex()})
    gg["sliced_cases"] = gcases
    words = ref_kernels.grain_sliced_words(gm, 100_000, 64)
    gg["long"] = {"nclocks": 100_000, "words_u8_sha256": sha(words.astype("<u8").tobytes()),
                  "lane_major_msb_sha256": sha(ref_kernels.words_lane_major_bytes(words, 64)),
                  "lane_major_lsb_sha256": sha(ref_kernels.words_lane_major_bytes(words, 64, "lsb"))}
    g["grain"] = gg

    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_text(json.dumps(g, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
