"""CPU-only checks of the host mirror and the C-ABI library (no compute calls)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1909_04750_b200 as pkg
from paper_1909_04750_b200 import _native, kernels, mickey, sharding
from paper_1909_04750_b200.mickey import MickeyKeyIv, MickeyKeyIvError

ROOT = Path(__file__).resolve().parents[1]


def test_library_loads_and_exports_every_declared_symbol():
    header = (ROOT / "include" / "mk2.h").read_text()
    declared = set(re.findall(r"\b(mk2_[a-z0-9_]+)\s*\(", header))
    declared.discard("mk2_ctx")
    assert declared, "no declarations parsed from include/mk2.h"
    L = C.CDLL(str(_native.library_path()))
    for name in sorted(declared):
        assert hasattr(L, name), f"libmk2.so does not export {name}"
    assert declared == set(_native.SYMBOLS), "ctypes table out of sync with include/mk2.h"
    assert _native.lib().mk2_abi_version() == _native.ABI_VERSION == 2
    assert _native.lib().mk2_lop3_per_clock() == 327


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pkg.Mk2Error, match="no CPU fallback"):
        pkg.MickeyGenerator(0)
    with pytest.raises(pkg.Mk2Error):
        pkg.mickey_sliced_words([MickeyKeyIv(bytes(10), b"")], 8)


def test_c_abi_from_plain_c_fails_loudly_without_device(c_abi_consumer):
    """A C program that includes only include/mk2.h links against libmk2.so; without an sm_100 device mk2_create
    returns MK2_E_NODEVICE with a message (exit code 3 of tests/c/abi_consumer.c) -- no crash, no CPU path."""
    import subprocess

    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_c_abi_from_plain_c in the GPU suite")
    res = subprocess.run([str(c_abi_consumer)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 3, (res.returncode, res.stdout, res.stderr)
    assert "no CPU fallback" in res.stderr


def test_product_package_never_imports_oracle():
    for path in (ROOT / "paper_1909_04750_b200").rglob("*.py"):
        text = path.read_text()
        assert "import oracle" not in text and "from oracle" not in text, path
    for path in (ROOT / "paper_1909_04750_b200" / "csrc").glob("*.cu*"):
        assert "oracle" not in path.read_text(), path


def test_constants_structure(golden):
    c = mickey.mickey_constants()
    assert len(c["RTAPS"]) == 50
    assert list(c["RTAPS"]) == golden["tables"]["RTAPS"]
    for name in ("COMP0", "COMP1", "FB0", "FB1"):
        assert list(c[name]) == golden["tables"][name]
    assert mickey.COMP0[0] == mickey.COMP0[99] == mickey.COMP1[0] == mickey.COMP1[99] == 0


def test_cuda_tables_match_python_tables():
    src = (ROOT / "paper_1909_04750_b200" / "csrc" / "mk2_clock.cuh").read_text()
    words = [int(x, 16) for x in re.findall(r"case \d+: return (0x[0-9A-Fa-f]+)u;", src)]
    assert len(words) == 20
    expect = mickey._R_MASK_WORDS + mickey._COMP0_WORDS + mickey._COMP1_WORDS + mickey._FB0_WORDS + mickey._FB1_WORDS
    assert tuple(words) == expect


def test_keyiv_validation():
    # tests/test_mickey.py:93-99
    with pytest.raises(MickeyKeyIvError):
        MickeyKeyIv(bytes(10), bytes(11))
    with pytest.raises(MickeyKeyIvError):
        MickeyKeyIv(bytes(10), [0] * 81)
    with pytest.raises(MickeyKeyIvError):
        MickeyKeyIv(bytes(9), b"")
    with pytest.raises(MickeyKeyIvError):
        MickeyKeyIv(bytes(10), [0, 2, 1])
    m = MickeyKeyIv(bytes(range(10)), b"\xa5")
    assert m.iv_bits() == [1, 0, 1, 0, 0, 1, 0, 1]
    assert m.key_bits()[:16] == [0] * 8 + [0, 0, 0, 0, 0, 0, 0, 1]
    assert isinstance(MickeyKeyIvError("x"), ValueError)


def test_pack_materials_errors_name_the_lane():
    # tests/test_mickey.py:140-145
    bad = type("Bad", (), {"iv_bits": lambda self: [0] * 81, "key_bits": lambda self: [0] * 80})()
    mats = [MickeyKeyIv(bytes(10), b"")] * 3 + [bad]
    with pytest.raises(MickeyKeyIvError, match="lane 3"):
        mickey.pack_materials(mats, 32)
    with pytest.raises(MickeyKeyIvError, match="at least one lane"):
        mickey.pack_materials([], 32)
    with pytest.raises(MickeyKeyIvError, match="exceed width"):
        mickey.pack_materials([MickeyKeyIv(bytes(10))] * 33, 32)
    with pytest.raises(ValueError, match="lane width"):
        mickey.MickeySliced.from_key_ivs([MickeyKeyIv(bytes(10))], width=48)


def test_pack_materials_layout():
    mats = [MickeyKeyIv(bytes(range(10)), b"\x80\x01"), MickeyKeyIv(bytes(10), [1, 0, 1])]
    keys, ivs, nbits, uniform = mickey.pack_materials(mats, 32)
    assert not uniform
    assert keys[0].tobytes() == bytes(range(10))
    assert ivs[0, :2].tobytes() == b"\x80\x01" and ivs[1, 0] == 0b10100000
    assert nbits[:2].tolist() == [16, 3] and set(nbits[2:].tolist()) == {_native.MK2_IV_UNUSED}
    keys, ivs, nbits, uniform = mickey.pack_materials([mats[0]] * 5, 64)
    assert uniform and set(nbits.tolist()) == {16} and not keys[5:].any()


def test_lane_helpers(golden):
    # tests/test_kernels.py:75-82
    h = golden["lane_helpers"]
    w = np.array(h["words"], dtype=np.uint64)
    assert kernels.words_to_lane_bits(w, 0).tolist() == h["lane0_bits"]
    assert kernels.words_to_lane_bits(w, 1).tolist() == h["lane1_bits"]
    assert kernels.words_to_lane_bytes(w, 0).hex() == h["lane0_msb"]
    assert kernels.words_to_lane_bytes(w, 0, "lsb").hex() == h["lane0_lsb"]
    assert kernels.words_lane_major_bytes(w, 2).hex() == h["lane_major_2"]
    with pytest.raises(ValueError):
        kernels.words_to_lane_bytes(w, 0, "middle")


def test_shard_partition_properties():
    for n in (0, 1, 31, 32, 33, 1000, 1 << 20, (1 << 20) + 17):
        for world in (1, 2, 3, 4, 8):
            shards = [sharding.shard_instances(n, world, r) for r in range(world)]
            assert sum(s.count for s in shards) == n
            pos = 0
            for s in shards:
                assert s.first == pos or s.count == 0
                assert s.first % 32 == 0 or s.count == 0
                assert s.group_offset * 32 == s.first or s.count == 0
                pos += s.count
            sizes = [s.groups for s in shards]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.shard_instances(10, 2, 2)


def test_checksum_i64_roundtrip():
    for u in (0, 1, (1 << 63) - 1, 1 << 63, (1 << 64) - 1, 0xDB93F1AC2EF9D52E):
        assert sharding.from_i64(sharding.to_i64(u)) == u
    assert sharding.allreduce_checksum(0xDB93F1AC2EF9D52E) == 0xDB93F1AC2EF9D52E


def test_master_seed_validation():
    # seedgen.py:45-54
    from paper_1909_04750_b200.seedgen import MasterSeed, SeedError

    with pytest.raises(SeedError):
        MasterSeed(bytes(31))
    with pytest.raises(SeedError):
        MasterSeed(bytes(32))
    with pytest.raises(SeedError):
        MasterSeed(bytes(range(32)), "rc4")
    with pytest.raises(SeedError):
        MasterSeed(bytes(range(32)), "grain")
    with pytest.raises(SeedError):
        MasterSeed(bytes(range(32)), "mickey", 0)
    assert isinstance(SeedError("x"), ValueError)
    assert MasterSeed(bytes(range(32)), "mickey", 1 << 20).lanes == 1 << 20


def test_grain_host_mirror(golden):
    from paper_1909_04750_b200 import grain

    c = grain.grain_constants()
    ref = golden["grain"]["constants"]
    for name in ("LFSR_TAPS", "NFSR_LINEAR_TAPS", "H_LFSR_TAPS", "OUTPUT_TAPS"):
        assert list(c[name]) == ref[name]
    assert [list(t) for t in c["NFSR_PRODUCT_TAPS"]] == ref["NFSR_PRODUCT_TAPS"] and c["H_NFSR_TAP"] == ref["H_NFSR_TAP"]
    with pytest.raises(grain.GrainKeyIvError):
        grain.GrainKeyIv(bytes(9), bytes(8))
    with pytest.raises(grain.GrainKeyIvError):
        grain.GrainKeyIv(bytes(10), bytes(7))
    m = grain.GrainKeyIv(bytes([0x01] + [0] * 9), bytes([0x80] + [0] * 7))
    assert m.key_bits()[:8] == [1, 0, 0, 0, 0, 0, 0, 0] and m.iv_bits()[:8] == [0, 0, 0, 0, 0, 0, 0, 1]  # LSB-first
    with pytest.raises(grain.GrainKeyIvError, match="at least one lane"):
        grain.pack_materials([], 32)
    with pytest.raises(grain.GrainKeyIvError, match="exceed width"):
        grain.pack_materials([m] * 33, 32)
    src = (ROOT / "paper_1909_04750_b200" / "csrc" / "mk2_grain.cuh").read_text()
    for term in grain.NFSR_LINEAR_TAPS:
        assert f"b[ix({term})]" in src   # ix(i) = window offset (or circular index) of bit i


def test_bench_reference_arm_prints_one_json_line():
    """bench.py --impl reference (the CPU arm the driver runs beside the GPU arm): stdout carries exactly one JSON
    line with the contract's keys, whatever the libraries underneath print; `--cpu-kind port` = the oracle's C port
    (the one place outside tests/ and smoke() that may execute oracle/), so it runs without the staged reference."""
    import json
    import subprocess
    import sys

    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--cpu-kind", "port", "--steps", "1",
                          "--warmup", "0", "--cpu-seconds", "1"], capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "Tb/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "Tb/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["metric"] == "keystream Tb/s, bitsliced MICKEY 2.0" and d["config"]["workload"].startswith("c2")
