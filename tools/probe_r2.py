"""Round-2 measurements on the B200 (run under gpurun): ragged-IV init against the uniform init, small-call
latency of the reference-shaped API with and without the context pool, pinned / pageable host-output rates."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1909_04750_b200 as pkg  # noqa: E402
from paper_1909_04750_b200 import hostmem  # noqa: E402

out = {}


def best(fn, reps=5):
    v = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        v.append(time.perf_counter() - t0)
    return min(v), sorted(v)[len(v) // 2]


def ragged():
    import torch
    N = 1 << 20
    rng = np.random.default_rng(1)
    keys = torch.from_numpy(rng.integers(0, 256, (N, 10), dtype=np.uint8)).cuda()
    ivs = torch.from_numpy(rng.integers(0, 256, (N, 10), dtype=np.uint8)).cuda()
    nb_bytes = torch.from_numpy((8 * rng.integers(0, 11, N)).astype(np.uint8)).cuda()
    nb_bits = torch.from_numpy(rng.integers(0, 81, N).astype(np.uint8)).cuda()
    res = {}
    with pkg.MickeyGenerator(0) as gen:
        def ms(fn):
            vals = []
            for _ in range(6):
                fn()
                vals.append(gen.last_kernel_ms)
            return min(vals[1:])
        res["uniform_80bit_ms"] = ms(lambda: gen.init_material(keys, ivs, 80))
        res["uniform_40bit_ms"] = ms(lambda: gen.init_material(keys, ivs, 40))
        res["ragged_bytes_0_10_ms"] = ms(lambda: gen.init_ragged(keys, ivs, nb_bytes))
        res["ragged_bits_0_80_ms"] = ms(lambda: gen.init_ragged(keys, ivs, nb_bits))
    res["ragged_over_uniform80"] = res["ragged_bytes_0_10_ms"] / res["uniform_80bit_ms"]
    res["note"] = "2^20 lanes, device-resident material, pack + init kernels (mk2_last_kernel_ms); ragged includes the D2H of the length array"
    out["ragged_init"] = res


def latency():
    key, iv = bytes.fromhex("123456789abcdef01234"), bytes.fromhex("21436587")
    mats = [pkg.MickeyKeyIv(key, iv)] * 64
    keys, ivs, nbits, _ = pkg.mickey.pack_materials(mats, 64)
    res = {}
    pkg.mickey_sliced_words(mats, 4096)
    b, med = best(lambda: pkg.mickey_sliced_words(mats, 4096), 30)
    res["mickey_sliced_words_64x4096_pooled_us"] = {"best": b * 1e6, "median": med * 1e6}

    def fresh():
        hostmem.drop_idle_contexts()
        pkg.mickey_sliced_words(mats, 4096)
    b, med = best(fresh, 10)
    res["mickey_sliced_words_64x4096_new_context_per_call_us"] = {"best": b * 1e6, "median": med * 1e6}
    t0 = time.perf_counter()
    for _ in range(20):
        pkg.mickey.pack_materials(mats, 64)
    res["python_pack_materials_us"] = (time.perf_counter() - t0) / 20 * 1e6
    with pkg.MickeyGenerator(0) as gen:
        gen.init_material(keys, ivs, 32).generate_colmajor(4096)
        kms = []
        tot = []
        for _ in range(30):
            t0 = time.perf_counter()
            gen.init_material(keys, ivs, 32)
            k = gen.last_kernel_ms
            gen.generate_colmajor(4096)
            k += gen.last_kernel_ms
            tot.append(time.perf_counter() - t0)
            kms.append(k)
        res["abi_init_plus_generate_us"] = {"wall_best": min(tot) * 1e6, "kernel_best": min(kms) * 1e3}
    res["overhead_over_kernel_us"] = res["mickey_sliced_words_64x4096_pooled_us"]["best"] - res["abi_init_plus_generate_us"]["kernel_best"]
    out["small_call_latency"] = res


def hostbuf():
    import torch
    N, T = 1 << 20, 16384
    key = bytes.fromhex("123456789abcdef01234")
    res = {}
    with pkg.MickeyGenerator(0) as gen:
        gen.init_counter(key, 0, N)
        pinned_c = torch.empty((T, N // 32), dtype=torch.int32).pin_memory()
        gen.generate_colmajor(T, pinned_c)
        b, _ = best(lambda: gen.generate_colmajor(T, pinned_c), 4)
        res["col_pinned_GBps"] = N * T / 8 / b / 1e9
        page = np.empty((T, N // 32), np.uint32)
        for th in (0, 2, 4, 8, 16):
            gen.set_host_threads(th)
            gen.generate_colmajor(T, page)
            b, _ = best(lambda: gen.generate_colmajor(T, page), 3)
            res[f"col_pageable_touched_threads{th}_GBps"] = N * T / 8 / b / 1e9
        gen.set_host_threads(0)
        vals = []
        for _ in range(3):
            fresh = np.empty((T, N // 32), np.uint32)          # untouched pages: first-touch faults inside the call
            t0 = time.perf_counter()
            gen.generate_colmajor(T, fresh)
            vals.append(time.perf_counter() - t0)
            del fresh
        res["col_pageable_fresh_GBps"] = N * T / 8 / min(vals) / 1e9
        vals = []
        for _ in range(4):
            t0 = time.perf_counter()
            arr = gen.generate_colmajor(T)                      # pool-backed fresh result array
            vals.append(time.perf_counter() - t0)
            del arr
        res["col_pool_array_GBps"] = {"first_call": N * T / 8 / vals[0] / 1e9, "steady": N * T / 8 / min(vals[1:]) / 1e9}
        # row-major one-shot
        keys = np.tile(np.frombuffer(key, np.uint8), (N, 1))
        ivs = np.zeros((N, 10), np.uint8)
        ivs[:, 2:] = np.arange(N, dtype=np.uint64).astype(">u8").view(np.uint8).reshape(N, 8)
        pinned_r = torch.empty((N, T // 8), dtype=torch.uint8).pin_memory()
        gen.bulk_rowmajor(keys, ivs, 80, T, pinned_r)
        b, _ = best(lambda: gen.bulk_rowmajor(keys, ivs, 80, T, pinned_r), 3)
        res["row_bulk_pinned_GBps"] = N * T / 8 / b / 1e9
        page_r = np.empty((N, T // 8), np.uint8)
        gen.bulk_rowmajor(keys, ivs, 80, T, page_r)
        b, _ = best(lambda: gen.bulk_rowmajor(keys, ivs, 80, T, page_r), 3)
        res["row_bulk_pageable_touched_GBps"] = N * T / 8 / b / 1e9
    import os
    res["host_cpus"] = os.cpu_count()
    out["host_buffers_2GiB"] = res


def e2e():
    """bench.py's e2e_pageable leg in isolation: pageable key/IV arrays in + one 2 GiB pageable output per step,
    by number of copy lanes; the pinned variant of the same step for comparison."""
    import torch
    N, T = 1 << 20, 16384
    key = bytes.fromhex("123456789abcdef01234")
    keys = np.tile(np.frombuffer(key, np.uint8), (N, 1))
    ivs = np.zeros((N, 10), np.uint8)
    ivs[:, 2:] = np.arange(N, dtype=np.uint64).astype(">u8").view(np.uint8).reshape(N, 8)
    res = {}
    with pkg.MickeyGenerator(0) as gen:
        pk, pi = torch.from_numpy(keys).pin_memory(), torch.from_numpy(ivs).pin_memory()
        pinned = torch.empty((T, N // 32), dtype=torch.int32).pin_memory()
        step = lambda: (gen.init_material(pk, pi, 80), gen.generate_colmajor(T, pinned))
        step()
        res["pinned_ms"] = best(step, 4)[0] * 1e3
        page = np.empty((T, N // 32), np.uint32)
        for th in (0, 8, 0, 8, 6, 16):
            gen.set_host_threads(th)
            step = lambda: (gen.init_material(keys, ivs, 80), gen.generate_colmajor(T, page))
            step()
            b, med = best(step, 5)
            res[f"pageable_lanes{th}_ms"] = {"best": b * 1e3, "median": med * 1e3}
        gen.set_host_threads(0)
        t0 = time.perf_counter()
        gen.init_material(keys, ivs, 80)
        res["init_from_pageable_inputs_ms"] = (time.perf_counter() - t0) * 1e3
    out["e2e_pageable_leg"] = res


for name, fn in (("ragged", ragged), ("latency", latency), ("hostbuf", hostbuf), ("e2e", e2e)):
    if len(sys.argv) < 2 or name in sys.argv[1:]:
        try:
            fn()
        except Exception as exc:  # keep the other sections
            out[name + "_error"] = repr(exc)
print(json.dumps(out, indent=1))
