#!/usr/bin/env python
"""bench.py -- keystream Tb/s of the bitsliced MICKEY 2.0 path on N B200s.

    python bench.py --gpus N --steps K --warmup W            (our CUDA path)
    python bench.py --impl reference --gpus N --steps K ...  (CPU arm: oracle port)

A step = one pass of the hot path over one batch of synthetic key/IV material:
device-side counter-IV synthesis, key/IV load + 100 pre-clocks, the keystream
loop and the stores.  Default workload = BASELINE.json configs[1]:
2^20 instances x 1 Mbit per GPU, column-major output resident in HBM (131 GB,
>> L2, so no L2 flush is needed between steps).  With N > 1 every rank takes a
disjoint key/IV (instance-index) range of the same size: weak scaling, no
data-path collective; one 8-byte checksum all-reduce after the timed region.

Prints ONE JSON line on rank 0 (see DESIGN.md "Measurement" for every field).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

KEY = bytes.fromhex("123456789abcdef01234")  # eSTREAM vector key (vectors.py:42)
METRIC = "keystream Tb/s, bitsliced MICKEY 2.0"
LOP3_PER_CLOCK_SURVEY = 327  # LOP3 per clock per 32-lane word, one clock at a time
# dram__bytes_read.sum + dram__bytes_write.sum of ONE launch of the dominant kernel, from the committed
# `ncu --set full` captures (per launch, like roofline.achieved); only for launches captured exactly.
NCU_TRAFFIC = {
    # (layout, instances, clocks): (bytes, source)
    ("colmajor", 1 << 20, 1_000_000): (131_438_553_000 + 512_053_248, "profiles/r01b_ncu_gen_colmajor_c2_full_1Mclk.txt"),
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("c2", "c3", "c5"), default="c2",
                    help="c2: 2^20 x 1 Mbit column-major (default, BASELINE configs[1]); "
                         "c3: 2^24 x 64 Kbit row-major; c5: 2^26 x 1 Kbit init-dominated")
    ap.add_argument("--instances-log2", type=int, default=None, help="override instances per GPU (log2)")
    ap.add_argument("--clocks", type=int, default=None, help="override keystream bits per instance")
    ap.add_argument("--e2e-clocks", type=int, default=16384, help="keystream bits per instance of one e2e step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-curand", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target size of the CPU sample")
    return ap.parse_args()


WORKLOADS = {  # name -> (instances log2, clocks, layout)
    "c2": (20, 1_000_000, "colmajor"),
    "c3": (24, 65_536, "rowmajor"),
    "c5": (26, 1_024, "rowmajor"),
}


def workload_of(args):
    lg, clocks, layout = WORKLOADS[args.workload]
    if args.instances_log2 is not None:
        lg = args.instances_log2
    if args.clocks is not None:
        clocks = args.clocks
    return 1 << lg, clocks, layout


# ----------------------------------------------------------------------------- clocks sampler

class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), line.strip()))

    def stop(self, t0: float, t1: float) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        rows = [r for t, r in self.rows if t0 <= t <= t1] or [r for _, r in self.rows]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1])); pw.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- CPU arm

def cpu_sample(seconds: float, threads: int | None = None) -> dict:
    """Time the oracle's port of the reference's compiled keystream loop
    (kernels._mickey_sliced_loop via bench._timed_run, bench.py:169-183): W=64,
    loop only, one independent generator per host thread (bench.py:265-282)."""
    from oracle import mickey_oracle as orc

    cores = threads or orc.max_threads()
    nclocks = 1 << 20
    t1 = orc.timed_loops(nclocks, cores, 1)                      # also the warm-up
    ncalls = max(1, min(4096, int(seconds / max(t1, 1e-3))))
    dt = orc.timed_loops(nclocks, cores, ncalls)
    bits = cores * 64 * nclocks * ncalls
    # the reference's protocol also quotes one worker (bench.measure(..., workers=1)) and the bit-per-cell
    # "naive" engine for its speed-up claim: both from the same C port
    t_one = orc.timed_loops(nclocks, 1, 4)
    st = orc.Scalar.from_key_iv(KEY, b"\x21\x43\x65\x87")
    t0 = time.perf_counter()
    st.keystream_bytes(1 << 16)
    t_naive = time.perf_counter() - t0
    return {"value": bits / dt / 1e12, "unit": "Tb/s", "cores": cores, "kind": "port",
            "seconds": round(dt, 3),
            "one_thread_gbit_s": 64 * nclocks * 4 / t_one / 1e9,
            "naive_one_thread_gbit_s": (1 << 19) / t_naive / 1e9,
            "sample": f"{cores} threads x 64 lanes x {nclocks} clocks x {ncalls} calls, keystream loop only "
                      f"(oracle/mickey_oracle.c port of kernels.py:46-95, gcc -O3 -march=x86-64-v3)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n, clocks, layout = workload_of(args)
    per_step = max(2.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(min(per_step, 2.0))
    vals = [cpu_sample(per_step) for _ in range(args.steps)]
    dt = sum(v["seconds"] for v in vals)
    bits = sum(v["value"] * 1e12 * v["seconds"] for v in vals)
    value = bits / dt / 1e12
    last = vals[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Tb/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: 2^{n.bit_length() - 1} instances x {clocks} bits per GPU, {layout} "
                               f"(CPU arm: bounded sample of the same keystream loop)"},
        "cpu_baseline": {**{k: last[k] for k in ("unit", "cores", "kind", "sample", "one_thread_gbit_s", "naive_one_thread_gbit_s")}, "value": value},
        "e2e": {"value": value, "unit": "Tb/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except ValueError:
            pass
    return {"hbm_gbs": 6650.0}, "fallback"


def curand_compare(torch, nbytes: int) -> dict:
    import ctypes as C

    from paper_1909_04750_b200 import build

    L = C.CDLL(str(build.build_curand()))
    L.mk2_curand_time.restype = C.c_float
    L.mk2_curand_time.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_int]
    buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {"bytes": nbytes, "unit": "Tb/s"}
    for kind, kname in ((0, "xorwow"), (1, "philox4_32_10")):
        for api, aname in ((0, "host_api"), (1, "device_api")):
            ms = L.mk2_curand_time(kind, api, buf.data_ptr(), nbytes, 3)
            out[f"{kname}_{aname}"] = (nbytes * 8 / (ms * 1e-3) / 1e12) if ms > 0 else None
    del buf
    return out


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1909_04750_b200 as pkg
    from paper_1909_04750_b200 import sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the MICKEY path has no CPU fallback")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n, clocks, layout = workload_of(args)
    G = n // 32
    first = rank * n                       # disjoint key/IV (instance index) range per rank
    stream = torch.cuda.current_stream()
    gen = pkg.MickeyGenerator(local)
    gen.set_stream(stream.cuda_stream)
    gen.set_async(True)                    # we time the stream ourselves
    gen.set_group_offset(first // 32)

    # ---- output buffer: whole keystream of one step resident in HBM when it fits
    out_bytes = n * clocks // 8
    free, _total = torch.cuda.mem_get_info()
    state_bytes = G * (800 + 8 + 640) + (1 << 30)
    if out_bytes + state_bytes <= free:
        chunk_clocks, out_mode = clocks, "full"
    else:
        budget = max(1 << 28, int(free * 0.5) - state_bytes)
        chunk_clocks = max(1024, budget * 8 // n // 1024 * 1024)
        out_mode = f"ring({chunk_clocks} clocks)"
    if layout == "colmajor":
        out = torch.empty((chunk_clocks, G), dtype=torch.int32, device=dev)
    else:
        out = torch.empty((n, chunk_clocks // 8), dtype=torch.uint8, device=dev)

    ev = lambda: torch.cuda.Event(enable_timing=True)
    gen_events = []
    launches = 0

    # c5 (fresh key/IV pairs, init-dominated): explicit material arrays resident in HBM, so that the row-major
    # key/IV bytes -> bitsliced input words transposition is part of the step; c2 / c3: the
    # counter-IV set synthesised on device
    explicit = args.workload == "c5"
    if explicit:
        gsrc = torch.Generator(device=dev).manual_seed(0x190904750 + rank)
        d_keys = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device=dev, generator=gsrc)
        d_ivs = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device=dev, generator=gsrc)

    def step(i: int, record: bool):
        nonlocal launches
        if explicit:
            gen.init_material(d_keys, d_ivs, 80)
        else:
            gen.init_counter(KEY, first + (i % 4) * world * n, n)
        launches += gen.last_kernel_launches
        done = 0
        while done < clocks:
            tc = min(chunk_clocks, clocks - done)
            e0, e1 = ev(), ev()
            e0.record(stream)
            if layout == "colmajor":
                gen.generate_colmajor(tc, out)
            else:
                gen.generate_rowmajor(tc, out)
            e1.record(stream)
            launches += gen.last_kernel_launches
            if record:
                gen_events.append((e0, e1, tc))
            done += tc

    for i in range(args.warmup):
        step(i, False)
    barrier()
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
        time.sleep(0.25)
    launches = 0
    t_wall0 = time.perf_counter()
    start, end = ev(), ev()
    barrier()
    start.record(stream)
    for i in range(args.steps):
        step(args.warmup + i, True)
    end.record(stream)
    barrier()
    t_wall1 = time.perf_counter()
    clocks_info = sampler.stop(t_wall0, t_wall1) if rank == 0 else None
    elapsed_ms = max_over_ranks(start.elapsed_time(end))
    gen_ms = [e0.elapsed_time(e1) for e0, e1, _ in gen_events]
    gen_clk = sum(tc for _, _, tc in gen_events)
    kernel_ms_total = sum(gen_ms)
    timed_launches = launches

    bits_per_step = world * n * clocks
    value = bits_per_step * args.steps / (elapsed_ms * 1e-3) / 1e12

    # ---- checksum: the only exchange (8 bytes, NCCL sum), outside the timed region
    csum = sharding.allreduce_checksum(gen.checksum(), device=dev)

    # ---- roofline of the dominant kernel (keystream loop), this rank
    peaks, peaks_src = measured_peaks()
    gen.set_async(False)
    lop3_peak, _ = gen.lop3_peak()
    # Algorithmic LOP3 per clock of the kernel as built: the clock runs in blocks of K clocks with R's
    # reduction deferred (csrc/mk2_clock.cuh); mk2_lop3_per_block is derived from the cipher's tables and
    # checked against the SASS by tests/test_structure.py.  SURVEY.md 8(d) counted 327 for the one-clock form.
    which = 0 if layout == "colmajor" else 1
    from paper_1909_04750_b200 import _native
    lib = _native.lib()
    rblock, per_block = lib.mk2_rblock(which), lib.mk2_lop3_per_block(which)
    lop3_per_clock = per_block / rblock
    lane_ops = n * gen_clk * lop3_per_clock / 32          # algorithmic LOP3 lane-ops in the timed launches
    achieved = lane_ops / (kernel_ms_total * 1e-3)
    achieved_survey = achieved * LOP3_PER_CLOCK_SURVEY / lop3_per_clock
    hbm_gbs = (n * gen_clk / 8) / (kernel_ms_total * 1e-3) / 1e9
    roofline = {
        "bound": "lop3", "kernel": "gen_colmajor_kernel" if layout == "colmajor" else "tmem::gen_rowmajor_kernel",
        "achieved": achieved / 1e12, "peak": lop3_peak / 1e12, "unit": "Tlane-op/s", "frac": achieved / lop3_peak,
        "peak_source": "measured live by mk2_lop3_peak (dependency-free LOP3 kernel) on this GPU",
        "algorithmic_ops_per_launch": lane_ops / max(1, len(gen_events)),
        "lop3_per_clock": {"executed": lop3_per_clock, "block_clocks": rblock, "lop3_per_block": per_block,
                           "survey_one_clock_form": LOP3_PER_CLOCK_SURVEY},
        "at_survey_count": {"achieved": achieved_survey / 1e12, "frac": achieved_survey / lop3_peak,
                            "note": "same run priced at SURVEY 8(d)'s 327 LOP3 per clock: above 1 because the "
                                    "deferred R reduction executes fewer LOP3 than the one-clock form"},
        "avg_launch_ms": kernel_ms_total / max(1, len(gen_events)),
        "kernel_share_of_step": kernel_ms_total / start.elapsed_time(end),
        "traffic": NCU_TRAFFIC.get((layout, n, gen_events[0][2] if gen_events else 0), (None, None))[0],
        "traffic_source": NCU_TRAFFIC.get((layout, n, gen_events[0][2] if gen_events else 0), (None, None))[1],
        "algorithmic_bytes_per_launch": n * (gen_events[0][2] if gen_events else 0) // 8,
        "hbm": {"bound": "hbm", "achieved": hbm_gbs, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": hbm_gbs / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None,
                "peak_source": f"MEASURED_PEAKS.json ({peaks_src})", "note": "0.125 B stored per keystream bit; not binding"},
    }

    # ---- e2e: host key/IV arrays in, host keystream out, through the public API
    e2e = None
    if not args.no_e2e:
        del out
        torch.cuda.empty_cache()
        e2e = run_e2e(args, torch, np, pkg, gen, n, clocks, layout, first, world, barrier, max_over_ranks)

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Tb/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {
                "workload": f"{args.workload}: 2^{n.bit_length() - 1} instances x {clocks} bits per GPU, {layout}, "
                            + ("explicit key/IV arrays (u8[N][10] each) resident in HBM, " if explicit else
                               "counter-IV material synthesised on device, ") + "init + keystream per step",
                "instances_per_gpu": n, "clocks": clocks, "layout": layout, "output": out_mode,
                "l2": f"no flush needed: each step streams {out_bytes / 1e9:.1f} GB of output per GPU (>> 126 MB L2)",
                "parallelism": f"{world} x disjoint key/IV ranges, no data-path collective",
            },
            "roofline": roofline, "clocks": clocks_info, "gpu_launches": timed_launches,
            "checksum_u64_sum": f"{csum:#018x}",
        }
        if e2e:
            line["e2e"] = e2e
        if not args.no_curand:
            try:
                line["curand"] = curand_compare(torch, 1 << 32)
            except Exception as exc:  # comparison only; never blocks the bench line
                line["curand"] = {"error": str(exc)}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_sample(args.cpu_seconds)
    gen.close()
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    if line:
        print(json.dumps(line), flush=True)


def run_e2e(args, torch, np, pkg, gen, n, clocks, layout, first, world, barrier, max_over_ranks):
    """Same metric through the C-ABI call with HOST buffers: pinned key/IV
    arrays in (H2D inside the call), pinned keystream buffer out (D2H inside)."""
    # bounded sample of the same workload: <= 2 GiB of keystream per step (the link bounds e2e, not the kernel)
    tc = min(args.e2e_clocks, clocks // 8 * 8)
    n_full = n
    n = max(1024, min(n, (1 << 34) // tc // 1024 * 1024))
    keys = torch.from_numpy(np.tile(np.frombuffer(KEY, np.uint8), (n, 1))).pin_memory()
    idx = (np.arange(n, dtype=np.uint64) + np.uint64(first))
    ivs_np = np.zeros((n, 10), np.uint8)
    ivs_np[:, 2:] = idx.astype(">u8").view(np.uint8).reshape(n, 8)   # 80-bit big-endian index
    ivs = torch.from_numpy(ivs_np).pin_memory()
    if layout == "colmajor":
        host = torch.empty((tc, n // 32), dtype=torch.int32).pin_memory()
    else:
        host = torch.empty((n, tc // 8), dtype=torch.uint8).pin_memory()
    gen.set_stream(None)
    gen.set_async(False)

    def one():
        if layout == "colmajor":
            gen.init_material(keys, ivs, 80)
            gen.generate_colmajor(tc, host)
        else:
            gen.bulk_rowmajor(keys, ivs, 80, tc, host)   # one-shot call: upload | init + keystream | download overlap

    for _ in range(max(1, min(args.warmup, 3))):
        one()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0)
    return {
        "value": world * n * tc * args.steps / dt / 1e12, "unit": "Tb/s",
        "h2d_bytes_per_step": int(keys.numel() + ivs.numel()), "d2h_bytes_per_step": int(host.numel() * host.element_size()),
        "ms_per_step": dt / args.steps * 1e3,
        "workload": f"bounded sample of the same workload: {n} of {n_full} instances x {tc} bits per GPU per call: "
                    + ("mk2_init_from_material(pinned host keys, IVs) + mk2_generate_colmajor(pinned host out); "
                       if layout == "colmajor" else
                       "mk2_bulk_rowmajor(pinned host keys, IVs -> pinned host out), instance blocks pipelined; ")
                    + "the host link, not the kernel, bounds it",
    }


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
