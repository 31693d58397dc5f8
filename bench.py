#!/usr/bin/env python
"""bench.py -- keystream Tb/s of the bitsliced MICKEY 2.0 path on N B200s.

    python bench.py --gpus N --steps K --warmup W            (our CUDA path)
    python bench.py --impl reference --gpus N --steps K ...  (CPU arm: the reference's numba loop, else the oracle port)

A step = one pass of the hot path over one batch of synthetic key/IV material:
device-side counter-IV synthesis (or explicit key/IV arrays), key/IV load + 100
pre-clocks, the keystream loop and the stores.  Headline workload = BASELINE.json
configs[1] ("c2"): 2^20 instances x 1 Mbit per GPU, column-major output resident
in HBM (131 GB, >> L2, so no L2 flush is needed between steps).  The same run
also measures configs[2] ("c3", 2^24 x 64 Kbit row-major) and configs[4] ("c5",
2^26 fresh key/IV pairs x 1 Kbit) as `extra_workloads`, each with its own
roofline record, and the host-buffer legs `e2e` (pinned) and `e2e_pageable`.

Multi-GPU (one process per GPU under torchrun): `--scaling weak` gives every rank
its own disjoint key/IV range of the workload's size; `--scaling strong
--total-bits B` splits B bits (configs[3]: 8e12 = 1 TB) over the ranks.  No
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
# dram__bytes_read.sum + dram__bytes_write.sum of ONE launch of the dominant kernel from the committed
# `ncu --set full` captures.  NOT measured in this run: quoted (with its source file) only for a launch of exactly
# this geometry, next to `traffic_model`, which IS computed in the run from the launch plan.
NCU_TRAFFIC = {
    # (layout, instances, clocks): (bytes, source)
    ("colmajor", 1 << 20, 1_000_000): (131_438_553_000 + 512_053_248, "profiles/r01b_ncu_gen_colmajor_c2_full_1Mclk.txt"),
}
try:  # captures added later in the round register themselves here (profiles/ncu_traffic.json)
    for _k, _v in json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text()).items():
        _layout, _n, _t = _k.split(":")
        NCU_TRAFFIC[(_layout, int(_n), int(_t))] = (int(_v["bytes"]), _v["source"])
except (OSError, ValueError, KeyError):
    pass

WORKLOADS = {  # name -> (instances log2, clocks, layout, BASELINE.json config index)
    "c2": (20, 1_000_000, "colmajor", 1),
    "c3": (24, 65_536, "rowmajor", 2),
    "c5": (26, 1_024, "rowmajor", 4),
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="c2",
                    help="headline workload: c2 2^20 x 1 Mbit column-major (default, BASELINE configs[1]); "
                         "c3 2^24 x 64 Kbit row-major; c5 2^26 x 1 Kbit init-dominated")
    ap.add_argument("--extras", default="auto",
                    help="other single-GPU configs measured in the same run as extra_workloads: 'auto' (the other two "
                         "at N=1 with the default workload), 'none', or a comma list of c2,c3,c5")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="process-group backend for N > 1.  nccl (default): one GPU per rank.  gloo: a debug mode that lets "
                         "several ranks share the GPUs there are (rank r drives cuda:(r mod device count)); the collectives "
                         "then carry CPU tensors.  It exists so that the whole N > 1 code path of this file runs on a "
                         "one-GPU box (tests/test_gpu_parity.py); its throughput is not a multi-GPU figure.")
    ap.add_argument("--total-bits", type=float, default=8e12,
                    help="strong scaling: keystream bits of the whole job (BASELINE configs[3]: 1 TB = 8e12)")
    ap.add_argument("--instances-log2", type=int, default=None, help="override instances per GPU (log2)")
    ap.add_argument("--clocks", type=int, default=None, help="override keystream bits per instance")
    ap.add_argument("--e2e-clocks", type=int, default=16384, help="keystream bits per instance of one host-output call")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-curand", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-ncu-traffic", action="store_true",
                    help="do not measure roofline.traffic live (one launch of each workload under ncu in a child process)")
    ap.add_argument("--traffic-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target size of the CPU sample")
    ap.add_argument("--cpu-kind", choices=("auto", "reference", "port"), default="auto",
                    help="--impl reference: the reference's own numba loop from oracle/_ref (auto: when importable), "
                         "or the oracle's C port")
    return ap.parse_args()


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


def reference_import():
    """The UNMODIFIED reference package staged under oracle/_ref by oracle/stage_ref.py (git-ignored; travels to
    the GPU box with the tree).  Returns (slicerng.bench module, None) or (None, reason)."""
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "slicerng" / "bench.py").exists():
        return None, "oracle/_ref/slicerng is not staged (run python oracle/stage_ref.py where /root/reference exists)"
    cache = Path(os.environ.get("NUMBA_CACHE_DIR") or "/tmp/mk2_numba_cache")   # kernels.py:27 uses cache=True
    cache.mkdir(parents=True, exist_ok=True)
    os.environ["NUMBA_CACHE_DIR"] = str(cache)
    sys.path.insert(0, str(ref))
    try:
        import slicerng.bench as rb
        return rb, None
    except Exception as exc:  # numba missing, import error ...
        sys.path.remove(str(ref))
        return None, f"import of oracle/_ref/slicerng failed: {exc!r}"


def reference_sample(rb, workers: int, mib_per_worker: int, repeats: int = 3) -> dict:
    """One bench.measure("mickey", "sliced", ...) of the reference itself (bench.py:228-283): its numba
    _mickey_sliced_loop (kernels.py:46-95), W=64, `workers` threads (the kernels are nogil), median of repeats."""
    nbytes = workers * (mib_per_worker << 20)
    t0 = time.perf_counter()
    res = rb.measure("mickey", "sliced", nbytes=nbytes, warmup=1, repeats=max(repeats, rb.MIN_REPEATS), workers=workers)
    wall = time.perf_counter() - t0
    med = statistics.median(res.runs) if hasattr(res, "runs") else res.seconds
    return {"value": res.nbytes * 8 / med / 1e12, "unit": "Tb/s", "cores": workers, "kind": "reference",
            "seconds": round(wall, 3), "median_run_s": med, "bytes": res.nbytes,
            "sample": f"slicerng.bench.measure('mickey','sliced', nbytes={res.nbytes}, repeats={len(getattr(res, 'runs', ()))}, "
                      f"workers={workers}): the reference's own numba loop (kernels.py:46-95), W=64, median of repeats; "
                      f"with workers > 1 its timed region includes each worker's pure-Python init (bench.py:265-282)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    lg, clocks, layout, _cfg = WORKLOADS[args.workload]
    n = 1 << (args.instances_log2 or lg)
    clocks = args.clocks or clocks
    cores = os.cpu_count() or 1
    rb, why = (None, "--cpu-kind port") if args.cpu_kind == "port" else reference_import()
    if rb is None and args.cpu_kind == "reference":
        emit({"impl": "reference", "unavailable": why})
        return
    budget = 150.0  # seconds for the whole arm
    if rb is not None:
        try:
            one = reference_sample(rb, 1, 64)                              # bench.measure(..., workers=1): BASELINE.md 4
            # size the all-core sample from the one-worker rate: about budget / (steps + warmup) seconds per step
            per_step = max(4.0, min(20.0, budget / max(1, args.steps + args.warmup)))
            rate = one["bytes"] / one["median_run_s"]                      # bytes/s of one worker
            mib = int(max(8, min(256, rate * per_step / 3 / (1 << 20))))   # 3 repeats per measure()
            for _ in range(min(args.warmup, 1)):
                reference_sample(rb, cores, max(8, mib // 4))
            vals = [reference_sample(rb, cores, mib) for _ in range(args.steps)]
            extra = {"one_thread_gbit_s": one["value"] * 1e3}
            try:
                naive = rb.measure("mickey", "naive", nbytes=rb.MIN_BYTES, repeats=rb.MIN_REPEATS)
                extra["naive_one_thread_gbit_s"] = naive.nbytes * 8 / statistics.median(naive.runs) / 1e9
            except Exception:
                pass
        except Exception as exc:
            rb, why = None, f"slicerng.bench.measure failed: {exc!r}"
    if rb is None:
        per_step = max(2.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
        for _ in range(args.warmup):
            cpu_sample(min(per_step, 2.0))
        vals = [cpu_sample(per_step) for _ in range(args.steps)]
        extra = {k: vals[-1][k] for k in ("one_thread_gbit_s", "naive_one_thread_gbit_s")}
        extra["reference_unavailable"] = why
    if vals[0]["kind"] == "reference":
        # every measure() call is one step: its value is the median-of-repeats rate the reference reports
        value = statistics.median(v["value"] for v in vals)
        ms_per_step = statistics.median(v["median_run_s"] for v in vals) * 1e3
    else:
        dt = sum(v["seconds"] for v in vals)
        value = sum(v["value"] * v["seconds"] for v in vals) / dt
        ms_per_step = dt / args.steps * 1e3
    last = vals[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Tb/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: 2^{n.bit_length() - 1} instances x {clocks} bits per GPU, {layout} "
                               f"(CPU arm: bounded sample of the same keystream loop)"},
        "cpu_baseline": {"value": value, "unit": "Tb/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"], **extra},
        "e2e": {"value": value, "unit": "Tb/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line)


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


class Env:
    """Process-wide context of the GPU arm: torch, ranks, the one context (generator) of this rank."""

    def __init__(self, args):
        import numpy as np
        import torch
        import torch.distributed as dist

        import paper_1909_04750_b200 as pkg
        from paper_1909_04750_b200 import _native

        self.args, self.np, self.torch, self.dist, self.pkg = args, np, torch, dist, pkg
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if not torch.cuda.is_available():
            raise SystemExit("bench.py: no CUDA device; the MICKEY path has no CPU fallback")
        self.backend = args.dist_backend
        if self.backend == "gloo":
            self.local %= torch.cuda.device_count()
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.cdev = self.dev if self.backend == "nccl" else torch.device("cpu")   # where collective tensors live
        # Under torchrun a process group exists even at world size 1, so that a one-GPU box still executes the
        # NCCL-specific calls of the N > 1 path (init, barrier(device_ids), CUDA-tensor collectives).
        self.grouped = self.world > 1 or ("RANK" in os.environ and "MASTER_ADDR" in os.environ)
        if self.grouped:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")
        self.stream = torch.cuda.current_stream()
        self.lib = _native.lib()
        self.gen = pkg.MickeyGenerator(self.local)
        self.gen.set_stream(self.stream.cuda_stream)
        self.gen.set_async(True)               # we time the stream ourselves
        self.peaks, self.peaks_src = measured_peaks()
        self.lop3_peak = None

    def barrier(self):
        if self.grouped:
            self.torch.cuda.synchronize()
            if self.backend == "nccl":
                self.dist.barrier(device_ids=[self.local])
            else:
                self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if not self.grouped:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.cdev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather_rows(self, row):
        """One small float64/int64 row per rank -> list of rows on every rank (after the timed region)."""
        torch = self.torch
        t = torch.tensor(row, dtype=torch.int64, device=self.cdev)
        if not self.grouped:
            return [t.tolist()]
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return [o.tolist() for o in out]

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)

    def peak(self):
        if self.lop3_peak is None:
            self.gen.set_async(False)
            self.lop3_peak, _ = self.gen.lop3_peak()
            self.gen.set_async(True)
        return self.lop3_peak


def measure_workload(env: Env, name: str, n: int, clocks: int, layout: str, first: int, steps: int, warmup: int,
                     stride_per_step: int, sampler: ClockSampler | None = None) -> dict:
    """W warm-up + K timed steps of one workload on this rank.  Returns the per-workload record (rank-local
    kernel figures; `elapsed_ms` is the max over ranks)."""
    torch, gen, stream = env.torch, env.gen, env.stream
    G = n // 32
    gen.set_group_offset(first // 32)

    # ---- output buffer: whole keystream of one step resident in HBM when it fits
    out_bytes = n * clocks // 8
    torch.cuda.empty_cache()
    free, _total = torch.cuda.mem_get_info()
    state_bytes = G * (800 + 8 + 640) + (1 << 30)
    if out_bytes + state_bytes <= free:
        chunk_clocks, out_mode = clocks, "full"
    else:
        budget = max(1 << 28, int(free * 0.5) - state_bytes)
        chunk_clocks = max(1024, budget * 8 // n // 1024 * 1024)
        out_mode = f"ring({chunk_clocks} clocks)"
    if layout == "colmajor":
        out = torch.empty((chunk_clocks, G), dtype=torch.int32, device=env.dev)
    else:
        out = torch.empty((n, chunk_clocks // 8), dtype=torch.uint8, device=env.dev)

    # c5 (fresh key/IV pairs, init-dominated): explicit material arrays resident in HBM, so that the row-major
    # key/IV bytes -> bitsliced input words transposition is part of the step; c2 / c3: the
    # counter-IV set synthesised on device
    explicit = name == "c5"
    if explicit:
        gsrc = torch.Generator(device=env.dev).manual_seed(0x190904750 + env.rank)
        d_keys = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device=env.dev, generator=gsrc)
        d_ivs = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device=env.dev, generator=gsrc)

    gen_events, init_events = [], []
    launches = 0
    plan = None

    # c5 is the reference's one-shot call (mickey_sliced_words restarts from the key/IV load on every call,
    # kernels.py:189-200): mk2_bulk_rowmajor with everything on the device = ONE fused kernel (csrc/mk2_fused.cuh)
    one_shot = explicit and out_mode == "full"

    one_shot_sum = 0

    def step(i: int, record: bool):
        nonlocal launches, plan, one_shot_sum
        e0, e1 = env.event(), env.event()
        if one_shot:
            e0.record(stream)
            _, one_shot_sum = gen.bulk_rowmajor(d_keys, d_ivs, 80, clocks, out)
            e1.record(stream)
            launches += gen.last_kernel_launches
            if record:
                gen_events.append((e0, e1, clocks))
            if plan is None:
                plan = gen.last_plan()
            return
        e0.record(stream)
        if explicit:
            gen.init_material(d_keys, d_ivs, 80)
        else:
            gen.init_counter(KEY, first + (i % 4) * stride_per_step, n)
        e1.record(stream)
        launches += gen.last_kernel_launches
        if record:
            init_events.append((e0, e1))
        done = 0
        while done < clocks:
            tc = min(chunk_clocks, clocks - done)
            e0, e1 = env.event(), env.event()
            e0.record(stream)
            if layout == "colmajor":
                gen.generate_colmajor(tc, out)
            else:
                gen.generate_rowmajor(tc, out)
            e1.record(stream)
            launches += gen.last_kernel_launches
            if record:
                gen_events.append((e0, e1, tc))
            if plan is None:
                plan = gen.last_plan()
            done += tc

    for i in range(warmup):
        step(i, False)
    env.barrier()
    if sampler is not None:
        sampler.start()
        time.sleep(0.25)
    launches = 0
    t_wall0 = time.perf_counter()
    start, end = env.event(), env.event()
    env.barrier()
    start.record(stream)
    for i in range(steps):
        step(warmup + i, True)
    end.record(stream)
    env.barrier()
    t_wall1 = time.perf_counter()
    clocks_info = sampler.stop(t_wall0, t_wall1) if sampler is not None else None
    local_ms = start.elapsed_time(end)
    elapsed_ms = env.max_over_ranks(local_ms)
    gen_ms = [e0.elapsed_time(e1) for e0, e1, _ in gen_events]
    init_ms = [e0.elapsed_time(e1) for e0, e1 in init_events]
    gen_clk = sum(tc for _, _, tc in gen_events)
    kernel_ms_total = sum(gen_ms)
    checksum = one_shot_sum if one_shot else gen.checksum()   # of the last step's keystream, this rank's range
    two_call = None
    if one_shot:                                       # the same batch as pack + init + keystream kernels, for the split
        ti, tg = [], []
        for _ in range(3):
            ev = [env.event() for _ in range(3)]
            ev[0].record(stream)
            gen.init_material(d_keys, d_ivs, 80)
            ev[1].record(stream)
            gen.generate_rowmajor(clocks, out)
            ev[2].record(stream)
            env.torch.cuda.synchronize()
            ti.append(ev[0].elapsed_time(ev[1]))
            tg.append(ev[1].elapsed_time(ev[2]))
        assert gen.checksum() == checksum, "one-shot and two-call checksums differ"
        two_call = {"init_ms": min(ti), "keystream_ms": min(tg), "ms_per_step": min(a + b for a, b in zip(ti, tg)),
                    "note": "mk2_init_from_material + mk2_generate_rowmajor (pack_uniform_kernel, init_kernel, "
                            "tmem::gen_rowmajor_kernel): input words and state pass through HBM; same checksum"}

    # ---- roofline of the dominant kernel (keystream loop), this rank.
    # Algorithmic LOP3 per clock of the kernel as built: the clock runs in blocks of K clocks with R's reduction
    # deferred (csrc/mk2_clock.cuh); mk2_lop3_per_block is derived from the cipher's tables and checked against
    # the SASS by tests/test_structure.py.  SURVEY.md 8(d) counted 327 for the one-clock form.
    lib = env.lib
    which = 0 if layout == "colmajor" else 1
    rblock, per_block = lib.mk2_rblock(which), lib.mk2_lop3_per_block(which)
    lop3_per_clock = per_block / rblock
    lop3_peak = env.peak()
    irb, ipb = lib.mk2_rblock(2), lib.mk2_lop3_per_block(2)
    lane_ops = n * gen_clk * lop3_per_clock / 32          # algorithmic LOP3 lane-ops in the timed launches
    if one_shot:                                          # the launch also runs the 160 load clocks + 100 pre-clocks
        lane_ops += n / 32 * (160 + 100) * ipb / irb * len(gen_events)
    achieved = lane_ops / (kernel_ms_total * 1e-3)
    achieved_survey = achieved * LOP3_PER_CLOCK_SURVEY / lop3_per_clock
    if one_shot:  # 329 per load clock, 327 per pre-clock and keystream clock
        achieved_survey = n / 32 * (160 * 329 + (100 + clocks) * 327) * len(gen_events) / (kernel_ms_total * 1e-3)
    hbm_gbs = (n * gen_clk / 8) / (kernel_ms_total * 1e-3) / 1e9
    launch_clocks = gen_events[0][2] if gen_events else 0
    # in-run traffic model of one launch: the stores of the keystream itself plus the state parking of the
    # persistent scheduler (every chain-chunk job loads and stores 200 state words + one 8-byte accumulator per
    # thread, through L2); everything else (scheduler ring, progress words) is below 1 MB
    block_threads, chunk = plan if plan else (0, 0)
    jobs = ((n + 1023) // 1024) * (-(-launch_clocks // chunk) if chunk else 0)
    traffic_model = n * launch_clocks // 8 + jobs * 32 * 2 * (800 + 8)
    alg_bytes = n * launch_clocks // 8
    if one_shot:                                          # rows out + key/IV records in; nothing else touches HBM
        jobs = (n + 1023) // 1024
        traffic_model = alg_bytes = n * launch_clocks // 8 + n * 20
    ncu_bytes, ncu_src = NCU_TRAFFIC.get((layout, n, launch_clocks), (None, None))
    peaks = env.peaks
    roofline = {
        "bound": "lop3", "kernel": ("gen_colmajor_kernel" if layout == "colmajor" else
                                    "fused::bulk_rowmajor_kernel (key/IV records -> input words -> load clocks -> "
                                    "pre-clocks -> keystream -> rows)" if one_shot else "tmem::gen_rowmajor_kernel"),
        "achieved": achieved / 1e12, "peak": lop3_peak / 1e12, "unit": "Tlane-op/s", "frac": achieved / lop3_peak,
        "peak_source": "measured live by mk2_lop3_peak (dependency-free LOP3 kernel) on this GPU",
        "algorithmic_ops_per_launch": lane_ops / max(1, len(gen_events)),
        "lop3_per_clock": {"executed": lop3_per_clock, "block_clocks": rblock, "lop3_per_block": per_block,
                           "survey_one_clock_form": LOP3_PER_CLOCK_SURVEY},
        "at_survey_count": {"achieved": achieved_survey / 1e12, "frac": achieved_survey / lop3_peak,
                            "note": "same run priced at SURVEY 8(d)'s 327 LOP3 per clock: above 1 because the "
                                    "deferred R reduction executes fewer LOP3 than the one-clock form"},
        "avg_launch_ms": kernel_ms_total / max(1, len(gen_events)),
        "kernel_share_of_step": kernel_ms_total / local_ms,
        "plan": {"threads_per_cta": block_threads, "chunk_clocks": chunk, "jobs_per_launch": jobs},
        "traffic": ncu_bytes,
        "traffic_source": (f"{ncu_src}: ncu --set full capture of a launch of exactly this geometry, committed earlier; "
                           f"NOT measured in this run") if ncu_src else None,
        "traffic_model": traffic_model,
        "traffic_model_source": ("computed in this run: keystream rows out + key/IV records in (input words and state "
                                 "stay on the SM)") if one_shot else
                                "computed in this run from the launch plan: keystream stores + state parking of every "
                                "chain-chunk job (2 x 808 B per thread)",
        "algorithmic_bytes_per_launch": alg_bytes,
        "hbm": {"bound": "hbm", "achieved": hbm_gbs, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": hbm_gbs / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None,
                "peak_source": f"MEASURED_PEAKS.json ({env.peaks_src})", "note": "0.125 B stored per keystream bit; not binding"},
    }
    # whole step (pack + key/IV load + pre-clocks + keystream) against the same LOP3 peak: 160 load clocks and
    # 100 pre-clocks per instance at the init kernel's block count, T keystream clocks at the keystream kernel's
    step_ops = n / 32 * ((160 + 100) * ipb / irb + clocks * lop3_per_clock) * steps
    split = {
        "one_shot": True, "ms_per_step": kernel_ms_total / max(1, steps),
        "note": "one fused kernel per step: key/IV records -> input words (tensor memory) -> 160 load clocks -> 100 "
                "pre-clocks -> keystream -> rows; roofline.frac counts the load and pre-clocks' LOP3 too",
        "whole_step_lop3_frac": step_ops / (local_ms * 1e-3) / lop3_peak,
        "two_call_path": two_call,
    } if one_shot else {
        "init_ms_per_step": sum(init_ms) / max(1, steps), "keystream_ms_per_step": kernel_ms_total / max(1, steps),
        "init_note": ("pack_uniform_kernel (u8[N][10] key / IV rows -> bitsliced input words) + init_kernel" if explicit
                      else "pack_counter_kernel + init_kernel") + ": 160 load clocks + 100 pre-clocks per instance",
        "whole_step_lop3_frac": step_ops / (local_ms * 1e-3) / lop3_peak,
        "init_kernel_lop3_frac": (n / 32 * 260 * ipb / irb * steps) / (sum(init_ms) * 1e-3) / lop3_peak if init_ms else None,
    }
    del out
    if explicit:
        del d_keys, d_ivs
    torch.cuda.empty_cache()
    return {
        "name": name, "n": n, "clocks": clocks, "layout": layout, "explicit": explicit, "out_mode": out_mode,
        "out_bytes": out_bytes, "steps": steps, "warmup": warmup, "elapsed_ms": elapsed_ms, "local_ms": local_ms,
        "launches": launches, "roofline": roofline, "split": split, "clocks_info": clocks_info, "checksum": checksum,
        "first": first,
    }


def workload_text(name, n, clocks, layout, explicit):
    return (f"{name}: 2^{n.bit_length() - 1} instances x {clocks} bits per GPU, {layout}, "
            + ("explicit key/IV arrays (u8[N][10] each) resident in HBM, " if explicit else
               "counter-IV material synthesised on device, ") + "init + keystream per step") if n & (n - 1) == 0 else \
           (f"{name}: {n} instances x {clocks} bits per GPU, {layout}, counter-IV material synthesised on device, "
            "init + keystream per step")


def checksum_crosscheck(env: Env, shards) -> dict:
    """The only collective of the path, checked in the run: every rank computes the checksum of a small slice of
    ITS key/IV range (first 2048 instances x 512 bits) and the values are summed with one all-reduce (NCCL);
    rank 0 then recomputes every slice alone on its own GPU and must get the same 64-bit sum."""
    from paper_1909_04750_b200 import sharding

    pkg = env.pkg
    T = 512

    def slice_sum(first, count):
        with pkg.MickeyGenerator(env.local) as g:
            g.set_group_offset(first // 32)
            g.init_counter(KEY, first, min(count, 2048))
            g.generate_colmajor(T, env.torch.empty((T, (min(count, 2048) + 31) // 32), dtype=env.torch.int32, device=env.dev))
            return g.checksum()

    first, count = shards[env.rank]
    mine = slice_sum(first, count)
    reduced = sharding.allreduce_checksum(mine, device=env.cdev)
    alone = 0
    if env.rank == 0:
        for f, c in shards:
            alone = (alone + slice_sum(f, c)) % (1 << 64)
    return {"slice": f"first {min(count, 2048)} instances of every rank x {T} bits", "allreduced": f"{reduced:#018x}",
            "single_rank_recomputation": f"{alone:#018x}", "equal": reduced == alone if env.rank == 0 else None,
            "collective": f"one int64 SUM all-reduce ({env.backend}, world size {env.world})" if env.grouped
                          else "none (no process group: single process)"}


def run_ours(args):
    env = Env(args)
    np, torch, pkg, gen = env.np, env.torch, env.pkg, env.gen
    from paper_1909_04750_b200 import sharding

    world, rank, local = env.world, env.rank, env.local
    lg, clocks, layout, cfg = WORKLOADS[args.workload]
    if args.instances_log2 is not None:
        lg = args.instances_log2
    if args.clocks is not None:
        clocks = args.clocks
    if args.scaling == "strong":
        # configs[3]: a fixed job of total_bits, split into disjoint contiguous key/IV ranges of whole groups
        total_n = max(32 * world, int(args.total_bits // clocks) // 32 * 32)
        sh = sharding.shard_instances(total_n, world, rank)
        n, first, stride = sh.count, sh.first, total_n
        shards = [(s.first, s.count) for s in (sharding.shard_instances(total_n, world, r) for r in range(world))]
    else:
        n = 1 << lg
        first, stride, total_n = rank * n, world * n, world * n   # disjoint key/IV (instance index) range per rank
        shards = [(r * n, n) for r in range(world)]

    sampler = ClockSampler(local) if rank == 0 else None
    main = measure_workload(env, args.workload, n, clocks, layout, first, args.steps, args.warmup, stride, sampler)
    bits_per_step = total_n * clocks
    value = bits_per_step * args.steps / (main["elapsed_ms"] * 1e-3) / 1e12

    # ---- per-rank record + the checksum all-reduce (the only exchange; outside the timed region)
    csum = sharding.allreduce_checksum(main["checksum"], device=env.cdev)
    rows = env.gather_rows([rank, first, n, int(round(main["local_ms"] * 1e3)), sharding.to_i64(main["checksum"])])
    ranks = [{"rank": r[0], "first": r[1], "count": r[2], "ms": r[3] / 1e3, "checksum": f"{sharding.from_i64(r[4]):#018x}"}
             for r in rows]
    check = checksum_crosscheck(env, shards)

    # ---- the other single-GPU configs of BASELINE.json, same process, same protocol
    extras = {}
    if args.extras == "auto":
        extra_names = [w for w in WORKLOADS if w != args.workload] if (world == 1 and args.workload == "c2"
                                                                      and args.scaling == "weak"
                                                                      and args.instances_log2 is None
                                                                      and args.clocks is None) else []
    elif args.extras == "none":
        extra_names = []
    else:
        extra_names = [w for w in args.extras.split(",") if w in WORKLOADS and w != args.workload]
    for w in extra_names:
        wlg, wclk, wlay, wcfg = WORKLOADS[w]
        wn = 1 << wlg
        k = max(1, min(args.steps, 5))
        rec = measure_workload(env, w, wn, wclk, wlay, rank * wn, k, max(3, min(args.warmup, 3)), world * wn)
        extras[w] = {
            "baseline_config": f"BASELINE.json configs[{wcfg}]",
            "workload": workload_text(w, wn, wclk, wlay, rec["explicit"]),
            "value": world * wn * wclk * k / (rec["elapsed_ms"] * 1e-3) / 1e12, "unit": "Tb/s",
            "ms_per_step": rec["elapsed_ms"] / k, "steps": k, "warmup": rec["warmup"], "output": rec["out_mode"],
            "gpu_launches": rec["launches"], "roofline": rec["roofline"], "step_split": rec["split"],
            "checksum_u64_sum": f"{rec['checksum']:#018x}",
        }

    # ---- host-buffer legs through the public API
    e2e = e2e_page = latency = None
    if not args.no_e2e:
        e2e, e2e_page = run_e2e(env, n, clocks, layout, first)
    ragged = None
    if not args.no_latency and rank == 0:
        latency = small_call_latency(env)
        ragged = ragged_init(env)

    # ---- roofline.traffic, live: DRAM bytes of one launch of every measured workload, counted by ncu in a child
    # process (default geometry only; the parent has released its output buffers by now)
    default_geometry = args.instances_log2 is None and args.clocks is None and args.scaling == "weak"
    if rank == 0 and not env.grouped and not args.no_ncu_traffic and default_geometry:
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        apply_live_traffic(main["roofline"], args.workload)
        for w in extras:
            apply_live_traffic(extras[w]["roofline"], w)

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Tb/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["elapsed_ms"] / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {
                "workload": workload_text(args.workload, n, clocks, layout, main["explicit"]),
                "baseline_config": f"BASELINE.json configs[{cfg}]" + (" shape per rank; configs[3] job" if args.scaling == "strong" else ""),
                "instances_per_gpu": n, "clocks": clocks, "layout": layout, "output": main["out_mode"],
                "total_instances": total_n, "total_bits_per_step": bits_per_step,
                "l2": f"no flush needed: each step streams {main['out_bytes'] / 1e9:.1f} GB of output per GPU (>> 126 MB L2)",
                "parallelism": f"{world} x disjoint key/IV ranges ({args.scaling} scaling), no data-path collective"
                               + ("" if env.backend == "nccl" or world == 1 else
                                  f"; DEBUG backend gloo: {world} ranks share {torch.cuda.device_count()} GPU(s), not a multi-GPU figure"),
            },
            "roofline": main["roofline"], "step_split": main["split"], "clocks": main["clocks_info"],
            "gpu_launches": main["launches"],
            "checksum_u64_sum": f"{csum:#018x}", "ranks": ranks, "checksum_check": check,
        }
        if extras:
            line["extra_workloads"] = extras
        if e2e:
            line["e2e"] = e2e
        if e2e_page:
            line["e2e_pageable"] = e2e_page
        if latency:
            line["small_call_latency"] = latency
        if ragged:
            line["ragged_init"] = ragged
        if not args.no_curand:
            try:
                line["curand"] = curand_compare(torch, 1 << 32)
            except Exception as exc:  # comparison only; never blocks the bench line
                line["curand"] = {"error": str(exc)}
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_sample(args.cpu_seconds)
    gen.close()
    if env.grouped:
        env.barrier()
        env.dist.destroy_process_group()
    if line:
        emit(line)


def run_e2e(env: Env, n, clocks, layout, first):
    """Same metric through the C-ABI call with HOST buffers, host<->device copies inside the timed region.
      e2e           pinned key/IV arrays in, pinned keystream out, the WHOLE workload length: column-major runs
                    the full `clocks` as resumable calls of --e2e-clocks bits into a ring of two pinned buffers
                    (the consumer owns one while the next fills); row-major is the one-shot mk2_bulk_rowmajor.
      e2e_pageable  the reference's calling convention (kernels.py:189-200): ordinary (pageable) numpy key/IV
                    arrays in, numpy keystream out -- into a caller-supplied pageable array (the library's copy
                    lanes) and into the fresh result array the package returns
                    (page-locked block from its pool).  Bounded sample: one --e2e-clocks call per step."""
    args, np, torch, pkg, gen = env.args, env.np, env.torch, env.pkg, env.gen
    world = env.world
    tc = max(8, min(args.e2e_clocks, clocks) // 8 * 8)
    n_full = n
    n = max(1024, min(n, (1 << 34) // tc // 1024 * 1024))      # <= 2 GiB of keystream per call
    keys_np = np.tile(np.frombuffer(KEY, np.uint8), (n, 1))
    idx = (np.arange(n, dtype=np.uint64) + np.uint64(first))
    ivs_np = np.zeros((n, 10), np.uint8)
    ivs_np[:, 2:] = idx.astype(">u8").view(np.uint8).reshape(n, 8)   # 80-bit big-endian index
    keys, ivs = torch.from_numpy(keys_np).pin_memory(), torch.from_numpy(ivs_np).pin_memory()
    gen.set_stream(None)
    gen.set_async(False)
    steps = max(1, min(args.steps, 3))
    G = n // 32

    def timed(fn, reps, warm=2):
        for _ in range(warm):
            fn()
        env.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return env.max_over_ranks(time.perf_counter() - t0) / reps

    def timed_calls(fn, reps, warm=2):
        """Median of individually timed calls (every call ends with its result complete in host memory): the
        short host-buffer legs are CPU-side work on a shared host, where one disturbed call skews a 3-call mean."""
        for _ in range(warm):
            fn()
        env.barrier()
        v = []
        for _ in range(max(reps, 5)):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            v.append(time.perf_counter() - t0)
        return env.max_over_ranks(statistics.median(v))

    # ---- pageable numpy in / numpy out (bounded sample: one call of tc bits per step)
    res = {"unit": "Tb/s", "h2d_bytes_per_step": int(keys_np.nbytes + ivs_np.nbytes), "d2h_bytes_per_step": int(n * tc // 8),
           "steps": max(steps, 5), "timing": "median of individually timed calls, 2 warm-up calls"}
    if layout == "colmajor":
        pinned_one = torch.empty((tc, G), dtype=torch.int32).pin_memory()
        dt_pin = timed_calls(lambda: (gen.init_material(keys, ivs, 80), gen.generate_colmajor(tc, pinned_one)), steps)
        del pinned_one
        page = np.empty((tc, G), np.uint32)
        dt_page = timed_calls(lambda: (gen.init_material(keys_np, ivs_np, 80), gen.generate_colmajor(tc, page)), steps)
        del page
        dt_fresh = timed_calls(lambda: pkg.bulk_colmajor(keys_np, ivs_np, 80, tc, device=env.local), steps)
        calls = ("caller-supplied pageable array: mk2_init_from_material + mk2_generate_colmajor",
                 "pkg.bulk_colmajor(keys, ivs, 80, T) returning a fresh array")
    else:
        pinned_one = torch.empty((n, tc // 8), dtype=torch.uint8).pin_memory()
        dt_pin = timed_calls(lambda: gen.bulk_rowmajor(keys, ivs, 80, tc, pinned_one), steps)
        del pinned_one
        page = np.empty((n, tc // 8), np.uint8)
        dt_page = timed_calls(lambda: gen.bulk_rowmajor(keys_np, ivs_np, 80, tc, page), steps)
        del page
        dt_fresh = timed_calls(lambda: pkg.bulk_rowmajor(keys_np, ivs_np, 80, tc, device=env.local), steps)
        calls = ("caller-supplied pageable array: mk2_bulk_rowmajor", "pkg.bulk_rowmajor(keys, ivs, 80, T) returning a fresh array")
    bits = world * n * tc
    res.update({
        "value": bits / dt_page / 1e12, "ms_per_step": dt_page * 1e3, "d2h_gb_s": n * tc / 8 / dt_page / 1e9,
        "fresh_result_array": {"value": bits / dt_fresh / 1e12, "ms_per_step": dt_fresh * 1e3, "call": calls[1],
                               "note": "the package's result arrays are page-locked blocks from a cached pool (hostmem.py)"},
        "pinned_same_sample": {"value": bits / dt_pin / 1e12, "ms_per_step": dt_pin * 1e3},
        "pageable_over_pinned": dt_pin / dt_page, "fresh_over_pinned": dt_pin / dt_fresh,
        "workload": f"{n} of {n_full} instances x {tc} bits per GPU per call, pageable numpy key/IV arrays in; value = "
                    + calls[0] + " (copy lanes inside the library: host threads with their own stream and page-locked slots)",
    })
    # ---- pinned, whole length
    if layout == "colmajor":
        ring = [torch.empty((tc, G), dtype=torch.int32).pin_memory() for _ in range(2)]
        full_clocks = clocks if n == n_full else tc
        ncalls = -(-full_clocks // tc)

        def one():
            gen.init_material(keys, ivs, 80)
            done, i = 0, 0
            while done < full_clocks:
                c = min(tc, full_clocks - done)
                gen.generate_colmajor(c, ring[i & 1][:c])
                done += c
                i += 1

        dt = timed(one, steps, warm=1)
        d2h = n * full_clocks // 8
        how = (f"mk2_init_from_material(pinned host keys, IVs) + {ncalls} resumable mk2_generate_colmajor calls of {tc} bits "
               f"into a ring of two pinned {tc * G * 4 >> 20} MiB host buffers")
        del ring
    else:
        host = torch.empty((n, tc // 8), dtype=torch.uint8).pin_memory()
        full_clocks = tc

        def one():
            gen.bulk_rowmajor(keys, ivs, 80, tc, host)   # one-shot call: upload | init + keystream | download overlap

        dt = timed(one, steps)
        d2h = n * tc // 8
        how = "mk2_bulk_rowmajor(pinned host keys, IVs -> pinned host out), instance blocks pipelined"
        del host
    e2e = {
        "value": world * n * full_clocks / dt / 1e12, "unit": "Tb/s",
        "h2d_bytes_per_step": int(keys.numel() + ivs.numel()), "d2h_bytes_per_step": int(d2h),
        "ms_per_step": dt * 1e3, "steps": steps, "d2h_gb_s": d2h / dt / 1e9,
        "workload": (f"{n} of {n_full} instances x {full_clocks} of {clocks} bits per GPU per step: " if (n, full_clocks) != (n_full, clocks)
                     else f"the whole workload, {n} instances x {clocks} bits per GPU per step: ")
                    + how + "; the host link, not the kernel, bounds it",
    }

    gen.set_async(True)
    return e2e, res


def ragged_init(env: Env) -> dict:
    """Key/IV load + pre-clocks of 2^20 instances whose IV lengths differ (uniform over 0, 8, ..., 80 bits: the
    reference's acceptance workload, tests/test_acceptance.py:103-135; mickey.py:287-289 gives such sets a per-lane
    scalar init) against the uniform 80-bit init of the same instances.  Device-resident material; device time of
    the packing + init kernels (mk2_last_kernel_ms), best of 5 after a warm-up call."""
    np, torch, pkg = env.np, env.torch, env.pkg
    n = 1 << 20
    rng = np.random.default_rng(1)
    keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).to(env.dev)
    ivs = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).to(env.dev)
    nb_bytes = torch.from_numpy((8 * rng.integers(0, 11, n)).astype(np.uint8)).to(env.dev)
    nb_bits = torch.from_numpy(rng.integers(0, 81, n).astype(np.uint8)).to(env.dev)
    with pkg.MickeyGenerator(env.local) as g:
        def ms(fn):
            v = []
            for _ in range(6):
                fn()
                v.append(g.last_kernel_ms)
            return min(v[1:])
        uni = ms(lambda: g.init_material(keys, ivs, 80))
        rb = ms(lambda: g.init_ragged(keys, ivs, nb_bytes))
        rbit = ms(lambda: g.init_ragged(keys, ivs, nb_bits))
    return {"instances": n, "uniform_80bit_ms": uni, "ragged_iv_0_to_10_bytes_ms": rb, "ragged_iv_0_to_80_bits_ms": rbit,
            "ragged_over_uniform": rb / uni,
            "note": "pack_ragged_kernel (128-bit loads, funnel shifts, 32x32 bit transposes) + init_kernel<true> (masked "
                    "4-clock blocks, +5 LOP3 per IV clock); ragged includes the D2H of the 1 MiB length array"}


def small_call_latency(env: Env) -> dict:
    """The reference's batching pattern (cli.py:219-231): one mickey_sliced_words call per 64 lanes.  Wall time of
    a 64-lane x 4096-clock call with an idle context of the thread reused (the default) and with a new context per
    call (round 1 behaviour), against the device time of its kernels."""
    from paper_1909_04750_b200 import hostmem

    pkg = env.pkg
    mats = [pkg.MickeyKeyIv(KEY, bytes.fromhex("21436587"))] * 64

    def best(fn, reps):
        v = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            v.append(time.perf_counter() - t0)
        return min(v) * 1e6, statistics.median(v) * 1e6

    pkg.mickey_sliced_words(mats, 4096, device=env.local)
    pooled = best(lambda: pkg.mickey_sliced_words(mats, 4096, device=env.local), 30)

    def fresh():
        hostmem.drop_idle_contexts()
        pkg.mickey_sliced_words(mats, 4096, device=env.local)
    unpooled = best(fresh, 8)
    keys, ivs, nbits, _ = pkg.mickey.pack_materials(mats, 64)
    pack_us = best(lambda: pkg.mickey.pack_materials(mats, 64), 10)[0]
    def abi_calls(small_batch: bool):
        with pkg.MickeyGenerator(env.local) as g:
            g.set_small_batch(small_batch)
            g.init_material(keys, ivs, 32).generate_colmajor(4096)
            kern, wall = [], []
            for _ in range(20):
                t0 = time.perf_counter()
                g.init_material(keys, ivs, 32)
                k = g.last_kernel_ms
                g.generate_colmajor(4096)
                k += g.last_kernel_ms
                wall.append(time.perf_counter() - t0)
                kern.append(k)
        return kern, wall

    kern, wall = abi_calls(True)
    kern_tpg, _ = abi_calls(False)
    return {"call": "mickey_sliced_words(64 lanes, 4096 clocks) -> uint64[4096] on the host",
            "idle_context_reused_us": {"best": pooled[0], "median": pooled[1]},
            "new_context_per_call_us": {"best": unpooled[0], "median": unpooled[1]},
            "python_validation_and_packing_us": pack_us,
            "c_abi_init_plus_generate_us": {"wall_best": min(wall) * 1e6, "device_kernels_best": min(kern) * 1e3},
            "kernels": "warp-per-group small-batch kernels (csrc/mk2_coop.cuh): the 200 state bits of a 32-instance group "
                       "spread over the lanes of one warp",
            "device_kernels_thread_per_group_us": min(kern_tpg) * 1e3,
            "small_batch_speedup_on_device": min(kern_tpg) / min(kern),
            "overhead_over_kernel_time_us": pooled[0] - min(kern) * 1e3,
            "overhead_over_kernel_time_excluding_python_packing_us": pooled[0] - min(kern) * 1e3 - pack_us}


def traffic_child(args):
    """Child of measure_traffic_live: two launches of the workload's keystream kernel at its exact geometry (ncu
    skips the first and counts the DRAM bytes of the second).  Nothing is timed here."""
    import torch

    import paper_1909_04750_b200 as pkg

    lg, clocks, layout, _cfg = WORKLOADS[args.workload]
    n = 1 << lg
    dev = torch.device("cuda", 0)
    with pkg.MickeyGenerator(0) as gen:
        if args.workload == "c5":
            g = torch.Generator(device=dev).manual_seed(0x190904750)
            d_keys = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device=dev, generator=g)
            d_ivs = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device=dev, generator=g)
        out = (torch.empty((clocks, n // 32), dtype=torch.int32, device=dev) if layout == "colmajor"
               else torch.empty((n, clocks // 8), dtype=torch.uint8, device=dev))
        for _ in range(2):
            if args.workload == "c5":
                gen.bulk_rowmajor(d_keys, d_ivs, 80, clocks, out)
                continue
            gen.init_counter(KEY, 0, n)
            gen.generate_colmajor(clocks, out) if layout == "colmajor" else gen.generate_rowmajor(clocks, out)
        torch.cuda.synchronize()


def measure_traffic_live(workload: str, timeout_s: float = 300.0):
    """roofline.traffic measured in THIS run: dram__bytes_read.sum + dram__bytes_write.sum of one launch of the
    workload's keystream kernel at its full geometry, counted by ncu around a child process of this script (a
    number taken under a profiler is never a timing; DRAM byte counts are what the profiler is for).
    Returns (bytes, source) or (None, reason)."""
    import csv
    import io
    import shutil

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).exists():
        return None, "ncu not found"
    layout = WORKLOADS[workload][2]
    kern = "gen_colmajor_kernel" if layout == "colmajor" else "bulk_rowmajor_kernel" if workload == "c5" else "gen_rowmajor_kernel"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none", "--print-units", "base",
           "--csv", "-k", f"regex:{kern}", "--launch-skip", "1", "--launch-count", "1",
           sys.executable, str(Path(__file__).resolve()), "--traffic-child", "--workload", workload]
    try:
        res = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, timeout=timeout_s, cwd=str(ROOT))
    except (OSError, subprocess.TimeoutExpired) as exc:
        return None, f"ncu child failed: {exc!r}"[:200]
    start = res.stdout.find('"ID"')
    if res.returncode != 0 or start < 0:
        tail = (res.stdout + res.stderr).strip().splitlines()[-1:] or ["no output"]
        return None, f"ncu child rc={res.returncode}: {tail[0]}"[:200]
    total, seen = 0, 0
    for row in csv.DictReader(io.StringIO(res.stdout[start:])):
        if row.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += int(float(row["Metric Value"].replace(",", "")))
            seen += 1
    if seen != 2:
        return None, "ncu output without the two DRAM counters"
    return total, ("measured in this run: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none around "
                   f"a child process of bench.py, one {kern} launch of exactly this geometry (second of two)")


def apply_live_traffic(roofline: dict, workload: str):
    live, src = measure_traffic_live(workload)
    roofline["traffic_committed_profile"] = {"bytes": roofline.get("traffic"), "source": roofline.get("traffic_source")}
    if live is not None:
        roofline["traffic"], roofline["traffic_source"] = live, src
        alg = roofline.get("algorithmic_bytes_per_launch")
        roofline["traffic_over_algorithmic"] = live / alg if alg else None
    else:
        roofline["traffic_live_unavailable"] = src


_JSON_OUT = None


def claim_stdout():
    """stdout must carry exactly ONE JSON line, but libraries write there too (NCCL prints its version banner to
    stdout when NCCL_DEBUG is set, numba and ncu children may warn): keep a private handle on the real stdout for
    the line and point file descriptor 1 at stderr for everybody else."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict):
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    args = parse_args()
    claim_stdout()
    if args.traffic_child:
        traffic_child(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
