"""The bench line's e2e leg (whole config-2 workload through pinned host buffers) with every call timed: where do slow
runs lose their time?  usage: probe_e2e_full.py [steps]"""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1909_04750_b200 as pkg
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n, clocks, tc = 1 << 20, 1_000_000, 16384
G = n // 32
KEY = bytes.fromhex("123456789abcdef01234")
keys = torch.from_numpy(np.tile(np.frombuffer(KEY, np.uint8), (n, 1))).pin_memory()
ivs = torch.from_numpy(np.arange(n, dtype=">u8").view(np.uint8).reshape(n, 8)).contiguous()
ivs = torch.cat([torch.zeros((n, 2), dtype=torch.uint8), ivs], dim=1).contiguous().pin_memory()
ring = [torch.empty((tc, G), dtype=torch.int32).pin_memory() for _ in range(2)]
with pkg.MickeyGenerator(0) as gen:
    for s in range(steps + 1):
        t_step = time.perf_counter()
        gen.init_material(keys, ivs, 80)
        done, i, v = 0, 0, []
        while done < clocks:
            c = min(tc, clocks - done)
            t0 = time.perf_counter(); gen.generate_colmajor(c, ring[i & 1][:c]); v.append((time.perf_counter() - t0, c))
            done += c; i += 1
        dt = time.perf_counter() - t_step
        rates = sorted(c * G * 4 / t / 1e9 for t, c in v[:-1])
        slow = sum(1 for r in rates if r < 54)
        print(f"step {s}{' (warm-up)' if s == 0 else ''}: {dt * 1e3:8.1f} ms  {n * clocks / 8 / dt / 1e9:5.2f} GB/s = {n * clocks / dt / 1e12:.4f} Tb/s | per call GB/s: min {rates[0]:.1f} "
              f"p10 {rates[len(rates) // 10]:.1f} median {rates[len(rates) // 2]:.1f} max {rates[-1]:.1f}; calls below 54 GB/s: {slow} of {len(rates)}", flush=True)
