"""Raw device-to-host copy rate of the box over time (1 GiB cudaMemcpyAsync into pinned memory, nothing else running):
the ceiling and the noise floor of every host-buffer (e2e) figure.  usage: probe_d2h_stability.py [seconds]"""
import sys, time, torch
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 40
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
h.copy_(x); torch.cuda.synchronize()
t_end = time.perf_counter() + secs
rates = []
while time.perf_counter() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); h.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
    rates.append((1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
rates.sort()
n = len(rates)
print(f"{n} copies of 1 GiB in {secs:.0f} s: min {rates[0]:.1f}  p10 {rates[n // 10]:.1f}  median {rates[n // 2]:.1f}  p90 {rates[9 * n // 10]:.1f}  max {rates[-1]:.1f} GB/s")
