import sys, time; sys.path.insert(0, ".")
from paper_1909_04750_b200 import cli
seed = bytes([0x11]) * 32
cli.suite_streams(seed, 4, 8192)
for _ in range(2):
    t0 = time.perf_counter(); rows = cli.suite_streams(seed, 100, 1_000_000); dt = time.perf_counter() - t0
    print("suite_streams(100 x 1 Mbit):", round(dt * 1e3, 1), "ms", rows.shape, flush=True)
