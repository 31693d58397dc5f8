#!/bin/bash
# host-buffer (e2e) throughput, default library vs variants given as arguments, interleaved
for rep in 1 2 3; do
for lib in "" "$@"; do
  echo "== rep $rep lib=${lib:-default}"
  MK2_LIB=$lib python - <<'PY'
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch, paper_1909_04750_b200 as pkg
KEY = bytes.fromhex("123456789abcdef01234")
def run(layout, n, tc):
    gen = pkg.MickeyGenerator(0)
    keys = torch.from_numpy(np.tile(np.frombuffer(KEY, np.uint8), (n, 1))).pin_memory()
    ivs_np = np.zeros((n, 10), np.uint8); ivs_np[:, 2:] = np.arange(n, dtype=np.uint64).astype(">u8").view(np.uint8).reshape(n, 8)
    ivs = torch.from_numpy(ivs_np).pin_memory()
    host = (torch.empty((tc, n // 32), dtype=torch.int32) if layout == "col" else torch.empty((n, tc // 8), dtype=torch.uint8)).pin_memory()
    def one():
        if layout == "col":
            gen.init_material(keys, ivs, 80); gen.generate_colmajor(tc, host)
        else:
            gen.bulk_rowmajor(keys, ivs, 80, tc, host)
    for _ in range(2): one()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(4): one()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 4
    print(f"{layout} n=2^{n.bit_length()-1} T={tc}: {dt*1e3:.2f} ms/step {n*tc/dt/1e12:.4f} Tb/s  D2H {host.numel()*host.element_size()/dt/1e9:.1f} GB/s", flush=True)
    gen.close()
run("col", 1 << 20, 16384); run("row", 1 << 20, 16384); run("row", 1 << 24, 1024)
PY
done; done
