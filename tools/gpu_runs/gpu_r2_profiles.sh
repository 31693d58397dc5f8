#!/bin/bash
# Round 2: driver-shaped bench line (c2 + c3/c5 extras + e2e legs), reference arm, strong-scaling mode at world 1,
# ncu launch list of the bench command, ncu --set full captures of the c3 / c5 keystream kernels and of the ragged
# init (summaries only: the .ncu-rep files stay in /tmp on the box).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/r02_smoke.log
(time python bench.py --steps 5 --warmup 3) > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"; tail -4 gpurun_out/r02_bench_default.err
(time python bench.py --impl reference --steps 5 --warmup 1) > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err; echo "ref rc=$?"; tail -4 gpurun_out/r02_bench_reference_arm.err
python bench.py --scaling strong --total-bits 8e12 --steps 2 --warmup 3 --no-e2e --no-curand --no-cpu-baseline --no-latency > gpurun_out/r02_bench_strong_1gpu.json 2> gpurun_out/r02_bench_strong.err; echo "strong rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 2 --warmup 3 --extras none --no-e2e --no-curand --no-cpu-baseline --no-latency > gpurun_out/r02_bench_torchrun_1gpu.json 2> gpurun_out/r02_bench_torchrun.err; echo "torchrun rc=$?"
# launch list of the bench command (per-launch times are serialised and cold: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_ncu_launches_bench_default.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-curand --no-cpu-baseline --no-latency > /tmp/ncu_bench.json 2> /tmp/ncu_bench.err; echo "ncu launches rc=$?"
# full captures: one launch of each kernel at the bench geometry
ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor --launch-skip 3 --launch-count 1 -f -o /tmp/r02_c3 \
    python bench.py --workload c3 --extras none --steps 1 --warmup 3 --no-e2e --no-curand --no-cpu-baseline --no-latency > /dev/null 2> /tmp/ncu_c3.err; echo "ncu c3 rc=$?"
python tools/ncu_summary.py /tmp/r02_c3.ncu-rep gpurun_out/r02_ncu_gen_rowmajor_c3_full.txt "tmem::gen_rowmajor_kernel, BASELINE config 3 at full size (2^24 instances x 65536 bits, 137 GB)" > /dev/null
ncu --set full --clock-control none --import-source on -k regex:'gen_rowmajor|init_kernel|pack_uniform' --launch-skip 9 --launch-count 3 -f -o /tmp/r02_c5 \
    python bench.py --workload c5 --extras none --steps 1 --warmup 3 --no-e2e --no-curand --no-cpu-baseline --no-latency > /dev/null 2> /tmp/ncu_c5.err; echo "ncu c5 rc=$?"
python tools/ncu_summary.py /tmp/r02_c5.ncu-rep gpurun_out/r02_ncu_c5_pack_init_keystream.txt "BASELINE config 5 at full size (2^26 pairs x 1024 bits): pack_uniform_kernel, init_kernel<false>, tmem::gen_rowmajor_kernel of one step" > /dev/null
ncu --set full --clock-control none --import-source on -k regex:'init_kernel|pack_ragged' --launch-skip 8 --launch-count 2 -f -o /tmp/r02_ragged \
    python tools/probe_r2.py ragged > /dev/null 2> /tmp/ncu_ragged.err; echo "ncu ragged rc=$?"
python tools/ncu_summary.py /tmp/r02_ragged.ncu-rep gpurun_out/r02_ncu_ragged_init.txt "ragged IV lengths at 2^20 lanes: pack_ragged_kernel (vectorised) + init_kernel<true> (masked 4-clock blocks)" > /dev/null
ls -la gpurun_out | tail -20
