#!/bin/bash
# Round 2: compute-sanitizer over every kernel and the new host paths (tools/sanitize.py), then memcheck over the
# GPU parity tests that do not need tens of GB.
mkdir -p gpurun_out
: > gpurun_out/r02_compute_sanitizer.txt
for tool in memcheck racecheck initcheck; do
  echo "== compute-sanitizer --tool $tool python tools/sanitize.py" >> gpurun_out/r02_compute_sanitizer.txt
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize.py > /tmp/san_$tool.log 2>&1; echo "$tool rc=$?" >> /tmp/san_$tool.log
  grep -v "^$" /tmp/san_$tool.log | tail -6 >> gpurun_out/r02_compute_sanitizer.txt
done
echo "== compute-sanitizer --tool memcheck python -m pytest tests -m gpu (everything except the full-size / 2^20+-instance tests)" >> gpurun_out/r02_compute_sanitizer.txt
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest tests -m gpu -q -x \
  -k "not full_size and not full_coverage and not full_length and not c2_instance and not c3_instance and not large and not at_scale and not nist and not two_ranks and not failures and not acceptance and not randomized and not pageable and not reuse_idle" > /tmp/san_pytest.log 2>&1; echo "pytest memcheck rc=$?" >> /tmp/san_pytest.log
grep -v "^$" /tmp/san_pytest.log | tail -6 >> gpurun_out/r02_compute_sanitizer.txt
cat gpurun_out/r02_compute_sanitizer.txt
