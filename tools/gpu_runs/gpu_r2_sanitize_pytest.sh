#!/bin/bash
# memcheck over the GPU parity tests that do not need tens of GB (second part of gpu_r2_sanitize.sh, rerun).
# test_reference_shaped_calls_reuse_idle_contexts is left out: it counts the idle contexts of the thread, and under
# compute-sanitizer the Python frame of every call that allocates device memory is kept alive by the tool's saved
# allocation backtrace (gc.get_referrers shows a materialised frame of keystream_words that nothing in Python
# holds), so engine objects are not finalised when the test deletes them.  It passes in the plain run.
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest tests -m gpu -q \
  -k "not full_size and not full_coverage and not full_length and not c2_instance and not c3_instance and not large and not at_scale and not nist and not two_ranks and not failures and not acceptance and not randomized and not pageable and not reuse_idle" > /tmp/san_pytest.log 2>&1; echo "pytest memcheck rc=$?" >> /tmp/san_pytest.log
grep -v "^$" /tmp/san_pytest.log | tail -12 | tee gpurun_out/r02_compute_sanitizer_pytest.txt
