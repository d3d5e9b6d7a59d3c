# Round 2, GPU call 6: compute-sanitizer memcheck of the workload that touches every kernel path
# (one sanitizer tool per call), the sharded GPU tests after the estimate change, sharded world-1 timings.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -x -q > gpurun_out/r02i_pytest_sharded.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02i_pytest_sharded.log
for o in replicated sharded; do
  timeout 600 python tools/profile_sharded.py --config c4 --operands $o > gpurun_out/r02i_sharded_n1_$o.log 2>&1; echo sh=$?
  tail -n 4 gpurun_out/r02i_sharded_n1_$o.log
done
timeout 600 python tools/sanitize_run.py > gpurun_out/r02i_sanitize_plain.log 2>&1 && \
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 7 python tools/sanitize_run.py > gpurun_out/r02i_memcheck.log 2>&1; echo memcheck=$?
tail -8 gpurun_out/r02i_memcheck.log
