# Round 2, GPU call 9: sharded tests (Gram split, guesses), whole GPU suite with NaN-poisoned allocations,
# fused small sweep after the k-loop unroll.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -x -q > gpurun_out/r02l_pytest_sharded.log 2>&1; echo pytest_sharded=$?
tail -3 gpurun_out/r02l_pytest_sharded.log
IBMI_MEM_POISON=1 timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02l_pytest_poison.log 2>&1; echo pytest_poison=$?
tail -3 gpurun_out/r02l_pytest_poison.log
for i in 1 2; do
  timeout 300 python tools/profile_sweep.py --config c1 --sweeps 6 > gpurun_out/r02l_c1_fused_$i.log 2>&1
  tail -1 gpurun_out/r02l_c1_fused_$i.log
done
timeout 600 python bench.py --config c1 --no-alt > gpurun_out/r02l_bench_c1.json 2> gpurun_out/r02l_bench_c1.err; echo bench_c1=$?
head -c 200 gpurun_out/r02l_bench_c1.json; echo
