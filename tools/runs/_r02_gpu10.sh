# Round 2, GPU call 10: split-K fix-up fused into the TMA GEMM (ibmi_tune key 15): suite, A/B on c2/c3/c4, benches.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02m_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02m_pytest.log
for c in c2 c3 c4; do
  for t in 1 0; do
    timeout 600 python tools/profile_sweep.py --config $c --sweeps 4 --tune 15=$t > gpurun_out/r02m_${c}_splitfused$t.log 2>&1
    echo "$c key15=$t: $(tail -1 gpurun_out/r02m_${c}_splitfused$t.log)"
  done
done
for c in c4 c2 c3; do
  timeout 1200 python bench.py --config $c --no-alt > gpurun_out/r02m_bench_$c.json 2> gpurun_out/r02m_bench_$c.err; echo bench_$c=$?
  head -c 160 gpurun_out/r02m_bench_$c.json; echo
done
