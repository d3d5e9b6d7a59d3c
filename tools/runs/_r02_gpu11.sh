# Round 2, GPU call 11: final binary (fused split-K off by default): suite, smoke, bench lines.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02n_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02n_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n_smoke.log 2>&1; echo smoke=$?
for c in c4 c1 c2 c3; do
  timeout 1200 python bench.py --config $c > gpurun_out/r02n_bench_$c.json 2> gpurun_out/r02n_bench_$c.err; echo bench_$c=$?
  head -c 160 gpurun_out/r02n_bench_$c.json; echo
done
