# Round 2, GPU call 12: the default split-K GEMM instance without the fix-up code (template parameter): suite + benches.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02o_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02o_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.log 2>&1; echo smoke=$?
for c in c4 c3 c2 c1; do
  timeout 1200 python bench.py --config $c > gpurun_out/r02o_bench_$c.json 2> gpurun_out/r02o_bench_$c.err; echo bench_$c=$?
  head -c 160 gpurun_out/r02o_bench_$c.json; echo
done
timeout 600 python tools/profile_sweep.py --config c4 --sweeps 3 --tune 15=1 > gpurun_out/r02o_c4_fused.log 2>&1; tail -1 gpurun_out/r02o_c4_fused.log
