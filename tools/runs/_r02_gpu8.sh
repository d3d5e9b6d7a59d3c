# Round 2, GPU call 8: final-code suite + smoke, bench lines c1-c4 (warm-up context), c5 DMMA bench + Ozaki run.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02k_pytest.log 2>&1; echo pytest=$?
tail -4 gpurun_out/r02k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/r02k_smoke.log
for c in c4 c1 c2 c3; do
  timeout 1200 python bench.py --config $c > gpurun_out/r02k_bench_$c.json 2> gpurun_out/r02k_bench_$c.err; echo bench_$c=$?
  head -c 160 gpurun_out/r02k_bench_$c.json; echo
done
timeout 1500 python bench.py --config c5 --steps 2 --warmup 1 --no-alt > gpurun_out/r02k_bench_c5.json 2> gpurun_out/r02k_bench_c5.err; echo bench_c5=$?
head -c 400 gpurun_out/r02k_bench_c5.json; echo
timeout 900 python tools/run_c5.py 14 16 > gpurun_out/r02k_c5_ozaki.log 2>&1; echo c5oz=$?
tail -4 gpurun_out/r02k_c5_ozaki.log | cut -c1-200
