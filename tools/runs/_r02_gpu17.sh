# Round 2, GPU call 17: power-iteration kernels with tree sums / one division: suite + bench lines + c2/c1 iteration fits.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r03c_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r03c_pytest.log
for c in c2 c1 c3 c4; do
  timeout 1200 python bench.py --config $c > gpurun_out/r03c_bench_$c.json 2> gpurun_out/r03c_bench_$c.err; echo bench_$c=$?
  head -c 160 gpurun_out/r03c_bench_$c.json; echo
done
for t in 1 0; do
  timeout 300 python tools/profile_sweep.py --config c2 --sweeps 14 --tune 13=$t > gpurun_out/r03c_c2_ll$t.log 2>&1
  grep "power iterations" gpurun_out/r03c_c2_ll$t.log | tr '\n' ';'; echo
done
timeout 300 python tools/profile_sweep.py --config c3 --sweeps 6 > gpurun_out/r03c_c3.log 2>&1; grep "power iterations" gpurun_out/r03c_c3.log | tr '\n' ';'; echo
timeout 300 python tools/profile_sweep.py --config c1 --sweeps 6 > gpurun_out/r03c_c1.log 2>&1; grep "power iterations" gpurun_out/r03c_c1.log | tr '\n' ';'; echo
timeout 900 python tools/ll_determinism_stress.py 200 > gpurun_out/r03c_ll_stress.log 2>&1; tail -1 gpurun_out/r03c_ll_stress.log
