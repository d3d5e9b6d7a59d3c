# Round 2, GPU call 5: suite + smoke on the potrs-style inverse and c4 tol 1e-7; bench lines c4 (headline) and
# c1-c3; cuBLAS DGEMM yardstick; ncu launch list of one c2 sweep and --set full of the flag-exchange power kernel.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02h_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/r02h_smoke.log
timeout 1200 python bench.py > gpurun_out/r02h_bench_c4.json 2> gpurun_out/r02h_bench_c4.err; echo bench=$?
head -c 300 gpurun_out/r02h_bench_c4.json
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/r02h_bench_$c.json 2> gpurun_out/r02h_bench_$c.err; echo bench_$c=$?
  head -c 200 gpurun_out/r02h_bench_$c.json; echo
done
timeout 300 python tools/dgemm_probe.py > gpurun_out/r02h_dgemm_probe.log 2>&1; cat gpurun_out/r02h_dgemm_probe.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 python tools/profile_sweep.py --config c2 --sweeps 2 > gpurun_out/r02h_c2_plain.log 2>&1 && \
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02h_c2_launches.csv python tools/profile_sweep.py --config c2 --sweeps 2 > gpurun_out/r02h_ncu1.log 2>&1; echo ncu1=$?
timeout 900 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:power_gram_ll -c 1 \
  -o gpurun_out/r02h_c2_power_ll python tools/profile_sweep.py --config c2 --sweeps 2 > gpurun_out/r02h_ncu2.log 2>&1; echo ncu2=$?
python tools/launch_summary.py gpurun_out/r02h_c2_launches.csv > gpurun_out/r02h_c2_launches.md; cat gpurun_out/r02h_c2_launches.md
ls -la gpurun_out/*.ncu-rep
