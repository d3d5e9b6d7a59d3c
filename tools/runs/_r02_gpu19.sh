# Round 2, GPU call 19: final tree: suite, smoke, bench lines c1-c4, c1 launch list + ncu of the fused kernel.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r03h_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r03h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03h_smoke.log 2>&1; echo smoke=$?
for c in c4 c1 c2 c3; do
  timeout 1200 python bench.py --config $c > gpurun_out/r03h_bench_$c.json 2> gpurun_out/r03h_bench_$c.err; echo bench_$c=$?
  head -c 160 gpurun_out/r03h_bench_$c.json; echo
done
IBMI_SS_TRACE=1 timeout 300 python tools/profile_sweep.py --config c1 --sweeps 3 > gpurun_out/r03h_c1_trace.log 2>&1; grep -E "phases" gpurun_out/r03h_c1_trace.log | tail -2
NCU=/usr/local/cuda/bin/ncu
timeout 600 python tools/profile_sweep.py --config c1 --sweeps 2 > gpurun_out/r03h_c1_plain.log 2>&1 && \
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r03h_c1_launches.csv python tools/profile_sweep.py --config c1 --sweeps 2 > gpurun_out/r03h_ncu1.log 2>&1; echo ncu1=$?
timeout 900 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:small_sweep -c 1 \
  -o gpurun_out/r03h_c1_small_sweep python tools/profile_sweep.py --config c1 --sweeps 2 > gpurun_out/r03h_ncu2.log 2>&1; echo ncu2=$?
