# Round 2, GPU call 3: full GPU suite (operand-sharded mode, flag-exchange power iteration,
# sym_rows kernel), c4 through the floor vs the reference fixture, c2 power-iteration A/B,
# sharded world-1 timings in both operand modes, panel-GEMM DRAM traffic per config.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02d_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02d_pytest.log
timeout 900 python tools/c4_long_compare.py > gpurun_out/r02d_c4long_compare.log 2>&1; echo c4long=$?
tail -32 gpurun_out/r02d_c4long_compare.log
for t in 1 0; do
  timeout 300 python tools/profile_sweep.py --config c2 --sweeps 6 --tune 13=$t > gpurun_out/r02d_c2_power_ll$t.log 2>&1; echo c2=$?
  tail -1 gpurun_out/r02d_c2_power_ll$t.log
  timeout 300 python tools/profile_sweep.py --config c3 --sweeps 6 --tune 13=$t > gpurun_out/r02d_c3_power_ll$t.log 2>&1
  tail -1 gpurun_out/r02d_c3_power_ll$t.log
done
timeout 600 python bench.py --config c2 --no-alt > gpurun_out/r02d_bench_c2.json 2> gpurun_out/r02d_bench_c2.err; echo bench_c2=$?
head -c 600 gpurun_out/r02d_bench_c2.json
for o in replicated sharded; do
  timeout 600 python tools/profile_sharded.py --config c4 --operands $o > gpurun_out/r02d_sharded_n1_$o.log 2>&1; echo sh=$?
  tail -4 gpurun_out/r02d_sharded_n1_$o.log
done
NCU=/usr/local/cuda/bin/ncu
for c in c1 c2 c3 c4; do
  timeout 900 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --profile-from-start off -k regex:gemm_tma --csv --log-file gpurun_out/r02d_traffic_$c.csv \
    python tools/profile_sweep.py --config $c > gpurun_out/r02d_traffic_$c.log 2>&1; echo ncu_$c=$?
done
python tools/panel_traffic.py c1=gpurun_out/r02d_traffic_c1.csv c2=gpurun_out/r02d_traffic_c2.csv \
  c3=gpurun_out/r02d_traffic_c3.csv c4=gpurun_out/r02d_traffic_c4.csv > gpurun_out/r02d_panel_traffic.json; echo traffic=$?
cat gpurun_out/r02d_panel_traffic.json | head -40
timeout 1200 python tools/c4_floor_probe.py c4 30 > gpurun_out/r02d_c4_floor_probe.log 2>&1; echo probe=$?
cat gpurun_out/r02d_c4_floor_probe.log
