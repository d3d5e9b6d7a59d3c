# Round 2, first GPU call: full GPU suite with the new linalg/boundary tests, the
# sharded world-1 sweep timing + launch list (to find its overhead vs the graph path),
# and the single-GPU launch list of one c4 sweep for comparison.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02a_pytest.log
timeout 600 python tools/profile_sharded.py --config c4 > gpurun_out/r02a_sharded_times.log 2>&1; echo sh=$?
tail -5 gpurun_out/r02a_sharded_times.log
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02a_sharded_launches.csv python tools/profile_sharded.py --config c4 --sweeps 0 > gpurun_out/r02a_ncu1.log 2>&1; echo ncu1=$?
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02a_single_launches.csv python tools/profile_sweep.py --config c4 > gpurun_out/r02a_ncu2.log 2>&1; echo ncu2=$?
python tools/launch_summary.py gpurun_out/r02a_sharded_launches.csv > gpurun_out/r02a_sharded_launches.md
python tools/launch_summary.py gpurun_out/r02a_single_launches.csv > gpurun_out/r02a_single_launches.md
cat gpurun_out/r02a_sharded_launches.md gpurun_out/r02a_single_launches.md
