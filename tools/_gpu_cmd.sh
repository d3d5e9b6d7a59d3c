set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/reentry3_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/reentry3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/reentry3_smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/reentry3_smoke.log
timeout 900 python bench.py > gpurun_out/reentry3_bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/reentry3_bench.log | head -c 600
