set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/r02c_smoke.log
timeout 900 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo bench=$?
head -c 1500 gpurun_out/r02c_bench.json
