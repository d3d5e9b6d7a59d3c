set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_linalg.py tests/test_gpu_sharded.py tests/test_bench_contract.py -m gpu -x -q > gpurun_out/r02b_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02b_pytest.log
timeout 600 python tools/profile_sharded.py --config c4 > gpurun_out/r02b_sharded_times.log 2>&1; echo sh=$?
tail -4 gpurun_out/r02b_sharded_times.log
timeout 600 python tools/profile_sharded.py --config c4 --exchange p2p > gpurun_out/r02b_sharded_times_p2p.log 2>&1; echo sh=$?
tail -4 gpurun_out/r02b_sharded_times_p2p.log
