set -x
mkdir -p gpurun_out
for c in c4 c3 c2; do
  for t in 1 0; do
    timeout 300 python tools/profile_setup.py --config $c --tune 16=$t > gpurun_out/r02r_setup_${c}_prio$t.log 2>&1
    echo "$c key16=$t: $(grep setup gpurun_out/r02r_setup_${c}_prio$t.log | tr '\n' ';')"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not c5" > gpurun_out/r02r_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/r02r_pytest.log
