# Round 2, GPU call 18: lagged-evaluation flag-exchange power iteration (ibmi_tune key 16): tests + c2/c3 A/B + stress.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -m gpu -x -q -k "two_norm or c2_ or c3_ or spec or analysis or condition" > gpurun_out/r03d_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r03d_pytest.log
for t in 1 0; do
  timeout 300 python tools/profile_sweep.py --config c2 --sweeps 14 --tune 16=$t > gpurun_out/r03d_c2_lazy$t.log 2>&1
  echo "key16=$t: $(grep 'power iterations' gpurun_out/r03d_c2_lazy$t.log | tr '\n' ';')"
done
for t in 1 0; do
  timeout 300 python tools/profile_sweep.py --config c3 --sweeps 6 --tune 16=$t > gpurun_out/r03d_c3_lazy$t.log 2>&1
  echo "c3 key16=$t: $(grep 'power iterations' gpurun_out/r03d_c3_lazy$t.log | tr '\n' ';')"
done
timeout 900 python tools/ll_determinism_stress.py 200 > gpurun_out/r03d_ll_stress.log 2>&1; tail -7 gpurun_out/r03d_ll_stress.log | grep -v Warning | grep -v two_norm
