# Round 2, GPU call 13: flag-exchange power iteration with all polling rounds in flight: tests + c2/c3 A/B vs barrier.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_norm or c2_full or c3_full or spec or small_cases" > gpurun_out/r02p_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02p_pytest.log
for t in 1 0; do
  timeout 300 python tools/profile_sweep.py --config c2 --sweeps 6 --tune 13=$t > gpurun_out/r02p_c2_ll$t.log 2>&1
  echo "c2 key13=$t $(tail -1 gpurun_out/r02p_c2_ll$t.log)"
done
timeout 600 python bench.py --config c2 --no-alt > gpurun_out/r02p_bench_c2.json 2> gpurun_out/r02p_bench_c2.err; echo bench_c2=$?
head -c 200 gpurun_out/r02p_bench_c2.json; echo
