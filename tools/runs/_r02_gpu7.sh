# Round 2, GPU call 7: fused small-problem sweep kernel (p <= 1024): suite, c1 bench A/B, launch list + ncu of the kernel.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02j_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02j_pytest.log
timeout 600 python bench.py --config c1 > gpurun_out/r02j_bench_c1.json 2> gpurun_out/r02j_bench_c1.err; echo bench_c1=$?
head -c 300 gpurun_out/r02j_bench_c1.json; echo
for t in 1 0; do
  timeout 300 python tools/profile_sweep.py --config c1 --sweeps 6 --tune 14=$t > gpurun_out/r02j_c1_fused$t.log 2>&1; echo c1=$?
  tail -1 gpurun_out/r02j_c1_fused$t.log
done
NCU=/usr/local/cuda/bin/ncu
timeout 600 python tools/profile_sweep.py --config c1 --sweeps 2 > gpurun_out/r02j_c1_plain.log 2>&1 && \
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02j_c1_launches.csv python tools/profile_sweep.py --config c1 --sweeps 2 > gpurun_out/r02j_ncu1.log 2>&1; echo ncu1=$?
timeout 900 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:small_sweep -c 1 \
  -o gpurun_out/r02j_c1_small_sweep python tools/profile_sweep.py --config c1 --sweeps 2 > gpurun_out/r02j_ncu2.log 2>&1; echo ncu2=$?
python tools/launch_summary.py gpurun_out/r02j_c1_launches.csv 30 > gpurun_out/r02j_c1_launches.md; cat gpurun_out/r02j_c1_launches.md
