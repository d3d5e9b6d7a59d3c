# Round-1 final refresh: bench lines c1-c4 (DMMA headline + Ozaki alt), the reference arm at c4,
# the launch list of one c4 sweep and ncu --set full of one panel GEMM launch (one GPU).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in c4 c1 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/final2_bench_$c.json 2> gpurun_out/final2_bench_$c.err; echo bench_$c=$?
done
timeout 600 python bench.py --impl reference > gpurun_out/final2_bench_reference_c4.json 2> gpurun_out/final2_ref.err; echo ref=$?
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/final2_c4_launches.csv python tools/profile_sweep.py --config c4 > gpurun_out/final2_ncu1.log 2>&1; echo ncu1=$?
timeout 1200 $NCU --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:gemm_tma_kernel --launch-skip 6 -c 1 -o gpurun_out/final2_c4_panel -f \
  python tools/profile_sweep.py --config c4 > gpurun_out/final2_ncu2.log 2>&1; echo ncu2=$?
timeout 900 $NCU --set full --clock-control none --profile-from-start off \
  -k regex:power_gram_kernel -c 1 -o gpurun_out/final2_c2_power -f \
  python tools/profile_sweep.py --config c2 > gpurun_out/final2_ncu3.log 2>&1; echo ncu3=$?
