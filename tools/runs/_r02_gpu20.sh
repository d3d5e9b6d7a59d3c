# Round 2, GPU call 20: round-2 ncu evidence of the headline kernel: launch list of one c4 sweep and --set full of the panel GEMM.
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python tools/profile_sweep.py --config c4 --sweeps 1 > gpurun_out/r03l_c4_plain.log 2>&1 && \
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r03l_c4_launches.csv python tools/profile_sweep.py --config c4 --sweeps 1 > gpurun_out/r03l_ncu1.log 2>&1; echo ncu1=$?
timeout 1200 $NCU --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_tma -s 2 -c 1 \
  -o gpurun_out/r03l_c4_panel python tools/profile_sweep.py --config c4 --sweeps 1 > gpurun_out/r03l_ncu2.log 2>&1; echo ncu2=$?
python tools/launch_summary.py gpurun_out/r03l_c4_launches.csv > gpurun_out/r03l_c4_launches.md; head -12 gpurun_out/r03l_c4_launches.md
