set -x
mkdir -p gpurun_out
for t in 1 0; do
  timeout 300 python tools/profile_sweep.py --config c2 --sweeps 14 --tune 13=$t > gpurun_out/r02q_c2_ll$t.log 2>&1
  grep "power iterations" gpurun_out/r02q_c2_ll$t.log | tr '\n' ';'; echo
done
timeout 300 python tools/profile_sweep.py --config c3 --sweeps 6 > gpurun_out/r02q_c3.log 2>&1; grep "power iterations" gpurun_out/r02q_c3.log | tr '\n' ';'; echo
timeout 300 python tools/profile_sweep.py --config c1 --sweeps 6 > gpurun_out/r02q_c1.log 2>&1; grep "power iterations" gpurun_out/r02q_c1.log | tr '\n' ';'; echo
