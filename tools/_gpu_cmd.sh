timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q -k overflow > gpurun_out/oz_overflow.log 2>&1; echo tests=$?; tail -2 gpurun_out/oz_overflow.log
for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo $c=$?
done
timeout 900 python bench.py --gemm ozaki --no-alt > gpurun_out/bench_c4_oz.log 2>&1; echo c4oz=$?
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/oz_launches.csv python tools/ozaki_probe.py profile:c4:16 > gpurun_out/ncu_oz.log 2>&1; echo ncu=$?
