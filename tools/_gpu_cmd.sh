for c in c1 c2 c3 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo $c=$?
done
timeout 900 python bench.py --gemm ozaki --no-alt > gpurun_out/bench_c4_oz.log 2>&1; echo c4oz=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
