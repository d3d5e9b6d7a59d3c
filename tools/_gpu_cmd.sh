timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('alt') or {}; print(d['value'], d['e2e'], d['roofline'], d['time_to_tol']); print(a.get('value'), a.get('sigma_rel_fro_vs_headline'), a.get('roofline'), a.get('time_to_tol'), a.get('kernel_ms_per_sweep'))"
timeout 900 python bench.py --gemm ozaki --no-alt > gpurun_out/bench_c4_oz.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_c4_oz.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['roofline'], d['time_to_tol'], d['kernel_ms_per_sweep'])"
