timeout 900 python bench.py --gemm ozaki --no-alt > gpurun_out/bench_c4_oz.log 2>&1; echo c4oz=$?
tail -1 gpurun_out/bench_c4_oz.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['int8_peak_tops_measured'], d['roofline'])"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"igemm_tc2|oz_crt|oz_update|oz_split" -c 5 -o gpurun_out/oz_full4 python tools/ozaki_probe.py profile:c4:16 > gpurun_out/ncu_oz_full.log 2>&1; echo ncufull=$?
