# Round 2, GPU call 16: final validation of the committed tree: GPU suite, smoke, default bench, reference arm (short).
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02s_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02s_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/r02s_smoke.log
timeout 1200 python bench.py > gpurun_out/r02s_bench_c4.json 2> gpurun_out/r02s_bench_c4.err; echo bench=$?
head -c 200 gpurun_out/r02s_bench_c4.json; echo
timeout 1200 python bench.py --sharded --no-alt > gpurun_out/r02s_bench_c4_sharded.json 2> gpurun_out/r02s_bench_c4_sharded.err; echo bench_sharded=$?
head -c 200 gpurun_out/r02s_bench_c4_sharded.json; echo
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02s_bench_reference_c4.json 2> gpurun_out/r02s_bench_reference_c4.err; echo bench_ref=$?
head -c 300 gpurun_out/r02s_bench_reference_c4.json; echo
