# Round 2, GPU call 4: potrs-style SPD inverse (back substitution instead of the L^-T L^-1 product):
# full GPU suite, c4 through the floor against the reference fixture, c4 bench (setup time), c5 first sweep.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02g_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02g_pytest.log
timeout 900 python tools/c4_long_compare.py > gpurun_out/r02g_c4long_compare.log 2>&1; echo c4long=$?
tail -12 gpurun_out/r02g_c4long_compare.log
IBMI_PHASE_TIMER=1 timeout 900 python bench.py --no-alt > gpurun_out/r02g_bench_c4.json 2> gpurun_out/r02g_bench_c4.err; echo bench=$?
head -c 400 gpurun_out/r02g_bench_c4.json
python tools/profile_setup.py > gpurun_out/r02g_setup.log 2>&1; tail -15 gpurun_out/r02g_setup.log
