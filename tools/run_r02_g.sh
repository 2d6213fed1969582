set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_g.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_gpu_g.log
tail -4 gpurun_out/r02_pytest_gpu_g.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_g.json 2> gpurun_out/r02_bench_g.err; tail -2 gpurun_out/r02_bench_g.err; cut -c1-600 gpurun_out/r02_bench_g.json
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-banded > gpurun_out/r02_bench_g2.json 2> gpurun_out/r02_bench_g2.err; cut -c1-700 gpurun_out/r02_bench_g2.json
python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-banded > gpurun_out/r02_bench_c3_g.json 2> gpurun_out/r02_bench_c3_g.err; cut -c1-900 gpurun_out/r02_bench_c3_g.json; tail -2 gpurun_out/r02_bench_c3_g.err
python bench.py --config c1 --steps 3 --warmup 2 --no-cpu-baseline --no-banded > gpurun_out/r02_bench_c1_g.json 2> gpurun_out/r02_bench_c1_g.err; cut -c1-900 gpurun_out/r02_bench_c1_g.json
python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_bench_c4_g.json 2> gpurun_out/r02_bench_c4_g.err; cut -c1-900 gpurun_out/r02_bench_c4_g.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_g.txt 2>&1; tail -2 gpurun_out/r02_smoke_g.txt
python tools/soak_blocked_sweeps.py 6144 4 256 12 > gpurun_out/r02_blocked_sweeps_soak.txt 2>&1; python tools/soak_blocked_sweeps.py 8192 8 152 6 >> gpurun_out/r02_blocked_sweeps_soak.txt 2>&1; cat gpurun_out/r02_blocked_sweeps_soak.txt
python tools/trace_step.py c3 > gpurun_out/r02_final_trace_c3.txt 2>&1; head -12 gpurun_out/r02_final_trace_c3.txt
