set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_a.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_gpu_a.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_a.json 2> gpurun_out/r02_bench_a.err
for t in c1 c2 c3; do python tools/trace_compare.py $t > gpurun_out/r02_trace_$t.txt 2>&1; done
timeout 2400 python tools/c5_full.py > gpurun_out/r02_c5_full.log 2>&1
tail -3 gpurun_out/r02_pytest_gpu_a.log; cat gpurun_out/r02_bench_a.json; tail -5 gpurun_out/r02_c5_full.log
