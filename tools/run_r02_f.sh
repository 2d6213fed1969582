set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_f.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_gpu_f.log
tail -4 gpurun_out/r02_pytest_gpu_f.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_f.json 2> gpurun_out/r02_bench_f.err; tail -2 gpurun_out/r02_bench_f.err; cut -c1-3000 gpurun_out/r02_bench_f.json
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r02_bench_ref_f.json 2> gpurun_out/r02_bench_ref_f.err; cut -c1-1200 gpurun_out/r02_bench_ref_f.json
python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_bench_c4_f.json 2> gpurun_out/r02_bench_c4_f.err; cut -c1-1500 gpurun_out/r02_bench_c4_f.json; tail -2 gpurun_out/r02_bench_c4_f.err
python tools/shipped_c1.py > gpurun_out/r02_shipped_c1.json 2> gpurun_out/r02_shipped_c1.err; cat gpurun_out/r02_shipped_c1.json
