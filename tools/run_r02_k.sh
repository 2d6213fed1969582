set -x
python -m pytest tests/test_gpu_sparse.py -x -q > gpurun_out/r02_pytest_k.log 2>&1; tail -2 gpurun_out/r02_pytest_k.log
bash tools/prof_round2.sh > gpurun_out/r02_prof_round2.log 2>&1
tail -3 gpurun_out/r02_prof_round2.log
