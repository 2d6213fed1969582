set -x
python -m pytest tests/test_gpu_band_spike.py tests/test_gpu_drivers.py -x -q > gpurun_out/r02_pytest_c.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_c.log
tail -5 gpurun_out/r02_pytest_c.log
python tools/prof_band.py 5 > gpurun_out/r02_band_time_c.txt 2>&1; cat gpurun_out/r02_band_time_c.txt
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r02_band_launches_c.csv python tools/prof_band.py 1 > gpurun_out/r02_ncu_c.log 2>&1
