set -x
python -m pytest tests/test_gpu_band_spike.py tests/test_gpu_reference_pump.py -x -q > gpurun_out/r02_pytest_b.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_b.log
tail -5 gpurun_out/r02_pytest_b.log
python tools/prof_band.py 5 > gpurun_out/r02_band_time_b.txt 2>&1; cat gpurun_out/r02_band_time_b.txt
python tools/prof_lub.py > gpurun_out/r02_lub_b.txt 2>&1; tail -8 gpurun_out/r02_lub_b.txt
ncu --set full --import-source on --clock-control none -k regex:"band_psolve_fwd|band_psolve_bwd|band_correct_accumulate" -c 3 -o gpurun_out/r02_band_b python tools/prof_band.py 1 > gpurun_out/r02_ncu_b.log 2>&1
tail -3 gpurun_out/r02_ncu_b.log
