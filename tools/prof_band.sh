# C4 band kernels: timing, then one ncu --set full capture of each sweep kernel
python tools/prof_band.py 5 > gpurun_out/band_time.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:band_psolve_bwd -s 1 -c 1 -f -o gpurun_out/band_bwd python tools/prof_band.py 1 > gpurun_out/ncu_band_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:band_psolve_fwd -s 1 -c 1 -f -o gpurun_out/band_fwd python tools/prof_band.py 1 > gpurun_out/ncu_band_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:band_correct2 -c 1 -f -o gpurun_out/band_corr python tools/prof_band.py 1 > gpurun_out/ncu_band_corr.log 2>&1
