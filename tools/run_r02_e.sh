set -x
ncu --set full --import-source on --clock-control none -k regex:"band_psolve_bwd_t4" -s 2 -c 1 -o gpurun_out/r02_bwdt4_e python tools/prof_band.py 1 > gpurun_out/r02_ncu_e.log 2>&1
tail -3 gpurun_out/r02_ncu_e.log
