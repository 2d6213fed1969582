set -x
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none --csv --log-file gpurun_out/r02_band_launches_d.csv python tools/prof_band.py 1 > gpurun_out/r02_ncu_d.log 2>&1
tail -3 gpurun_out/r02_ncu_d.log
