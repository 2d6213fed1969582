# Round-end evidence: per-config timelines, band/reduced timings, LU DRAM traffic
# and one ncu --set full capture per hot kernel (read back with tools/ncu_brief.py).
set -x
for c in c1 c2 c3 c4; do python tools/trace_step.py $c > gpurun_out/final_trace_$c.txt 2>&1; done
python tools/prof_band.py 5 > gpurun_out/final_band_time.txt 2>&1
python tools/prof_reduced.py > gpurun_out/final_reduced.txt 2>&1
python tools/prof_gemm.py > gpurun_out/final_gemm.txt 2>&1
python tools/prof_lub.py 4096 8 3 > gpurun_out/final_lub.txt 2>&1
python tools/prof_lub.py 8192 16 2 >> gpurun_out/final_lub.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/final_lu_metrics.csv python tools/prof_lub.py 4096 8 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on -f"
$NCU -k regex:zgemm_fast -c 1 -o gpurun_out/final_zgemm_trailing python tools/prof_lub.py 4096 8 1 > /dev/null 2>&1
$NCU -k regex:sweep_kernel -c 1 -o gpurun_out/final_sweep python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
$NCU -k regex:panel_cluster -s 40 -c 1 -o gpurun_out/final_panel python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
$NCU -k regex:reduced_cluster -c 1 -o gpurun_out/final_reduced python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
$NCU -k regex:band_psolve_fwd -s 2 -c 1 -o gpurun_out/final_band_fwd python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:band_psolve_bwd -s 2 -c 1 -o gpurun_out/final_band_bwd python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:zgemm_fast -c 1 -o gpurun_out/final_band_correct python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:accumulate_terms -c 1 -o gpurun_out/final_accumulate python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:band_matvec -c 1 -o gpurun_out/final_band_matvec python tools/prof_band.py 1 > /dev/null 2>&1
ls gpurun_out/final_*
