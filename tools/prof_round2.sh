# Round-2 evidence (one B200): per-config timelines, band / LU timings, the bench
# command's ncu launch list, LU DRAM traffic, and one ncu --set full capture per
# hot kernel (read back here with tools/ncu_brief.py -> profiles/r02_*).
set -x
O=gpurun_out
for c in c1 c2 c3 c4; do python tools/trace_step.py $c > $O/r02_final_trace_$c.txt 2>&1; done
python tools/prof_band.py 5 > $O/r02_final_band_time.txt 2>&1
python tools/prof_lub.py 4096 8 3 > $O/r02_final_lub.txt 2>&1
python tools/prof_lub.py 8192 16 2 >> $O/r02_final_lub.txt 2>&1
python tools/prof_lub.py 4096 1 3 >> $O/r02_final_lub.txt 2>&1
python tools/prof_reduced.py > $O/r02_final_reduced.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $O/r02_final_lu_metrics.csv python tools/prof_lub.py 4096 8 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_final_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
R=/tmp/fb_ncu; mkdir -p $R   # reports stay on the box (large); only the briefs come back
NCU="ncu --set full --clock-control none --import-source on -f"
$NCU -k regex:zgemm_tma -s 10 -c 1 -o $R/zgemm_trailing python tools/prof_lub.py 4096 8 1 > /dev/null 2>&1
$NCU -k regex:sweep_kernel -c 1 -o $R/sweep python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-banded > /dev/null 2>&1
$NCU -k regex:panel_cluster -s 40 -c 1 -o $R/panel python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-banded > /dev/null 2>&1
$NCU -k regex:block_solve_kernel -s 3 -c 1 -o $R/block_solve python tools/soak_blocked_sweeps.py 6144 4 160 1 > /dev/null 2>&1
$NCU --kernel-name-base demangled -k 'regex:zgemm_tma_kernel<.bool.1, .int.64>' -s 3 -c 1 -o $R/zgemm_adjoint python tools/soak_blocked_sweeps.py 6144 4 152 1 > /dev/null 2>&1
$NCU --kernel-name-base demangled -k 'regex:zgemm_tma_kernel<.bool.0, .int.32>' -s 3 -c 1 -o $R/zgemm_tail32 python tools/soak_blocked_sweeps.py 6144 4 152 1 > /dev/null 2>&1
$NCU -k regex:band_psolve_fwd -s 2 -c 1 -o $R/band_fwd python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:band_psolve_bwd_t4 -s 2 -c 1 -o $R/band_bwd python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:band_correct_accumulate -s 1 -c 1 -o $R/band_fused python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:band_rsolve -c 1 -o $R/band_rsolve python tools/prof_band.py 1 > /dev/null 2>&1
$NCU -k regex:band_matvec -c 1 -o $R/band_matvec python tools/prof_band.py 1 > /dev/null 2>&1
for k in zgemm_trailing zgemm_adjoint zgemm_tail32 block_solve sweep panel band_fwd band_bwd band_fused band_rsolve band_matvec; do
  echo "## $k"; python tools/ncu_brief.py $R/$k.ncu-rep; python tools/ncu_opmix.py $R/$k.ncu-rep
done > $O/r02_ncu_final_kernels.txt 2>&1
ls -la $O/r02_final_* $O/r02_ncu_final_kernels.txt
