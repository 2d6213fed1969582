set -x
python tools/trace_step.py c2 > gpurun_out/trace_c2.txt 2>&1
python tools/trace_step.py c3 > gpurun_out/trace_c3.txt 2>&1
python tools/prof_gemm.py > gpurun_out/gemm.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -f -o gpurun_out/zgemm_k128 python tools/prof_gemm.py > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -f -o gpurun_out/sweep_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_cluster -s 40 -c 1 -f -o gpurun_out/panel_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_panel.log 2>&1
ls -la gpurun_out
