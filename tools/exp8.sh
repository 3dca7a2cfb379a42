python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -2
python -m pytest tests/test_gpu_forward.py -q -x 2>&1 | tail -2
for mode in tma ldg; do
TA_GEMM_RESID=$mode ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$mode.csv python tools/launch_list.py -8 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/ll_$mode.csv > gpurun_out/ll_$mode.txt; echo $mode; head -8 gpurun_out/ll_$mode.txt
TA_GEMM_RESID=$mode ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll0_$mode.csv python tools/launch_list.py 0 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/ll0_$mode.csv > gpurun_out/ll0_$mode.txt; echo $mode g0; head -8 gpurun_out/ll0_$mode.txt
done
