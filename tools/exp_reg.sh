python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py -q -x -k "gemm_bf16 or splitk or fusion" 2>&1 | tail -2
for L in var/lib_r02e.so paper_2401_05031_b200/libtokadapt_cuda.so; do
 for G in 0 -16; do
  TA_LIB=$L ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rg_$(basename $L .so)_$G.csv python tools/launch_list.py $G > /dev/null 2>&1
  echo "$L g=$G"; python tools/launch_table.py gpurun_out/rg_$(basename $L .so)_$G.csv > gpurun_out/rg_tab.txt; head -10 gpurun_out/rg_tab.txt
 done
done
