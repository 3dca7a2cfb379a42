python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm_bf16" 2>&1 | tail -2
for T in 69 101 117 197; do TA_LIB=var/lib_trace.so T=$T LINES=400 python tools/attn_trace.py > gpurun_out/atr_$T.txt 2>&1; done
SHAPES="256,21,12,64;256,37,12,64;256,53,12,64;256,69,12,64;256,85,12,64;256,101,12,64;256,117,12,64;256,133,12,64;256,197,12,64" python tools/attn_bench.py 2>&1 | tail -30
