python -m pytest tests/test_gpu_kernels.py tests/test_gpu_attention_backends.py -q -x -k "attention or attn" 2>&1 | tail -2
S="256,69,12,64;256,85,12,64;256,101,12,64;256,117,12,64;256,128,12,64;256,197,12,64"
for i in 1 2; do
TA_ATTN_KV=2 SHAPES=$S python tools/attn_bench.py 2>&1 | sed 's/^/kv2 /'
SHAPES=$S python tools/attn_bench.py 2>&1 | sed 's/^/kv4 /'
done
TA_LIB=var/lib_trace.so T=69 LINES=400 python tools/attn_trace.py > gpurun_out/atr4_69.txt 2>&1
bash tools/ab_env.sh TA_ATTN_KV 2 4 2
