S="256,117,12,64;256,197,12,64;256,261,12,64;256,325,12,64;256,389,12,64;512,257,16,80"
for i in 1 2; do
TA_LIB=var/lib_r02e.so SHAPES=$S python tools/attn_bench.py 2>&1 | sed 's/^/old /'
SHAPES=$S python tools/attn_bench.py 2>&1 | sed 's/^/new /'
done
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_attention_backends.py -q -x -k "attention or attn" 2>&1 | tail -2
