python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -2
python -m pytest tests/test_gpu_attention_backends.py -q -x 2>&1 | tail -2
export SHAPES="256,197,12,64;256,181,12,64;256,165,12,64;256,149,12,64;256,133,12,64;256,189,12,64;256,141,12,64;512,233,16,80;256,197,16,64"
for i in 1 2; do
echo swap; python tools/attn_bench.py
echo noswap; TA_ATTN_QSWAP=0 python tools/attn_bench.py
done
