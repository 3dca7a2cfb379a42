python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -1
python -m pytest tests/test_gpu_attention_backends.py -q -x 2>&1 | tail -1
export SHAPES="256,69,12,64;256,117,12,64;256,133,12,64;256,165,12,64;256,181,12,64;256,197,12,64;512,165,16,80;256,181,16,64"
for i in 1 2; do
echo osep0; TA_ATTN_OSEP=0 python tools/attn_bench.py
echo osep1; python tools/attn_bench.py
done
