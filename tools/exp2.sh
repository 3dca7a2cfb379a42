nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/sfu_rate tools/micro/sfu_rate.cu && tools/micro/sfu_rate
echo pair; python tools/gemm_n768.py
echo single128; TA_GEMM_TINY_M=1000000 python tools/gemm_n768.py
