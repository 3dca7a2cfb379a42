# Profiling build: the library with the attention clock64 trace (-DTA_ATTN_TRACE) into var/.
set -e
cd "$(dirname "$0")/../paper_2401_05031_b200/csrc"
mkdir -p ../../var/trace_build
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for s in gemm rowops tome attention attention_tc attention_tp attention_fa match_tc forward; do
  /usr/local/cuda/bin/nvcc $F -DTA_ATTN_TRACE ${EXTRA} -c $s.cu -o ../../var/trace_build/$s.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../var/lib_trace.so ../../var/trace_build/*.o
