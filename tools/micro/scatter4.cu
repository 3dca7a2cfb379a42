// TMA tile::scatter4 semantics check (sm_100a): a 32-row x 128-byte SW128 staging box (the GEMM
// epilogue's layout) stored as 8 scatter4 instructions to arbitrary destination rows.  Tries the
// tensor map with box {32, 1} and {32, 4}; prints which destination rows hold which source row.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k(const __grid_constant__ CUtensorMap tm, const int* rows) {
  __shared__ __align__(1024) float box[32 * 32];
  const int r = threadIdx.x;  // thread = row
  for (int j = 0; j < 8; ++j) {  // 16-byte chunk j of row r at (j ^ (r & 7))
    float4 v = make_float4(r * 100 + 4 * j, r * 100 + 4 * j + 1, r * 100 + 4 * j + 2, r * 100 + 4 * j + 3);
    *reinterpret_cast<float4*>(reinterpret_cast<char*>(box) + r * 128 + ((j ^ (r & 7)) << 4)) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (r == 0) {
    for (int g = 0; g < 8; ++g) {
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];"
                   :: "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(reinterpret_cast<char*>(box) + g * 512)),
                      "r"(0), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3]) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const int R = 80;
  float* out; int* rows;
  cudaMalloc(&out, R * 32 * 4); cudaMalloc(&rows, 32 * 4);
  int h_rows[32];
  for (int i = 0; i < 32; ++i) h_rows[i] = (i * 37 + 5) % 64;  // a permutation into 64 rows
  h_rows[31] = 1000;  // out of bounds: must be dropped
  cudaMemcpy(rows, h_rows, sizeof(h_rows), cudaMemcpyHostToDevice);
  for (int bh : {1, 4}) {
    cudaMemset(out, 0, R * 32 * 4);
    CUtensorMap tm;
    cuuint64_t dims[2] = {32, (cuuint64_t)R};
    cuuint64_t strides[1] = {32 * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)bh};
    cuuint32_t es[2] = {1, 1};
    CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) { printf("box {32,%d}: encode failed %d\n", bh, (int)rc); continue; }
    k<<<1, 32>>>(tm, rows);
    cudaError_t e = cudaDeviceSynchronize();
    float h[R * 32];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    int ok = 0, bad = 0;
    for (int i = 0; i < 31; ++i) {
      const int d = h_rows[i];
      bool good = true;
      for (int c = 0; c < 32; ++c) good &= h[d * 32 + c] == i * 100 + c;
      ok += good; bad += !good;
      if (!good && bad < 4) printf("  src row %d -> dst %d: got %g %g %g ...\n", i, d, h[d * 32], h[d * 32 + 1], h[d * 32 + 4]);
    }
    int stray = 0;
    for (int d = 64; d < R; ++d) for (int c = 0; c < 32; ++c) stray += h[d * 32 + c] != 0.f;
    printf("box {32,%d}: %s, %d rows ok, %d bad, stray writes past 64: %d\n", bh, cudaGetErrorString(e), ok, bad, stray);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
