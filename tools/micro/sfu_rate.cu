// Throughput of ex2.approx.ftz.f32 (MUFU.EX2), fma.rn.f32x2 (FFMA2) and a mix, per SM, with W
// warps per SM and 8 independent chains per thread.  Prints ops/clk/SM.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

template <int kMode>
__global__ void rate(float* out, unsigned long long* clk, int iters) {
  float v[8];
  uint64_t w[8];
  for (int i = 0; i < 8; ++i) { v[i] = threadIdx.x * 1e-3f + i * 1e-4f; w[i] = (uint64_t)__float_as_uint(v[i]) | ((uint64_t)__float_as_uint(v[i] + 1.f) << 32); }
  const uint64_t a = 0x3f8000003f800000ull, b = 0x3c0000003c000000ull;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (kMode == 0) v[i] = ex2(v[i]) * -0.5f;       // MUFU + FMUL
      if (kMode == 1) w[i] = ffma2(w[i], a, b);        // FFMA2
      if (kMode == 2) { v[i] = ex2(v[i]) * -0.5f; w[i] = ffma2(w[i], a, b); w[i] = ffma2(w[i], a, b); }
      if (kMode == 3) {  // bf16x2 pack only (F2FP): which pipe, what rate
        uint32_t p; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(v[i]), "f"(v[(i + 1) & 7]));
        v[i] = __uint_as_float(p) * 1.0001f;
      }
      if (kMode == 5) {  // ex2.approx.f16x2: two exponentials per lane and instruction
        uint32_t h = __float_as_uint(v[i]), y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(h));
        v[i] = __uint_as_float(y ^ 0x80008000u);
      }
      if (kMode == 6) {  // the softmax chunk in f16: x = s c - m (FFMA2), cvt f16x2, ex2 f16x2, hmul2 weight
        const uint64_t x = ffma2(w[i], a, b);
        uint32_t h, y, z;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(__uint_as_float((uint32_t)(x >> 32))), "f"(__uint_as_float((uint32_t)x)));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(h));
        asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(z) : "r"(y), "r"(0x3c003c00u));
        w[i] = x ^ z;
      }
      if (kMode == 4) {  // ex2 + one pack per element pair
        v[i] = ex2(v[i]) * -0.5f;
        uint32_t p; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(v[i]), "f"(v[(i + 1) & 7]));
        w[i] ^= p;
      }
    }
  }
  const unsigned long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += v[i] + __uint_as_float((uint32_t)w[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int kMode>
void run(const char* name, int warps, float* d, unsigned long long* c) {
  const int iters = 4096;
  rate<kMode><<<148, warps * 32>>>(d, c, iters);
  rate<kMode><<<148, warps * 32>>>(d, c, iters);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  const double ops = (double)iters * 8 * warps * 32;
  printf("%-26s warps=%2d  %.2f thread-ops/clk/SM (%s)\n", name, warps, ops / avg, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* d; unsigned long long* c;
  cudaMalloc(&d, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  for (int w : {4, 8, 16}) run<0>("ex2 (+fmul)", w, d, c);
  for (int w : {4, 8, 16}) run<1>("ffma2 (pairs)", w, d, c);
  for (int w : {8, 16}) run<2>("mix ex2 + 2 ffma2", w, d, c);
  for (int w : {8, 16}) run<3>("bf16x2 pack (+fmul)", w, d, c);
  for (int w : {8, 16}) run<4>("ex2 + bf16x2 pack", w, d, c);
  for (int w : {4, 8, 16}) run<5>("ex2.f16x2 (instr)", w, d, c);
  for (int w : {8, 16}) run<6>("f16 chunk (pairs)", w, d, c);
  return 0;
}
