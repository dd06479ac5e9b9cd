// Micro-benchmark: cycles for the forward softmax's exponential block (one
// 128-column S row per thread: FFMA2 scale-and-subtract, exp2 on MUFU or the
// FMA-pipe cubic, FADD2 row sums, F2FP packing), one warp per SM
// sub-partition, for polynomial fractions 0, 1/8, 1/4, 1/2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_15758_b200/csrc \
//   -o /tmp/exps_rate tools/micro/exps_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace a2d;

template <int POLY>  // pairs on the polynomial: jj/2 % 8 < POLY
__global__ void k(float* out, long long* cyc, int iters, float m) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = 0.01f * ((threadIdx.x * 7 + i * 13) % 97);
  const float2 sc = make_float2(1.4427f, 1.4427f);
  uint32_t sink = 0;
  float tot = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    const float2 nb = make_float2(-m - it * 1e-7f, -m - it * 1e-7f);
    uint32_t pk[64];
#pragma unroll
    for (int jj = 0; jj < 128; jj += 2) {
      const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
      float2 e;
      if (((jj >> 1) & 7) < POLY) e = exp2_poly2(x);
      else e = make_float2(ex2(x.x), ex2(x.y));
      acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
      pk[jj / 2] = pack_bf16(e.x, e.y);
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) sink ^= pk[i];
    const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    tot += a.x + a.y;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot + __uint_as_float(sink & 0x3fffffff);
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 4 + threadIdx.x / 32] = t1 - t0;
}

template <int POLY>
double run(float* out, long long* cyc, int iters) {
  long long h[148 * 4];
  for (int rep = 0; rep < 2; ++rep) {
    k<POLY><<<148, 128>>>(out, cyc, iters, 0.5f);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148 * 4; ++i) mean += h[i];
  return mean / (148 * 4) / iters;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 128 * 4);
  cudaMalloc(&cyc, 148 * 4 * 8);
  const int iters = 512;
  printf("poly 0/8: %.0f cycles per 128-column row\n", run<0>(out, cyc, iters));
  printf("poly 1/8: %.0f cycles per 128-column row\n", run<1>(out, cyc, iters));
  printf("poly 2/8: %.0f cycles per 128-column row\n", run<2>(out, cyc, iters));
  printf("poly 4/8: %.0f cycles per 128-column row\n", run<4>(out, cyc, iters));
  return 0;
}
