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

template <int POLY, int NC = 128>  // pairs on the polynomial: jj/2 % 8 < POLY; NC columns per row
__global__ void k(float* out, long long* cyc, int iters, float m) {
  float s[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) s[i] = 0.01f * ((threadIdx.x * 7 + i * 13) % 97);
  const float2 sc = make_float2(1.4427f, 1.4427f);
  uint32_t sink = 0;
  float tot = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    const float2 nb = make_float2(-m - it * 1e-7f, -m - it * 1e-7f);
    uint32_t pk[NC / 2];
#pragma unroll
    for (int jj = 0; jj < NC; jj += 2) {
      const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
      float2 e;
      if (((jj >> 1) & 7) < POLY) e = exp2_poly2(x);
      else e = make_float2(ex2(x.x), ex2(x.y));
      acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
      pk[jj / 2] = pack_bf16(e.x, e.y);
    }
#pragma unroll
    for (int i = 0; i < NC / 2; ++i) sink ^= pk[i];
    const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    tot += a.x + a.y;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot + __uint_as_float(sink & 0x3fffffff);
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

// NC = 128: one warp per sub-partition, one 128-column row per thread;
// NC = 64: two warps per sub-partition, each row split over two threads
// (same elements per sub-partition per iteration)
template <int POLY, int NC = 128>
double run(float* out, long long* cyc, int iters) {
  constexpr int T = 128 * (128 / NC);
  long long h[148 * 8];
  for (int rep = 0; rep < 2; ++rep) {
    k<POLY, NC><<<148, T>>>(out, cyc, iters, 0.5f);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
  }
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < 148 * (T / 32); ++i) mean += h[i];
  return mean / (148 * (T / 32)) / iters;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&cyc, 148 * 8 * 8);
  const int iters = 512;
  printf("poly 0/8: %.0f cycles per 128-column row\n", run<0>(out, cyc, iters));
  printf("poly 1/8: %.0f cycles per 128-column row\n", run<1>(out, cyc, iters));
  printf("poly 2/8: %.0f cycles per 128-column row\n", run<2>(out, cyc, iters));
  printf("poly 4/8: %.0f cycles per 128-column row\n", run<4>(out, cyc, iters));
  printf("2 warps/SMSP x 64 columns, poly 0/8: %.0f cycles per iteration\n", run<0, 64>(out, cyc, iters));
  printf("2 warps/SMSP x 64 columns, poly 1/8: %.0f cycles per iteration\n", run<1, 64>(out, cyc, iters));
  printf("2 warps/SMSP x 64 columns, poly 2/8: %.0f cycles per iteration\n", run<2, 64>(out, cyc, iters));
  return 0;
}
