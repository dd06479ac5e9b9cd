// Micro-benchmark: issue rate of MUFU.EX2 and of the packed FFMA2 / FADD2 /
// F2FP stream per SM sub-partition (one warp per sub-partition, 4 warps per
// CTA, one CTA per SM).  Build + run: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o /tmp/mufu_rate tools/micro/mufu_rate.cu && /tmp/mufu_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = 0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) {  // MUFU.EX2
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
        a[i] = y * 0.5f;
      } else if (MODE == 1) {  // fp32 FMA
        a[i] = fmaf(a[i], 0.999f, 0.001f);
      } else {  // packed FFMA2 on pairs
        float2 x = make_float2(a[i], a[(i + 1) & 15]);
        float2 r;
        asm volatile("{\n\t.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %3};\n\t"
                     "fma.rn.f32x2 rd, ra, ra, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
                     : "=f"(r.x), "=f"(r.y) : "f"(x.x), "f"(x.y));
        a[i] = r.x;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 4 + threadIdx.x / 32] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 128 * 4);
  cudaMalloc(&cyc, 148 * 4 * 8);
  long long h[148 * 4];
  const int iters = 4096;
  const char* names[3] = {"MUFU.EX2 (1 warp / SMSP)", "FFMA      (1 warp / SMSP)", "FFMA2     (1 warp / SMSP)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 128>>>(out, cyc, iters);
      if (mode == 1) k<1><<<148, 128>>>(out, cyc, iters);
      if (mode == 2) k<2><<<148, 128>>>(out, cyc, iters);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 148 * 4; ++i) mean += h[i];
    mean /= 148 * 4;
    printf("%s: %.2f cycles per warp instruction\n", names[mode], mean / (iters * 16.0));
  }
  return 0;
}
