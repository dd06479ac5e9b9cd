// Micro-benchmark: issue rate of the packed half-precision exponentials
// (ex2.approx.f16x2 / ex2.approx.ftz.bf16x2) against MUFU.EX2 f32, and of the
// conversions a packed-exponential softmax needs (f32x2 -> f16x2 / bf16x2
// packs, f16 -> f32 unpacks), one warp per SM sub-partition.
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu16_rate
//   tools/micro/mufu16_rate.cu && /tmp/mufu16_rate
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  unsigned a[16];
  float f[16];
  for (int i = 0; i < 16; ++i) {
    f[i] = 0.001f * (threadIdx.x + i);
    a[i] = 0x3c003c00u + threadIdx.x + i;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) {  // f32 MUFU.EX2
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f[i]));
        f[i] = y;
      } else if (MODE == 1) {  // ex2.approx.f16x2
        unsigned y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
        a[i] = y;
      } else if (MODE == 2) {  // ex2.approx.ftz.bf16x2
        unsigned y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(a[i]));
        a[i] = y;
      } else if (MODE == 3) {  // f32x2 -> f16x2 pack
        unsigned y;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(f[i]), "f"(f[(i + 1) & 15]));
        f[i] = __uint_as_float(y);
      } else if (MODE == 4) {  // f32x2 -> bf16x2 pack
        unsigned y;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(f[i]), "f"(f[(i + 1) & 15]));
        f[i] = __uint_as_float(y);
      } else if (MODE == 6) {  // MUFU.EX2 and an independent bf16x2 pack per step
        float y;
        unsigned z;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f[i]));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(z) : "f"(__uint_as_float(a[i])), "f"(__uint_as_float(a[(i + 1) & 15])));
        f[i] = y;
        a[i] = z;
      } else if (MODE == 7) {  // MUFU.EX2 and an independent FFMA2 per step
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f[i]));
        float2 x = make_float2(__uint_as_float(a[i]), __uint_as_float(a[(i + 1) & 15]));
        float2 r;
        asm volatile("{\n\t.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %3};\n\t"
                     "fma.rn.f32x2 rd, ra, ra, ra;\n\tmov.b64 {%0, %1}, rd;\n\t}"
                     : "=f"(r.x), "=f"(r.y) : "f"(x.x), "f"(x.y));
        f[i] = y;
        a[i] = __float_as_uint(r.x);
      } else if (MODE == 5) {  // f16 -> f32 unpack (both halves)
        float lo, hi;
        asm volatile("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n\t}"
                     : "=f"(lo), "=f"(hi) : "r"(a[i]));
        a[i] = __float_as_uint(lo + hi);
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += f[i] + __uint_as_float(a[i]);
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
  const char* names[8] = {"ex2.approx.ftz.f32     ", "ex2.approx.f16x2       ", "ex2.approx.ftz.bf16x2  ",
                          "cvt.rn.f16x2.f32       ", "cvt.rn.bf16x2.f32      ", "cvt.f32.f16 x2 (+FADD) ",
                          "EX2 f32 + bf16x2 pack  ", "EX2 f32 + FFMA2         "};
  for (int mode = 0; mode < 8; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (mode) {
        case 0: k<0><<<148, 128>>>(out, cyc, iters); break;
        case 1: k<1><<<148, 128>>>(out, cyc, iters); break;
        case 2: k<2><<<148, 128>>>(out, cyc, iters); break;
        case 3: k<3><<<148, 128>>>(out, cyc, iters); break;
        case 4: k<4><<<148, 128>>>(out, cyc, iters); break;
        case 5: k<5><<<148, 128>>>(out, cyc, iters); break;
        case 6: k<6><<<148, 128>>>(out, cyc, iters); break;
        case 7: k<7><<<148, 128>>>(out, cyc, iters); break;
      }
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
