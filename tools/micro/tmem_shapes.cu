// Layout probe for the tcgen05.ld / tcgen05.st 16x256b and 16x128b shapes:
// TMEM is filled through 32x32b stores with code(lane, col) = lane * 1000 +
// col, then read back with 16x256b.x2 (from lane base 0 and 16 of each warp's
// quadrant) and printed per thread; a 16x128b.x1 store of thread codes is
// read back with 32x32b.  Results: profiles/r2_ab.md (session 3).
// Build + run (repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2503_15758_b200/csrc \
//     -o /tmp/tmem_shapes tools/micro/tmem_shapes.cu && /tmp/tmem_shapes
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace a2d;

__global__ void __launch_bounds__(128, 1) probe(float* out_ld, float* out_st) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    tmem_alloc(smem_u32(&slot), 64);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t qbase = tmem + (uint32_t(warp * 32) << 16);
  float v[32];
  for (int i = 0; i < 32; ++i) v[i] = float((warp * 32 + lane) * 1000 + i);
  tmem_st32(qbase, v);
  tmem_wait_st();
  // 16x256b.x2 from lane base 0: 8 registers per thread
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(qbase));
  tmem_wait_ld();
  for (int i = 0; i < 8; ++i) out_ld[threadIdx.x * 16 + i] = __uint_as_float(r[i]);
  // lane base 16 of the quadrant
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(qbase + (16u << 16)));
  tmem_wait_ld();
  for (int i = 0; i < 8; ++i) out_ld[threadIdx.x * 16 + 8 + i] = __uint_as_float(r[i]);
  // 16x128b.x1 store of thread codes into columns 32.. (2 registers per thread)
  const uint32_t a = __float_as_uint(float(threadIdx.x * 10 + 1)), b = __float_as_uint(float(threadIdx.x * 10 + 2));
  asm volatile("tcgen05.st.sync.aligned.16x128b.x1.b32 [%0], {%1, %2};" ::"r"(qbase + 32), "r"(a),
               "r"(b)
               : "memory");
  tmem_wait_st();
  tmem_ld32(qbase + 32, v);
  tmem_wait_ld();
  for (int i = 0; i < 8; ++i) out_st[threadIdx.x * 8 + i] = v[i];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

int main() {
  float *d_ld, *d_st;
  cudaMalloc(&d_ld, 128 * 16 * 4);
  cudaMalloc(&d_st, 128 * 8 * 4);
  probe<<<1, 128>>>(d_ld, d_st);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  float h_ld[128 * 16], h_st[128 * 8];
  cudaMemcpy(h_ld, d_ld, sizeof(h_ld), cudaMemcpyDeviceToHost);
  cudaMemcpy(h_st, d_st, sizeof(h_st), cudaMemcpyDeviceToHost);
  printf("16x256b.x2 (lane*1000+col), warp 1, per thread: base0 r0..7 | base16 r0..7\n");
  for (int t = 32; t < 64; ++t) {
    printf("t%02d:", t - 32);
    for (int i = 0; i < 16; ++i) printf(" %6.0f", h_ld[t * 16 + i]);
    printf("\n");
  }
  printf("16x128b.x1 store of (thread*10+1, thread*10+2), read by 32x32b: lane: cols 0..7\n");
  for (int l = 32; l < 64; ++l) {
    printf("lane%02d:", l - 32);
    for (int i = 0; i < 8; ++i) printf(" %5.0f", h_st[l * 8 + i]);
    printf("\n");
  }
  return 0;
}
