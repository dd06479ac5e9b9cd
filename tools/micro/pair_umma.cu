// Micro-benchmark + layout probe for tcgen05 on CTA pairs (cta_group::2):
//   rate:   cycles per K=128 unit (8 x K16 MMAs, straight-line issue by one
//           thread) of cta_group::1 / ::2 shapes (SS and TS, N 64..256)
//   layout: D of one cta_group::2 M=128 N=128 MMA (A row codes / B column
//           codes) as seen by tcgen05.ld in each CTA of the pair
//   mixing: one cta_group::1 MMA per CTA after a cta_group::2 allocation
// Results: profiles/r2_ab.md ("Session 3").
// Build + run (repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2503_15758_b200/csrc \
//     -o /tmp/pair_umma tools/micro/pair_umma.cu -lcuda && /tmp/pair_umma
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace a2d;

namespace {
constexpr int SLAB = 128 * 128;

__device__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ void alloc2(uint32_t dst, uint32_t n) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(n) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ void dealloc2(uint32_t t, uint32_t n) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(n) : "memory");
}
__device__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b),
               "r"(id), "r"(acc) : "memory");
}
__device__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b),
               "r"(id), "r"(acc) : "memory");
}
__device__ void commit2(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
               " [%0], %1;" ::"r"(bar), "h"((uint16_t)3) : "memory");
}
__device__ uint32_t try_wait_cl(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ uint32_t kmajor_off(int m, int k) {
  return (k >> 6) * SLAB + m * 128 + ((((k & 63) >> 3) ^ (m & 7)) << 4) + (k & 7) * 2;
}

// mode >= 0: rate; mode == 10: layout probe (rows), 11: layout probe (cols), 12: mixing
template <bool G2, int M, int N, bool TS, bool TWO_D>
__global__ void __launch_bounds__(128, 1) k(int mode, int iters, long long* cyc, float* dump) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sa = smem_u32(smem), sbb = sa + 2 * SLAB, sbar = sbb + 2 * SLAB, stm = sbar + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  // A: 128 rows K-major; B: 128 rows ([n][k]) K-major
  for (int i = threadIdx.x; i < 128 * 128; i += 128) {
    const int m = i / 128, kk = i % 128;
    float av = 0.f, bv = 0.f;
    if (mode == 10 && kk == 0) { av = float(rank * 128 + m + 1); bv = 1.f; }
    if (mode == 11 && kk == 0) { av = 1.f; bv = float(rank * 128 + m + 1); }
    if (mode == 12 && kk == 0) { av = float(m + 1); bv = float(rank + 1); }
    if (mode < 10) { av = 1e-3f; bv = 1e-3f; }
    *reinterpret_cast<__nv_bfloat16*>(smem + kmajor_off(m, kk)) = __float2bfloat16(av);
    *reinterpret_cast<__nv_bfloat16*>(smem + 2 * SLAB + kmajor_off(m, kk)) = __float2bfloat16(bv);
  }
  if (threadIdx.x == 0) { mbar_init(sbar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  if (warp == 0) alloc2(stm, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (stm - sa));
  // TS operand: A rows in TMEM columns [384, 448)
  if (TS) {
    float pk[32];
    for (int i = 0; i < 32; ++i) pk[i] = __uint_as_float(0x3a833a83u);
    tmem_st32(tmem + (uint32_t(warp * 32) << 16) + 384, pk);
    tmem_st32(tmem + (uint32_t(warp * 32) << 16) + 416, pk);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
  }
  uint64_t ad[8], bd[8];
  for (int kk = 0; kk < 8; ++kk) {
    ad[kk] = make_sdesc(sa + (kk >> 2) * SLAB + (kk & 3) * 32, 16, 1024);
    bd[kk] = make_sdesc(sbb + (kk >> 2) * SLAB + (kk & 3) * 32, 16, 1024);
  }
  long long t0 = clock64();
  if (mode < 10 && threadIdx.x == 0 && (!G2 || rank == 0)) {
    const uint32_t id = make_idesc_bf16(M, N, 0, 0);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t d = TWO_D ? tmem + (kk & 1) * 256 : tmem + (it & 1) * 256;
        const uint32_t acc = TWO_D ? (it > 0 || kk > 1) : (kk > 0);
        if (G2 && TS) mma2_ts(d, tmem + 384 + kk * 8, bd[kk], id, acc);
        else if (G2) mma2(d, ad[kk], bd[kk], id, acc);
        else if (TS) umma_bf16_ts(d, tmem + 384 + kk * 8, bd[kk], id, acc);
        else umma_bf16(d, ad[kk], bd[kk], id, acc);
      }
    }
    if (G2) commit2(sbar);
    else umma_commit(sbar);
  }
  if (mode >= 10 && threadIdx.x == 0) {
    if (mode == 12) {  // each CTA: its own cta_group::1 MMA into columns [0,128)
      umma_bf16(tmem, ad[0], bd[0], make_idesc_bf16(128, 128, 0, 0), 0);
      umma_commit(sbar);
    } else if (rank == 0 && G2) {
      mma2(tmem, ad[0], bd[0], make_idesc_bf16(128, 128, 0, 0), 0);
      commit2(sbar);
    }
  }
  __syncwarp();
  if (mode == 0 || mode >= 12 || true) {
    if (threadIdx.x == 0 || mode >= 10) {
      if (!G2) { while (!mbar_try_wait(sbar, 0)) {} }
      else { while (!try_wait_cl(sbar, 0)) {} }
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_after();
  if (mode >= 10) {
    const int row = warp * 32 + lane;
    for (int c = 0; c < 128; c += 32) {
      float v[32];
      tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c, v);
      tmem_wait_ld();
      for (int i = 0; i < 32; ++i) dump[(blockIdx.x * 128 + row) * 128 + c + i] = v[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) { tc_fence_after(); dealloc2(tmem, 512); }
}
}  // namespace

using KFn = void (*)(int, int, long long*, float*);
struct Mode { const char* name; KFn fn; bool g2; };

int main() {
  const int smem = 4 * SLAB + 64;
  const Mode modes[] = {
      {"g1 M128 N128 SS", k<false, 128, 128, false, false>, false},
      {"g1 M128 N128 TS", k<false, 128, 128, true, false>, false},
      {"g1 M128 N128 SS 2D", k<false, 128, 128, false, true>, false},
      {"g2 M256 N128 SS", k<true, 256, 128, false, false>, true},
      {"g2 M256 N128 TS", k<true, 256, 128, true, false>, true},
      {"g2 M256 N256 SS", k<true, 256, 256, false, false>, true},
      {"g2 M256 N64 SS", k<true, 256, 64, false, false>, true},
      {"g2 M128 N128 SS", k<true, 128, 128, false, false>, true},
      {"g2 M256 N128 SS 2D", k<true, 256, 128, false, true>, true},
  };
  long long* cyc;
  float* dump;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&dump, 2 * 128 * 128 * sizeof(float));
  auto launch = [&](KFn fn, int mode, int iters, int ctas) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, mode, iters, cyc, dump);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return false; }
    return true;
  };
  const int iters = 2000;
  for (int ctas : {2, 148}) {
    for (const Mode& m : modes) {
      if (!launch(m.fn, 0, 10, ctas) || !launch(m.fn, 0, iters, ctas)) return 1;
      std::vector<long long> h(ctas);
      cudaMemcpy(h.data(), cyc, ctas * sizeof(long long), cudaMemcpyDeviceToHost);
      double s = 0; int n = 0;
      for (int i = 0; i < ctas; ++i) if (!m.g2 || i % 2 == 0) { s += h[i]; ++n; }
      printf("ctas=%3d %-20s %8.1f cycles per K=128 unit\n", ctas, m.name, s / n / iters);
    }
  }
  for (int mode = 10; mode <= 12; ++mode) {
    if (!launch(k<true, 128, 128, false, false>, mode, 1, 2)) return 1;
    std::vector<float> d(2 * 128 * 128);
    cudaMemcpy(d.data(), dump, d.size() * 4, cudaMemcpyDeviceToHost);
    printf("mode %d (%s)\n", mode, mode == 10 ? "row codes" : mode == 11 ? "column codes" : "mixing g1");
    for (int r = 0; r < 2; ++r) {
      printf(" CTA%d lane->col0:", r);
      for (int l = 0; l < 128; l += 8) printf(" %d:%g", l, d[(r * 128 + l) * 128]);
      printf("\n CTA%d lane0 cols:", r);
      for (int c = 0; c < 128; c += 8) printf(" %d:%g", c, d[(r * 128) * 128 + c]);
      printf("\n CTA%d lane64 cols:", r);
      for (int c = 0; c < 128; c += 8) printf(" %d:%g", c, d[(r * 128 + 64) * 128 + c]);
      printf("\n");
    }
  }
  return 0;
}
