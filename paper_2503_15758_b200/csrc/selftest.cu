// selftest.cu — one-CTA tcgen05 GEMM used to pin the UMMA descriptor
// encodings (K-major and MN-major SWIZZLE_128B operands) on the device.
#include "sm100.cuh"
#include "kernels.h"

namespace a2d {
namespace {

constexpr int SLAB = 128 * 128;  // 128 rows x 128 B

// element (m, k) of a K-major SW128 operand with 128 rows per slab
__device__ __forceinline__ uint32_t kmajor_off(int m, int k) {
  return (k >> 6) * SLAB + m * 128 + ((((k & 63) >> 3) ^ (m & 7)) << 4) + (k & 7) * 2;
}
// element (k, n) of an MN-major SW128 operand with 128 k-rows per 64-wide atom
__device__ __forceinline__ uint32_t mnmajor_off(int k, int n) {
  return (n >> 6) * SLAB + k * 128 + ((((n & 63) >> 3) ^ (k & 7)) << 4) + (n & 7) * 2;
}

__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __nv_bfloat16* a, const __nv_bfloat16* b, float* d, int n, int b_mn) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sa = smem_u32(smem);
  const uint32_t sbb = sa + 2 * SLAB;
  const uint32_t sbar = sbb + 2 * SLAB;
  const uint32_t stm = sbar + 8;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) {
    const int m = i / 128, k = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(smem + kmajor_off(m, k)) = a[i];
  }
  for (int i = threadIdx.x; i < 128 * n; i += blockDim.x) {
    if (b_mn) {  // b given as [k][n]
      const int k = i / n, nn = i % n;
      *reinterpret_cast<__nv_bfloat16*>(smem + 2 * SLAB + mnmajor_off(k, nn)) = b[i];
    } else {     // b given as [n][k]
      const int nn = i / 128, k = i % 128;
      *reinterpret_cast<__nv_bfloat16*>(smem + 2 * SLAB + kmajor_off(nn, k)) = b[i];
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(sbar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) {
    tmem_alloc(stm, 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (stm - sa));
  const bool a_tmem = (b_mn & 2) != 0;
  b_mn &= 1;
  if (a_tmem) {
    // A row `row` -> TMEM lane `row`, columns [128, 192): bf16 pairs (2c, 2c+1) in column c
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c0 = 0; c0 < 64; c0 += 32) {
      float pk[32];
      for (int i = 0; i < 32; ++i) {
        const __nv_bfloat16 lo = a[row * 128 + 2 * (c0 + i)];
        const __nv_bfloat16 hi = a[row * 128 + 2 * (c0 + i) + 1];
        const uint32_t u = (uint32_t)__bfloat16_as_ushort(lo) |
                           ((uint32_t)__bfloat16_as_ushort(hi) << 16);
        pk[i] = __uint_as_float(u);
      }
      tmem_st32(tmem + (uint32_t(warp * 32) << 16) + 128 + c0, pk);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, n, 0, b_mn);
    for (int kk = 0; kk < 8; ++kk) {
      uint64_t bd;
      if (b_mn) bd = make_sdesc(sbb + kk * 2048, SLAB, 1024);
      else bd = make_sdesc(sbb + (kk >> 2) * SLAB + (kk & 3) * 32, 16, 1024);
      if (a_tmem) {
        umma_bf16_ts(tmem, tmem + 128 + kk * 8, bd, idesc, kk > 0);
      } else {
        const uint64_t ad = make_sdesc(sa + (kk >> 2) * SLAB + (kk & 3) * 32, 16, 1024);
        umma_bf16(tmem, ad, bd, idesc, kk > 0);
      }
    }
    umma_commit(sbar);
  }
  __syncwarp();
  mbar_wait(sbar, 0);
  tc_fence_after();
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c = 0; c < n; c += 32) {
    float v[32];
    tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) d[row * n + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace

int launch_selftest_umma(const void* a, const void* b, float* d, int n, int b_mn_major,
                         cudaStream_t stream) {
  const int smem = 4 * SLAB + 64 + 1024;
  cudaError_t e =
      cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(selftest)");
  selftest_kernel<<<1, 128, smem, stream>>>(reinterpret_cast<const __nv_bfloat16*>(a),
                                            reinterpret_cast<const __nv_bfloat16*>(b), d, n,
                                            b_mn_major);
  return check_launch("selftest_kernel");
}

namespace {

// tcgen05 issue-rate probe: one elected thread per CTA issues `iters` units
// of K=128 (8 x K16 MMAs) of one operand shape / majorness, back to back.
__global__ void __launch_bounds__(128, 1) umma_bench_kernel(int variant, int iters,
                                                            long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sa = smem_u32(smem);
  const uint32_t sbb = sa + 65536;
  const uint32_t sbar = sbb + 65536;
  const uint32_t stm = sbar + 8;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(sbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(stm, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (stm - sa));
  if (threadIdx.x == 0) {
    int N = 128, am = 0, bm = 0;
    switch (variant) {
      case 0: N = 128; break;
      case 1: N = 128; bm = 1; break;
      case 2: N = 64; break;
      case 3: N = 64; am = 1; bm = 1; break;
      case 4: N = 256; break;
      case 5: N = 128; am = 1; bm = 1; break;
      case 6: N = 64; bm = 1; break;
      case 7: N = 128; break;            // A from TMEM (TS)
      case 8: N = 128; bm = 1; break;    // TS, B MN-major
      case 9: N = 64; break;             // TS
      case 10: N = 256; break;           // TS
      default: N = 32; break;
    }
    const bool ts = variant >= 7 && variant <= 10;
    const uint32_t idesc = make_idesc_bf16(128, N, am, bm);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      ad[kk] = am ? make_sdesc(sa + kk * 2048, SLAB, 1024)
                  : make_sdesc(sa + (kk >> 2) * SLAB + (kk & 3) * 32, 16, 1024);
      bd[kk] = bm ? make_sdesc(sbb + kk * 2048, SLAB, 1024)
                  : make_sdesc(sbb + (kk >> 2) * (N * 128) + (kk & 3) * 32, 16, 1024);
    }
    const long long t0 = clock64();
    if (ts) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts(tmem + (it & 1) * 128, tmem + 384 + kk * 8, bd[kk], idesc, kk > 0);
      }
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tmem + (it & 1) * 256, ad[kk], bd[kk], idesc, kk > 0);
      }
    }
    umma_commit(sbar);
    mbar_wait(sbar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Fills shared memory and all 512 TMEM columns of every SM with NaN bit
// patterns, so a later kernel that consumes on-chip memory it never wrote
// shows up as NaNs instead of passing by luck (tests/test_gpu_tile.py).
__global__ void __launch_bounds__(128, 1) poison_kernel(int mode, int smem_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (mode & 1) {
    for (int i = threadIdx.x * 16; i < smem_bytes; i += blockDim.x * 16)
      *reinterpret_cast<uint4*>(smem + i) = make_uint4(0x7fc07fc0u, 0x7fc07fc0u, 0x7fc07fc0u, 0x7fc07fc0u);
  }
  __syncthreads();
  if (mode & 2) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
      tmem_alloc(smem_u32(&slot), 512);
      tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(0x7fc00000u);
    for (int c = 0; c < 512; c += 32) tmem_st32(tmem + (uint32_t(warp * 32) << 16) + c, v);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
      tc_fence_after();
      tmem_dealloc(tmem, 512);
    }
  }
}

}  // namespace

int launch_poison(int mode, int num_sms, cudaStream_t stream) {
  const int smem = 227 * 1024 - 1024;  // leaves room for the static TMEM slot
  cudaError_t e = cudaFuncSetAttribute(poison_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(poison)");
  poison_kernel<<<num_sms * 2, 128, smem, stream>>>(mode, smem);
  return check_launch("poison_kernel");
}

int launch_bench_umma(int variant, int iters, long long* out, int ctas, cudaStream_t stream) {
  const int smem = 2 * 65536 + 64 + 1024;
  cudaError_t e =
      cudaFuncSetAttribute(umma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(bench)");
  umma_bench_kernel<<<ctas, 128, smem, stream>>>(variant, iters, out);
  return check_launch("umma_bench_kernel");
}

}  // namespace a2d
