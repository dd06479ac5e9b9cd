// lse_merge.cu — bandwidth-bound kernels around the tile:
//   * k-way log-sum-exp merge of partial (O, LSE): attn_fix folded over the
//     partials of one query row (reference attention.py:194-214) fused with
//     finalize (attention.py:217-222).  Written in LSE form, which is the
//     same algebra with (m, n, d) = (lse, O, 1):
//         lse = log sum_c exp(lse_c);   O = sum_c exp(lse_c - lse) O_c
//   * delta = rowsum(dO * O): the backward's preprocessing
//     (numpy_backend.py:49, numba_backend.py:84-86);
//   * dq = scale * dq_acc: the backward's final scaling (numpy_backend.py:61).
// One warp per row, 16-byte vector loads, streaming cache hints.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include "kernels.h"

namespace a2d {
namespace {

constexpr int kMaxParts = 16;

// four fp32 -> four 16-bit outputs (A2D_BF16 or A2D_F16), round to nearest
__device__ __forceinline__ uint2 pack4(int dtype, float4 v) {
  uint2 u;
  if (dtype == A2D_F16) {
    __half2 lo = __floats2half2_rn(v.x, v.y), hi = __floats2half2_rn(v.z, v.w);
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
  } else {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
  }
  return u;
}

__device__ __forceinline__ float4 ld_stream_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// Every load of a row group is issued before the first use: the K partial
// LSEs (warp-uniform broadcast loads) and the K x RPW float4 slices of O are
// independent, so each lane keeps K*RPW 16-byte loads in flight instead of
// waiting on the LSE before touching O.
template <int K, int RPW>
__global__ void __launch_bounds__(256) lse_merge_kernel(
    const float* __restrict__ o_parts, const float* __restrict__ lse_parts, int k,
    long long pso, long long psl, long long rows, int h, long long rs, void* __restrict__ o_out,
    int out_dtype, long long out_rs, float* __restrict__ lse_out) {
  const long long row0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RPW;
  const int lane = threadIdx.x & 31;
  if (row0 >= rows) return;
  const int kk = K > 0 ? K : k;
  for (int e = lane * 4; e < h; e += 128) {
    float4 v[K > 0 ? K : kMaxParts][RPW];
    float l[K > 0 ? K : kMaxParts][RPW];
#pragma unroll
    for (int c = 0; c < (K > 0 ? K : kMaxParts); ++c) {
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const long long row = row0 + r;
        const bool ok = c < kk && row < rows;
        l[c][r] = ok ? __ldg(lse_parts + c * psl + row) : -INFINITY;
        v[c][r] = ok ? ld_stream_f4(o_parts + c * pso + row * rs + e) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const long long row = row0 + r;
      if (row >= rows) break;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < (K > 0 ? K : kMaxParts); ++c) mx = fmaxf(mx, l[c][r]);
      float tot = 0.f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int c = 0; c < (K > 0 ? K : kMaxParts); ++c) {
        // an empty partial (lse = -inf) contributes exactly nothing, whatever its O holds
        const float w = (mx == -INFINITY || l[c][r] == -INFINITY) ? 0.f : __expf(l[c][r] - mx);
        // products rounded before they are summed (no FMA contraction), so a
        // two-way merge is bitwise commutative like the reference's attn_fix
        // (test_attention.py:203-210)
        tot += w;
        if (w != 0.f) {
          acc.x = __fadd_rn(acc.x, __fmul_rn(w, v[c][r].x));
          acc.y = __fadd_rn(acc.y, __fmul_rn(w, v[c][r].y));
          acc.z = __fadd_rn(acc.z, __fmul_rn(w, v[c][r].z));
          acc.w = __fadd_rn(acc.w, __fmul_rn(w, v[c][r].w));
        }
      }
      const float inv = tot > 0.f ? 1.f / tot : 0.f;
      acc.x *= inv; acc.y *= inv; acc.z *= inv; acc.w *= inv;
      if (out_dtype == A2D_F32) {
        __stcs(reinterpret_cast<float4*>(reinterpret_cast<float*>(o_out) + row * out_rs + e), acc);
      } else {
        *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(o_out) + row * out_rs + e) =
            pack4(out_dtype, acc);
      }
      if (lane == 0 && e == 0) lse_out[row] = tot > 0.f ? mx + __logf(tot) : -INFINITY;
    }
  }
}

template <bool F16>
__device__ __forceinline__ float2 to_f2(uint32_t u) {
  if (F16) return __half22float2(*reinterpret_cast<const __half2*>(&u));
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
}

template <bool F16>
__global__ void __launch_bounds__(256) bwd_preprocess_kernel(
    const uint16_t* __restrict__ o, const uint16_t* __restrict__ dout,
    float* __restrict__ delta, long long o_sbh, long long o_srow, long long do_sbh,
    long long do_srow, int bh, int n, int h) {
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= (long long)bh * n) return;
  const int b = (int)(gw / n);
  const int r = (int)(gw - (long long)b * n);
  const uint16_t* po = o + b * o_sbh + (long long)r * o_srow;
  const uint16_t* pd = dout + b * do_sbh + (long long)r * do_srow;
  float acc = 0.f;
  for (int e = lane * 4; e < h; e += 128) {
    const uint2 uo = *reinterpret_cast<const uint2*>(po + e);
    const uint2 ud = *reinterpret_cast<const uint2*>(pd + e);
    const float2 o0 = to_f2<F16>(uo.x), o1 = to_f2<F16>(uo.y);
    const float2 d0 = to_f2<F16>(ud.x), d1 = to_f2<F16>(ud.y);
    acc += o0.x * d0.x + o0.y * d0.y + o1.x * d1.x + o1.y * d1.y;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) delta[gw] = acc;
}

__global__ void __launch_bounds__(256) bwd_finalize_kernel(const float* __restrict__ acc,
                                                           long long asbh, long long asrow,
                                                           void* __restrict__ dq, int out_dtype,
                                                           long long sbh, long long srow, int bh,
                                                           int n, int h, float scale) {
  const long long total4 = (long long)bh * n * h / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total4;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * 4;
    const int c = (int)(e % h);
    const long long rr = e / h;
    const int r = (int)(rr % n);
    const int b = (int)(rr / n);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);  // acc == nullptr: zero fill
    if (acc != nullptr) {
      v = *reinterpret_cast<const float4*>(acc + b * asbh + (long long)r * asrow + c);
      v.x *= scale; v.y *= scale; v.z *= scale; v.w *= scale;
    }
    const long long dst = b * sbh + (long long)r * srow + c;
    if (out_dtype == A2D_F32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(dq) + dst) = v;
    } else {
      *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(dq) + dst) = pack4(out_dtype, v);
    }
  }
}

}  // namespace

int launch_lse_merge(const float* o_parts, const float* lse_parts, int k_parts,
                     long long part_stride_o, long long part_stride_lse, long long rows, int h,
                     long long row_stride, void* o_out, int out_dtype, long long out_row_stride,
                     float* lse_out, cudaStream_t stream) {
  if (rows == 0) return A2D_OK;
  const int warps = 8;
  auto go = [&](auto kern, int rpw) {
    const long long blocks = (rows + warps * rpw - 1) / (warps * rpw);
    kern<<<(unsigned)blocks, warps * 32, 0, stream>>>(o_parts, lse_parts, k_parts, part_stride_o,
                                                     part_stride_lse, rows, h, row_stride, o_out,
                                                     out_dtype, out_row_stride, lse_out);
  };
  switch (k_parts) {
    case 1: go(lse_merge_kernel<1, 4>, 4); break;
    case 2: go(lse_merge_kernel<2, 4>, 4); break;
    case 3: go(lse_merge_kernel<3, 2>, 2); break;
    case 4: go(lse_merge_kernel<4, 2>, 2); break;
    case 8: go(lse_merge_kernel<8, 1>, 1); break;
    default: go(lse_merge_kernel<0, 1>, 1); break;
  }
  return check_launch("lse_merge_kernel");
}

int launch_bwd_preprocess(const void* o, const void* dout, float* delta, long long o_sbh,
                          long long o_srow, long long do_sbh, long long do_srow, int bh, int n,
                          int h, bool f16, cudaStream_t stream) {
  const long long rows = (long long)bh * n;
  if (rows == 0) return A2D_OK;
  const int warps = 8;
  const unsigned blocks = (unsigned)((rows + warps - 1) / warps);
  auto kern = f16 ? bwd_preprocess_kernel<true> : bwd_preprocess_kernel<false>;
  kern<<<blocks, warps * 32, 0, stream>>>(reinterpret_cast<const uint16_t*>(o),
                                          reinterpret_cast<const uint16_t*>(dout), delta, o_sbh,
                                          o_srow, do_sbh, do_srow, bh, n, h);
  return check_launch("bwd_preprocess_kernel");
}

int launch_bwd_finalize(const float* dq_acc, long long asbh, long long asrow, void* dq,
                        int out_dtype, long long sbh, long long srow, int bh, int n, int h,
                        float scale, cudaStream_t stream) {
  const long long total4 = (long long)bh * n * h / 4;
  if (total4 == 0) return A2D_OK;
  long long blocks = (total4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  bwd_finalize_kernel<<<(unsigned)blocks, 256, 0, stream>>>(dq_acc, asbh, asrow, dq, out_dtype,
                                                            sbh, srow, bh, n, h, scale);
  return check_launch("bwd_finalize_kernel");
}

}  // namespace a2d
