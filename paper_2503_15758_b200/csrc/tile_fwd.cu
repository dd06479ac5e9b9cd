// tile_fwd.cu — Attention2D tile forward on sm_100a.
//
// Computes, for one (query tile of 128 rows, head) per CTA, the streaming
// softmax recurrence of the reference's flash_forward
// (pkg/src/attn2d/kernels/numpy_backend.py:24-43, numba_backend.py:38-76):
// S = scale Q K^T over key tiles of 128, running max / denominator, O += P V,
// causal masking by global token index, rows that see nothing stay empty.
// It emits the partial state (O normalised, LSE) that the k-way merge
// (lse_merge.cu) folds across the grid, exactly as attn_fix does
// (attention.py:194-214).
//
// Warp roles (192 threads, one CTA per SM):
//   warp 0     TMA producer: Q once, then K/V tiles into 2-stage rings
//   warp 1     tcgen05 MMA issuer (one elected lane) + TMEM owner
//   warps 2-5  softmax warpgroup: one query row per thread (= TMEM lane)
// TMEM (512 columns): S double buffer at [0,128) and [128,256), O at 256.
// S_{j+1} = Q K_{j+1}^T runs on the tensor pipe while the softmax
// warpgroup turns S_j into P_j; P_j goes to shared memory (bf16, 128B
// swizzle, K-major) and O += P_j V_j is issued as soon as it lands.
// The running max is only moved when it grows by more than 2^8 (log2
// domain), so O in TMEM is rarely rescaled; the final normalisation uses
// the same stale max for numerator and denominator, which is exact.
#include "sm100.cuh"
#include "tiles.cuh"
#include "kernels.h"
#include <stdlib.h>

#ifdef A2D_X_MMA_ONLY
#define XWAIT(b, ph) ((void)0)
#define XLOOP 0
#else
#define XWAIT(b, ph) mbar_wait(b, ph)
#define XLOOP 1
#endif
#ifdef A2D_X_NO_EXP
#define XEX2(x) (x)
#else
#define XEX2(x) ex2(x)
#endif

namespace a2d {

namespace {

constexpr int FWD_THREADS = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;

template <int HD>
struct FwdLayout {
  static constexpr int SLAB = TILE * 128;  // bytes of one 128-row x 64-col bf16 slab
  static constexpr int SLABS = HD / 64;
  static constexpr int TILE_BYTES = SLAB * SLABS;
  static constexpr int KST = 3;
  static constexpr int VST = 3;
  static constexpr int OFF_Q = 0;  // Q staging (moved into TMEM before the sweep)
  static constexpr int OFF_K = OFF_Q + TILE_BYTES;
  static constexpr int OFF_V = OFF_K + KST * TILE_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * TILE_BYTES;
  // barriers
  static constexpr int B_Q = 0;
  static constexpr int B_QREADY = 1;
  static constexpr int B_KFULL = 2;
  static constexpr int B_KEMPTY = B_KFULL + KST;
  static constexpr int B_VFULL = B_KEMPTY + KST;
  static constexpr int B_VEMPTY = B_VFULL + VST;
  static constexpr int B_SFULL = B_VEMPTY + VST;
  static constexpr int B_PFULL = B_SFULL + 2;   // 2 barriers: P_j arrives on [j & 1]
  static constexpr int B_PVDONE = B_PFULL + 2;  // 2 barriers: PV_j arrives on [j & 1]
  static constexpr int NBAR = B_PVDONE + 2;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TMEMPTR + 16;
  static_assert(SMEM <= 232448, "shared memory budget");
};

// TMEM (512 columns): S / P double buffer, O accumulator, Q (bf16 pairs, the
// A operand of S = Q K^T).  P overwrites the first half of its S buffer and
// feeds O += P V as the TMEM A operand, so neither Q nor P costs shared-memory
// bandwidth: per key tile the tensor core reads only K and V from SMEM.
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t TM_S = 0;    // S[b] at b*128 (P[b] in its first 64 columns)
constexpr uint32_t TM_O = 256;
constexpr uint32_t TM_Q = 384;

template <int HD>
__global__ void __launch_bounds__(FWD_THREADS, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ a2d_tile_fwd_args p) {
  using L = FwdLayout<HD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  if ((sb & 1023) != 0) __trap();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // q tiles vary fastest so co-resident CTAs share one head's K/V in L2;
  // within a head the heaviest (causal) tiles start first.
  const int bh = blockIdx.y;
  const int bh_kv = p.kv_group > 1 ? bh / p.kv_group : bh;  // GQA / MQA: shared k/v head
  const int qt_idx = gridDim.x - 1 - blockIdx.x;
  const int rot = qt_idx;  // rotated key sweep (TileCursor)
  auto bar = [&](int i) { return sb + L::OFF_BAR + 8 * i; };

  if (threadIdx.x == 0) {
    mbar_init(bar(L::B_Q), 1);
    mbar_init(bar(L::B_QREADY), 128);
    for (int i = 0; i < L::KST; ++i) {
      mbar_init(bar(L::B_KFULL + i), 1);
      mbar_init(bar(L::B_KEMPTY + i), 1);
    }
    for (int i = 0; i < L::VST; ++i) {
      mbar_init(bar(L::B_VFULL + i), 1);
      mbar_init(bar(L::B_VEMPTY + i), 1);
    }
    mbar_init(bar(L::B_SFULL + 0), 1);
    mbar_init(bar(L::B_SFULL + 1), 1);
    mbar_init(bar(L::B_PFULL + 0), 128);
    mbar_init(bar(L::B_PFULL + 1), 128);
    mbar_init(bar(L::B_PVDONE + 0), 1);
    mbar_init(bar(L::B_PVDONE + 1), 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) {
    tmem_alloc(sb + L::OFF_TMEMPTR, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + L::OFF_TMEMPTR);

  const bool causal = p.causal != 0;
  const TileRef qt = tile_ref(p.q_map, p.nq, qt_idx * TILE);
  TileRange kr;
  key_range(p.k_map, p.nk, causal, qt.gmax, kr);
  const int n_tiles = kr.total;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0 && n_tiles > 0) {
      mbar_expect_tx(bar(L::B_Q), L::TILE_BYTES);
      for (int s = 0; s < L::SLABS; ++s)
        tma_load_3d(sb + L::OFF_Q + s * L::SLAB, &tm_q, bar(L::B_Q), s * 64, qt.row0, bh);
      TileCursor cur;
      cur.start(kr, rot);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      for (int j = 0; j < n_tiles; ++j, cur.next(kr)) {
        const int krow = cur.row0(p.k_map);
        mbar_wait(bar(L::B_KEMPTY + ks), kph ^ 1);
        mbar_expect_tx(bar(L::B_KFULL + ks), L::TILE_BYTES);
        for (int s = 0; s < L::SLABS; ++s)
          tma_load_3d(sb + L::OFF_K + ks * L::TILE_BYTES + s * L::SLAB, &tm_k,
                      bar(L::B_KFULL + ks), s * 64, krow, bh_kv);
        if (++ks == L::KST) { ks = 0; kph ^= 1; }
        mbar_wait(bar(L::B_VEMPTY + vs), vph ^ 1);
        mbar_expect_tx(bar(L::B_VFULL + vs), L::TILE_BYTES);
        for (int s = 0; s < L::SLABS; ++s)
          tma_load_3d(sb + L::OFF_V + vs * L::TILE_BYTES + s * L::SLAB, &tm_v,
                      bar(L::B_VFULL + vs), s * 64, krow, bh_kv);
        if (++vs == L::VST) { vs = 0; vph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, HD, 0, 1);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      mbar_wait(bar(L::B_QREADY), 0);  // Q is in TMEM
      tc_fence_after();
      auto issue_qk = [&](int j) {
        mbar_wait(bar(L::B_KFULL + ks), kph);
        tc_fence_after();
        const uint32_t d = tmem + TM_S + (j & 1) * 128;
        const uint32_t kbase = sb + L::OFF_K + ks * L::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * L::SLAB + (kk & 3) * 32;
          umma_bf16_ts(d, tmem + TM_Q + kk * 8, make_sdesc(kbase + off, 16, 1024), idesc_qk,
                       kk > 0);
        }
        umma_commit(bar(L::B_KEMPTY + ks));
        umma_commit(bar(L::B_SFULL + (j & 1)));
        if (++ks == L::KST) { ks = 0; kph ^= 1; }
      };
      issue_qk(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) issue_qk(j + 1);
        XWAIT(bar(L::B_PFULL + (j & 1)), (j >> 1) & 1);
        mbar_wait(bar(L::B_VFULL + vs), vph);
        tc_fence_after();
        const uint32_t vbase = sb + L::OFF_V + vs * L::TILE_BYTES;
        const uint32_t pcol = tmem + TM_S + (j & 1) * 128;  // P_j (bf16 pairs) in TMEM
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk) {
          const uint64_t b = make_sdesc(vbase + kk * 2048, L::SLAB, 1024);
          umma_bf16_ts(tmem + TM_O, pcol + kk * 8, b, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(bar(L::B_VEMPTY + vs));
        umma_commit(bar(L::B_PVDONE + (j & 1)));
        if (++vs == L::VST) { vs = 0; vph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax WG
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    const float sl2 = p.scale * kLog2e;
    float m_run = -INFINITY;  // running max of scale*log2e*s
    float l_run = 0.f;
    if (n_tiles > 0) {
      // Q row -> TMEM (the A operand of S = Q K^T): the TMA-staged, 128B-swizzled
      // K-major row is re-read as bf16 pairs, one 32-bit TMEM column per pair.
      mbar_wait(bar(L::B_Q), 0);
      uint32_t qv[HD / 2];
#pragma unroll
      for (int s = 0; s < L::SLABS; ++s) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 u = *reinterpret_cast<const uint4*>(
              smem + L::OFF_Q + s * L::SLAB + row * 128 + ((c ^ (row & 7)) << 4));
          qv[32 * s + 4 * c + 0] = u.x;
          qv[32 * s + 4 * c + 1] = u.y;
          qv[32 * s + 4 * c + 2] = u.z;
          qv[32 * s + 4 * c + 3] = u.w;
        }
      }
#pragma unroll
      for (int c = 0; c < HD / 64; ++c)
        tmem_st32(tmem + lane_addr + TM_Q + 32 * c, reinterpret_cast<const float*>(qv + 32 * c));
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(L::B_QREADY));
    }
    TileCursor cur;
    cur.start(kr, rot);
    for (int j = 0; j < (XLOOP ? n_tiles : 0); ++j, cur.next(kr)) {
      const TileRef kt = tile_ref(p.k_map, p.nk, cur.row0(p.k_map));
      const PairMask pm = pair_mask(p.q_map, qt, kt, causal);
      int lim = TILE - 1;
      if (pm.partial) lim = row_limit(p.q_map, p.k_map, qt, kt, pm, causal, row);

      mbar_wait(bar(L::B_SFULL + (j & 1)), (j >> 1) & 1);
      tc_fence_after();
      float s[TILE];
#pragma unroll
      for (int c = 0; c < TILE / 32; ++c)
        tmem_ld32(tmem + lane_addr + TM_S + (j & 1) * 128 + c * 32, s + c * 32);
      tmem_wait_ld();
      if (pm.partial) {
#pragma unroll
        for (int jj = 0; jj < TILE; ++jj)
          if (jj > lim) s[jj] = -INFINITY;
      }
      const float mx = rowmax128(s);
      const float m_new = fmaxf(m_run, mx * sl2);
      float alpha = 1.f;
      if (m_new > m_run + kRescaleThreshold) {
        alpha = ex2(m_run - m_new);
        m_run = m_new;
      }
      const float mb = (m_run == -INFINITY) ? 0.f : m_run;
      uint32_t pk[TILE / 2];
      float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      const float2 sc = make_float2(sl2, sl2), nb = make_float2(-mb, -mb);
      if (pm.partial) {  // masked entries are -inf: the exact MUFU path keeps them 0
#pragma unroll
        for (int jj = 0; jj < TILE; jj += 2) {
          const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
          const float2 e = make_float2(XEX2(x.x), XEX2(x.y));
          acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
          pk[jj / 2] = pack_bf16(e.x, e.y);
        }
      } else {  // a quarter of the exponentials on the FMA pipe (MUFU offload)
#pragma unroll
        for (int jj = 0; jj < TILE; jj += 2) {
          const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
          float2 e;
          if (((jj >> 1) & 3) == 3) e = exp2_poly2(x);
          else e = make_float2(XEX2(x.x), XEX2(x.y));
          acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
          pk[jj / 2] = pack_bf16(e.x, e.y);
        }
      }
      const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
      const float2 a = fadd2(a01, a23);
      l_run = l_run * alpha + (a.x + a.y);

      // P_j (bf16 pairs) over the first 64 columns of its own S buffer: the
      // S values there were consumed above, and PV_{j-2} (the last reader of
      // this buffer's previous P) completed before QK_j was issued.
      const uint32_t pcol = tmem + lane_addr + TM_S + (j & 1) * 128;
      tmem_st32(pcol, reinterpret_cast<const float*>(pk));
      tmem_st32(pcol + 32, reinterpret_cast<const float*>(pk + 32));
      // O is rescaled only when the running max moved: that needs PV_{j-1}
      // to have landed in O first.
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        mbar_wait(bar(L::B_PVDONE + ((j - 1) & 1)), ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          float o[32];
          tmem_ld32(tmem + lane_addr + TM_O + c * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= alpha;
          tmem_st32(tmem + lane_addr + TM_O + c * 32, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      // a warp whose rows are all masked can reach tile j+1 (S_{j+1} is issued
      // before PV_j) while another is still on tile j: alternating barriers
      // keep its early arrival out of tile j's count
      mbar_arrive(bar(L::B_PFULL + (j & 1)));
    }

    // ------------------------------------------------------------ epilogue
    if (n_tiles > 0) {
      // PV_j arrives on PVDONE[j & 1], so each barrier sees every other PV and
      // a parity wait can never alias a phase two steps back: the last PV on
      // each barrier is awaited exactly.
      if (n_tiles > 1)
        mbar_wait(bar(L::B_PVDONE + ((n_tiles - 2) & 1)), ((n_tiles - 2) >> 1) & 1);
      mbar_wait(bar(L::B_PVDONE + ((n_tiles - 1) & 1)), ((n_tiles - 1) >> 1) & 1);
      tc_fence_after();
    }
    const bool valid = row < qt.nvalid;
    const int grow = qt.row0 + row;
    const float lse_new = (l_run > 0.f) ? (m_run + lg2(l_run)) * kLn2 : -INFINITY;
    float w_new = (l_run > 0.f) ? 1.f / l_run : 0.f;
    float w_old = 0.f;
    float lse_out = lse_new;
    float* lse_ptr = p.lse + (long long)bh * p.nq + grow;
    if (p.accumulate && valid) {
      const float lse_old = *lse_ptr;
      const float mxl = fmaxf(lse_old, lse_new);
      if (mxl == -INFINITY) {
        w_old = 0.f;
        w_new = 0.f;
        lse_out = -INFINITY;
      } else {
        const float eo = __expf(lse_old - mxl);
        const float en = __expf(lse_new - mxl);
        const float inv = 1.f / (eo + en);
        w_old = eo * inv;
        w_new *= en * inv;
        lse_out = mxl + __logf(eo + en);
      }
    }
    if (valid) *lse_ptr = lse_out;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      float o[32];
      if (n_tiles > 0) {
        tmem_ld32(tmem + lane_addr + TM_O + c * 32, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = 0.f;
      }
      if (!valid) continue;
      if (p.o_dtype == A2D_F32) {
        float* dst = reinterpret_cast<float*>(p.o) + (long long)bh * p.o_stride_bh +
                     (long long)grow * p.o_stride_row + c * 32;
        if (p.accumulate) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 old = *reinterpret_cast<const float4*>(dst + i);
            float4 v;
            v.x = old.x * w_old + o[i + 0] * w_new;
            v.y = old.y * w_old + o[i + 1] * w_new;
            v.z = old.z * w_old + o[i + 2] * w_new;
            v.w = old.w * w_old + o[i + 3] * w_new;
            *reinterpret_cast<float4*>(dst + i) = v;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + i) =
                make_float4(o[i] * w_new, o[i + 1] * w_new, o[i + 2] * w_new, o[i + 3] * w_new);
        }
      } else {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.o) +
                             (long long)bh * p.o_stride_bh + (long long)grow * p.o_stride_row +
                             c * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 v;
          v.x = pack_bf16(o[i + 0] * w_new, o[i + 1] * w_new);
          v.y = pack_bf16(o[i + 2] * w_new, o[i + 3] * w_new);
          v.z = pack_bf16(o[i + 4] * w_new, o[i + 5] * w_new);
          v.w = pack_bf16(o[i + 6] * w_new, o[i + 7] * w_new);
          *reinterpret_cast<uint4*>(dst + i) = v;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace

template <int HD>
int launch_fwd_hd(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                  const CUtensorMap& tv, cudaStream_t stream) {
  using L = FwdLayout<HD>;
  static bool configured[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         L::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(fwd)");
    configured[dev & 63] = true;
  }
  const int q_tiles = (a.q_map.mode == A2D_IDX_AFFINE && a.q_map.nblocks > 1)
                          ? a.q_map.nblocks * (a.q_map.rows_per_block / TILE)
                          : (a.nq + TILE - 1) / TILE;
  dim3 grid(q_tiles, a.bh);
  fwd_kernel<HD><<<grid, FWD_THREADS, L::SMEM, stream>>>(tq, tk, tv, a);
  return check_launch("fwd_kernel");
}

int launch_tile_fwd(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, cudaStream_t stream) {
  // two query tiles per CTA (tile_fwd2.cu) unless A2D_FWD_V1 selects the
  // single-tile kernel (kept for A/B measurements)
  static const bool v1 = getenv("A2D_FWD_V1") != nullptr;
  if (!v1 || (a.h != 64 && a.h != 128)) return launch_tile_fwd2(a, tq, tk, tv, stream);
  if (a.h == 128) return launch_fwd_hd<128>(a, tq, tk, tv, stream);
  return launch_fwd_hd<64>(a, tq, tk, tv, stream);
}

}  // namespace a2d
