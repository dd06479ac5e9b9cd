// tile_fwd2.cu — Attention2D tile forward on sm_100a, two query tiles per CTA.
//
// Same contract as the single-tile kernel in tile_fwd.cu (the streaming
// softmax of the reference's flash_forward, numpy_backend.py:24-43 /
// numba_backend.py:38-76, emitting the (O, LSE) partial that attn_fix
// merges, attention.py:194-214), restructured so the tensor pipe never waits
// for one softmax warpgroup: each CTA owns TWO 128-row query tiles of one
// head and sweeps their common key range once.
//
// Warp roles (320 threads = 200 registers each, one CTA per SM):
//   warp 0       TMA producer: Q0/Q1 once, then K (3-stage) / V (2-stage) rings
//   warp 1       tcgen05 MMA issuer (one elected lane) + TMEM owner
//   warps 2-5    softmax warpgroup 0 (query tile 0, one row per thread; warp w
//                owns TMEM lanes 32*(w%4)..+31)
//   warps 6-9    softmax warpgroup 1 (query tile 1)
// TMEM (512 columns): S0 [0,128), S1 [128,256), O0 [256,256+H), O1 after it.
// P_t overwrites the first 64 columns of S_t and is the TMEM A operand of
// O_t += P_t V.  Per key tile j the MMA order is
//   PV0(j-1), QK0(j), PV1(j-1), QK1(j)
// so while warpgroup 0 turns S0(j) into P0(j), the tensor pipe runs PV1(j-1)
// and QK1(j) (and vice versa): two softmax phases in flight per SM sub-
// partition, 2 x 1024 tensor cycles per key tile for the pair.
// Because tcgen05 MMAs of one thread complete in order and S_t(j)'s commit
// is issued after PV_t(j-1), "S_t(j) full" also means "O_t holds PV_t(j-1)":
// the rare rescale of O_t needs no extra barrier.
#include "sm100.cuh"
#include "tiles.cuh"
#include "kernels.h"

namespace a2d {

namespace {

constexpr int F2_THREADS = 384;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;

template <int HD>
struct F2Layout {
  static constexpr int SLAB = TILE * 128;  // one 128-row x 64-col bf16 slab
  static constexpr int SLABS = HD / 64;
  static constexpr int TILE_BYTES = SLAB * SLABS;
  static constexpr int KST = 3;
  static constexpr int VST = HD == 128 ? 2 : 3;
  static constexpr int OFF_Q = 0;  // Q0, Q1
  static constexpr int OFF_K = OFF_Q + 2 * TILE_BYTES;
  static constexpr int OFF_V = OFF_K + KST * TILE_BYTES;
  static constexpr int OFF_BAR = OFF_V + VST * TILE_BYTES;
  static constexpr int B_Q = 0;
  static constexpr int B_KFULL = 1;
  static constexpr int B_KEMPTY = B_KFULL + KST;
  static constexpr int B_VFULL = B_KEMPTY + KST;
  static constexpr int B_VEMPTY = B_VFULL + VST;
  static constexpr int B_SFULL = B_VEMPTY + VST;  // [2]: S_t(j) computed (and PV_t(j-1) done)
  static constexpr int B_PFULL = B_SFULL + 2;     // [2]: P_t(j) stored (128 arrivals)
  static constexpr int B_ODONE = B_PFULL + 2;     // [2]: last PV_t done
  static constexpr int NBAR = B_ODONE + 2;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TMEMPTR + 16;
  static_assert(SMEM <= 232448, "shared memory budget");
};

constexpr uint32_t TMEM_COLS = 512;

template <int HD>
__device__ __forceinline__ void f2_epilogue(const a2d_tile_fwd_args& p, uint32_t tmem_o,
                                            bool have_o, int bh, int grow, bool valid,
                                            float m_run, float l_run) {
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
    if (have_o) {
      tmem_ld32(tmem_o + c * 32, o);
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
          const float4 old = *reinterpret_cast<const float4*>(dst + i);
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
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.o) + (long long)bh * p.o_stride_bh +
                           (long long)grow * p.o_stride_row + c * 32;
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

template <int HD>
__global__ void __launch_bounds__(F2_THREADS, 1)
    fwd2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ a2d_tile_fwd_args p,
                int q_tiles) {
  using L = F2Layout<HD>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  if ((sb & 1023) != 0) __trap();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // tile pairs vary fastest (co-resident CTAs share one head's K/V in L2);
  // the heaviest causal pairs of a head start first.
  const int bh = blockIdx.y;
  const int pair = gridDim.x - 1 - blockIdx.x;
  auto bar = [&](int i) { return sb + L::OFF_BAR + 8 * i; };
  const uint32_t TM_O0 = 256, TM_O1 = 256 + HD;

  if (threadIdx.x == 0) {
    mbar_init(bar(L::B_Q), 1);
    for (int i = 0; i < L::KST; ++i) {
      mbar_init(bar(L::B_KFULL + i), 1);
      mbar_init(bar(L::B_KEMPTY + i), 1);
    }
    for (int i = 0; i < L::VST; ++i) {
      mbar_init(bar(L::B_VFULL + i), 1);
      mbar_init(bar(L::B_VEMPTY + i), 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(bar(L::B_SFULL + t), 1);
      mbar_init(bar(L::B_PFULL + t), 128);
      mbar_init(bar(L::B_ODONE + t), 1);
    }
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
  const int t0 = 2 * pair, t1 = 2 * pair + 1;
  const bool has1 = t1 < q_tiles;
  const TileRef qt0 = tile_ref(p.q_map, p.nq, t0 * TILE);
  TileRef qt1 = qt0;
  if (has1) qt1 = tile_ref(p.q_map, p.nq, t1 * TILE);
  TileRange kr;
  key_range(p.k_map, p.nk, causal, has1 ? max(qt0.gmax, qt1.gmax) : qt0.gmax, kr);
  const int n_tiles = kr.total;
  const int rot = pair;  // rotated key sweep

  if (warp < 4) {
    regs_dec<96>();
    if (warp == 0 && lane == 0 && n_tiles > 0) {
      // -------------------------------------------------------- producer
      mbar_expect_tx(bar(L::B_Q), 2 * L::TILE_BYTES);
      for (int s = 0; s < L::SLABS; ++s) {
        tma_load_3d(sb + L::OFF_Q + s * L::SLAB, &tm_q, bar(L::B_Q), s * 64, qt0.row0, bh);
        // an absent second tile loads out of bounds (zero fill), never read
        tma_load_3d(sb + L::OFF_Q + L::TILE_BYTES + s * L::SLAB, &tm_q, bar(L::B_Q), s * 64,
                    has1 ? qt1.row0 : p.nq, bh);
      }
      TileCursor cur;
      cur.start(kr, rot);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      for (int j = 0; j < n_tiles; ++j, cur.next(kr)) {
        const int krow = cur.row0(p.k_map);
        mbar_wait(bar(L::B_KEMPTY + ks), kph ^ 1);
        mbar_expect_tx(bar(L::B_KFULL + ks), L::TILE_BYTES);
        for (int s = 0; s < L::SLABS; ++s)
          tma_load_3d(sb + L::OFF_K + ks * L::TILE_BYTES + s * L::SLAB, &tm_k,
                      bar(L::B_KFULL + ks), s * 64, krow, bh);
        if (++ks == L::KST) { ks = 0; kph ^= 1; }
        mbar_wait(bar(L::B_VEMPTY + vs), vph ^ 1);
        mbar_expect_tx(bar(L::B_VFULL + vs), L::TILE_BYTES);
        for (int s = 0; s < L::SLABS; ++s)
          tma_load_3d(sb + L::OFF_V + vs * L::TILE_BYTES + s * L::SLAB, &tm_v,
                      bar(L::B_VFULL + vs), s * 64, krow, bh);
        if (++vs == L::VST) { vs = 0; vph ^= 1; }
      }
    } else if (warp == 1 && lane == 0 && n_tiles > 0) {
      // -------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, HD, 0, 1);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      mbar_wait(bar(L::B_Q), 0);
      auto issue_qk = [&](int t) {  // S_t = Q_t K^T on the current K stage
        const uint32_t qbase = sb + L::OFF_Q + t * L::TILE_BYTES;
        const uint32_t kbase = sb + L::OFF_K + ks * L::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * L::SLAB + (kk & 3) * 32;
          umma_bf16(tmem + t * 128, make_sdesc(qbase + off, 16, 1024),
                    make_sdesc(kbase + off, 16, 1024), idesc_qk, kk > 0);
        }
        umma_commit(bar(L::B_SFULL + t));
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t V on the current V stage
        const uint32_t vbase = sb + L::OFF_V + vs * L::TILE_BYTES;
        const uint32_t pcol = tmem + t * 128;
        const uint32_t ocol = tmem + (t ? TM_O1 : TM_O0);
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk)
          umma_bf16_ts(ocol, pcol + kk * 8, make_sdesc(vbase + kk * 2048, L::SLAB, 1024),
                       idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
      };
      // prologue: S0(0), S1(0)
      mbar_wait(bar(L::B_KFULL + ks), kph);
      tc_fence_after();
      issue_qk(0);
      issue_qk(1);
      umma_commit(bar(L::B_KEMPTY + ks));
      if (++ks == L::KST) { ks = 0; kph ^= 1; }
      for (int j = 0; j < n_tiles; ++j) {
        const bool more = j + 1 < n_tiles;
        mbar_wait(bar(L::B_VFULL + vs), vph);
        // ---- tile 0: PV0(j), QK0(j+1)
        mbar_wait(bar(L::B_PFULL + 0), j & 1);
        tc_fence_after();
        issue_pv(0, j);
        if (more) {
          mbar_wait(bar(L::B_KFULL + ks), kph);
          tc_fence_after();
          issue_qk(0);
        } else {
          umma_commit(bar(L::B_ODONE + 0));
        }
        // ---- tile 1: PV1(j), QK1(j+1)
        mbar_wait(bar(L::B_PFULL + 1), j & 1);
        tc_fence_after();
        issue_pv(1, j);
        umma_commit(bar(L::B_VEMPTY + vs));
        if (++vs == L::VST) { vs = 0; vph ^= 1; }
        if (more) {
          issue_qk(1);
          umma_commit(bar(L::B_KEMPTY + ks));
          if (++ks == L::KST) { ks = 0; kph ^= 1; }
        } else {
          umma_commit(bar(L::B_ODONE + 1));
        }
      }
    }
  } else {
    regs_inc<200>();
    // ------------------------------------------------------------ softmax WGs
    const int t = (warp - 4) >> 2;  // query tile of this warpgroup
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_addr + t * 128;
    const uint32_t o_addr = tmem + lane_addr + (t ? TM_O1 : TM_O0);
    const bool present = (t == 0) || has1;
    const TileRef qt = t ? qt1 : qt0;
    const float sl2 = p.scale * kLog2e;
    float m_run = -INFINITY;  // running max of scale*log2e*s
    float l_run = 0.f;
    TileCursor cur;
    cur.start(kr, rot);
    for (int j = 0; j < n_tiles; ++j, cur.next(kr)) {
      const TileRef kt = tile_ref(p.k_map, p.nk, cur.row0(p.k_map));
      PairMask pm;
      int lim = TILE - 1;
      if (present) {
        pm = pair_mask(p.q_map, qt, kt, causal);
        if (pm.partial) lim = row_limit(p.q_map, p.k_map, qt, kt, pm, causal, row);
      } else {
        pm.partial = true;
        lim = -1;
      }
      mbar_wait(bar(L::B_SFULL + t), j & 1);
      tc_fence_after();
      float s[TILE];
#pragma unroll
      for (int c = 0; c < TILE / 32; ++c) tmem_ld32(s_addr + c * 32, s + c * 32);
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
          const float2 e = make_float2(ex2(x.x), ex2(x.y));
          acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
          pk[jj / 2] = pack_bf16(e.x, e.y);
        }
      } else {  // a quarter of the exponentials on the FMA pipe (MUFU offload)
#pragma unroll
        for (int jj = 0; jj < TILE; jj += 2) {
          const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
          float2 e;
          if (((jj >> 1) & 3) == 3) e = exp2_poly2(x);
          else e = make_float2(ex2(x.x), ex2(x.y));
          acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
          pk[jj / 2] = pack_bf16(e.x, e.y);
        }
      }
      const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
      const float2 a = fadd2(a01, a23);
      l_run = l_run * alpha + (a.x + a.y);
      // P_t(j) over the first 64 columns of S_t (the S values were consumed above)
      tmem_st32(s_addr, reinterpret_cast<const float*>(pk));
      tmem_st32(s_addr + 32, reinterpret_cast<const float*>(pk + 32));
      // O_t already holds PV_t(j-1) (its commit preceded S_t(j)'s): rescale
      // in place when this warp's running max moved
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          float o[32];
          tmem_ld32(o_addr + c * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= alpha;
          tmem_st32(o_addr + c * 32, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(L::B_PFULL + t));
    }
    // ------------------------------------------------------------ epilogue
    if (n_tiles > 0) {
      mbar_wait(bar(L::B_ODONE + t), 0);
      tc_fence_after();
    }
    if (present)
      f2_epilogue<HD>(p, o_addr, n_tiles > 0, bh, qt.row0 + row, row < qt.nvalid, m_run, l_run);
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
int launch_fwd2_hd(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                   const CUtensorMap& tv, cudaStream_t stream) {
  using L = F2Layout<HD>;
  static bool configured[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(fwd2_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(fwd2)");
    configured[dev & 63] = true;
  }
  const int q_tiles = (a.q_map.mode == A2D_IDX_AFFINE && a.q_map.nblocks > 1)
                          ? a.q_map.nblocks * (a.q_map.rows_per_block / TILE)
                          : (a.nq + TILE - 1) / TILE;
  dim3 grid((q_tiles + 1) / 2, a.bh);
  fwd2_kernel<HD><<<grid, F2_THREADS, L::SMEM, stream>>>(tq, tk, tv, a, q_tiles);
  return check_launch("fwd2_kernel");
}

int launch_tile_fwd2(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                     const CUtensorMap& tv, cudaStream_t stream) {
  if (a.h == 128) return launch_fwd2_hd<128>(a, tq, tk, tv, stream);
  return launch_fwd2_hd<64>(a, tq, tk, tv, stream);
}

}  // namespace a2d
