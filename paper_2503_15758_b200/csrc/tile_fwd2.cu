// tile_fwd2.cu — Attention2D tile forward on sm_100a, two query tiles per CTA.
//
// Same contract as the single-tile kernel in tile_fwd.cu (the streaming
// softmax of the reference's flash_forward, numpy_backend.py:24-43 /
// numba_backend.py:38-76, emitting the (O, LSE) partial that attn_fix
// merges, attention.py:194-214), restructured so the tensor pipe never waits
// for one softmax warpgroup: each CTA owns TWO 128-row query tiles of one
// head and sweeps their common key range once.
//
// Warp roles (one CTA per SM; CS = column split of the softmax, 1 or 2):
//   warp 0       TMA producer: Q0/Q1 once, then K (3-stage) / V (2-stage) rings
//   warp 1       tcgen05 MMA issuer (whole warp, one elected lane issues)
//   warps 2-3    idle (complete the register-reallocation warpgroup)
//   warps 4..    2*CS softmax warpgroups: warpgroup (t, h) owns query tile t,
//                key columns [h*128/CS, (h+1)*128/CS) of every S tile; warp w
//                owns TMEM lanes 32*(w%4)..+31 (one query row per thread).
//                With CS = 2 the two halves of a row exchange their maxima
//                through shared memory (64-thread named barrier per row
//                quarter), halving the per-tile softmax latency that sits on
//                the S -> P -> PV -> S critical path.
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

// which exponential pairs go to the FMA-pipe polynomial (MUFU offload)
#if defined(F2X_ALLMUFU)
#define F2_POLY(jj) false
#elif defined(F2X_POLYHALF)
#define F2_POLY(jj) (((jj) >> 1) & 1)
#elif defined(F2X_POLY1OF4)
#define F2_POLY(jj) ((((jj) >> 1) & 3) == 3)
#elif defined(F2X_POLY3)
#define F2_POLY(jj) ((((jj) >> 1) & 7) == 1 || (((jj) >> 1) & 7) == 4 || (((jj) >> 1) & 7) == 6)
#else  // one pair in eight (measured best on B200 once the max tree is gone)
#define F2_POLY(jj) ((((jj) >> 1) & 7) == 7)
#endif
#ifdef F2X_NOEXP
#define XEX2(x) (x)
#else
#define XEX2(x) ex2(x)
#endif
#ifdef F2X_SPIN
#define F2_WAIT mbar_wait
#else
#define F2_WAIT mbar_wait_sleep
#endif

#ifdef F2X_TRACE
__device__ long long g_f2trace[48][1024];
extern "C" int a2d_trace_dump(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_f2trace, sizeof(g_f2trace));
}
#define TR(row, i)                                                                  \
  do {                                                                              \
    if (blockIdx.x == TX && blockIdx.y == TY && (threadIdx.x & 31) == 0 && (i) < 1024) \
      g_f2trace[row][i] = clock64();                                                \
  } while (0)
#else
#define TR(row, i) ((void)0)
#endif

namespace a2d {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
#ifdef F2X_ROWMAX
constexpr float kRescaleThreshold = 8.0f;
#endif

template <int HD>
struct F2Layout {
  static constexpr int SLAB = TILE * 128;  // one 128-row x 64-col bf16 slab
  static constexpr int SLABS = HD / 64;
  static constexpr int TILE_BYTES = SLAB * SLABS;
#ifdef F2X_KST2
  static constexpr int KST = 2;
#else
  static constexpr int KST = 3;
#endif
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
  static constexpr int OFF_XCH = OFF_TMEMPTR + 16;  // [2 tiles][2 halves][128 rows] fp32
  static constexpr int SMEM = OFF_XCH + 2 * 2 * 128 * 4;
  static_assert(SMEM <= 232448, "shared memory budget");
};

constexpr uint32_t TMEM_COLS = 512;

template <int HD, int NCOL>
__device__ __forceinline__ void f2_epilogue(const a2d_tile_fwd_args& p, uint32_t tmem_o,
                                            bool have_o, int bh, int grow, bool valid,
                                            float m_run, float l_run, int col0, bool write_lse) {
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
  if (valid && write_lse) *lse_ptr = lse_out;
#pragma unroll
  for (int c = 0; c < NCOL / 32; ++c) {
    float o[32];
    if (have_o) {
      tmem_ld32(tmem_o + c * 32, o);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = 0.f;
    }
    if (!valid || col0 + c * 32 >= p.h) continue;  // columns past h are zero fill
    if (p.o_dtype == A2D_F32) {
      float* dst = reinterpret_cast<float*>(p.o) + (long long)bh * p.o_stride_bh +
                   (long long)grow * p.o_stride_row + col0 + c * 32;
      if (p.accumulate) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          if (col0 + c * 32 + i >= p.h) continue;
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
          if (col0 + c * 32 + i < p.h)
            *reinterpret_cast<float4*>(dst + i) =
                make_float4(o[i] * w_new, o[i + 1] * w_new, o[i + 2] * w_new, o[i + 3] * w_new);
      }
    } else {
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.o) + (long long)bh * p.o_stride_bh +
                           (long long)grow * p.o_stride_row + col0 + c * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        if (col0 + c * 32 + i >= p.h) continue;
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

template <int CS>
struct F2Threads {
  static constexpr int N = 384;  // producer/MMA warpgroup + 8 softmax warps (both modes)
};

template <int HD, int CS>
__global__ void __launch_bounds__(F2Threads<CS>::N, 1)
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
  const int bh_kv = p.kv_group > 1 ? bh / p.kv_group : bh;  // GQA / MQA: shared k/v head
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
      mbar_init(bar(L::B_PFULL + t), 128 * CS);
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
        F2_WAIT(bar(L::B_KEMPTY + ks), kph ^ 1);
        TR(45, j);
#ifdef F2X_NOTMA
        if (j >= L::KST) {
          mbar_arrive(bar(L::B_KFULL + ks));
          if (++ks == L::KST) { ks = 0; kph ^= 1; }
          F2_WAIT(bar(L::B_VEMPTY + vs), vph ^ 1);
          mbar_arrive(bar(L::B_VFULL + vs));
          if (++vs == L::VST) { vs = 0; vph ^= 1; }
          continue;
        }
#endif
        mbar_expect_tx(bar(L::B_KFULL + ks), L::TILE_BYTES);
        for (int s = 0; s < L::SLABS; ++s)
          tma_load_3d(sb + L::OFF_K + ks * L::TILE_BYTES + s * L::SLAB, &tm_k,
                      bar(L::B_KFULL + ks), s * 64, krow, bh_kv);
        if (++ks == L::KST) { ks = 0; kph ^= 1; }
        F2_WAIT(bar(L::B_VEMPTY + vs), vph ^ 1);
        TR(46, j);
        mbar_expect_tx(bar(L::B_VFULL + vs), L::TILE_BYTES);
        for (int s = 0; s < L::SLABS; ++s)
          tma_load_3d(sb + L::OFF_V + vs * L::TILE_BYTES + s * L::SLAB, &tm_v,
                      bar(L::B_VFULL + vs), s * 64, krow, bh_kv);
        if (++vs == L::VST) { vs = 0; vph ^= 1; }
      }
    } else if (warp == 1 && n_tiles > 0) {
      // -------------------------------------------------------- MMA issuer (whole warp, one elected lane issues)
      // head dims below the tile width: only ceil(h/16) K steps for Q K^T and
      // an N = 16 ceil(h/16) PV (the tile's other columns are zero fill)
      const int ksteps = (p.h + 15) / 16;
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0, 0);
      const uint32_t idesc_pv = make_idesc_bf16(128, ksteps * 16, 0, 1);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      F2_WAIT(bar(L::B_Q), 0);
      // Descriptors are built once; per MMA only a constant is added to the
      // start-address field (16-byte units, no carry: shared memory < 256 KB),
      // so the issue loop keeps pace with the 64-cycle N=128 MMA even while
      // two softmax warps share this warp's sub-partition.
      const uint64_t dq0 = make_sdesc(sb + L::OFF_Q, 16, 1024);
      const uint64_t dk0 = make_sdesc(sb + L::OFF_K, 16, 1024);
      const uint64_t dv0 = make_sdesc(sb + L::OFF_V, L::SLAB, 1024);
      auto issue_qk = [&](int t) {  // S_t = Q_t K^T on the current K stage
        const uint64_t dq = dq0 + uint64_t(t * (L::TILE_BYTES >> 4));
        const uint64_t dk = dk0 + uint64_t(ks * (L::TILE_BYTES >> 4));
        const uint32_t d = tmem + t * 128;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint64_t off = uint64_t(((kk >> 2) * L::SLAB + (kk & 3) * 32) >> 4);
            if (kk < ksteps) umma_bf16(d, dq + off, dk + off, idesc_qk, kk > 0);
          }
          umma_commit(bar(L::B_SFULL + t));
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t V on the current V stage
        const uint64_t dv = dv0 + uint64_t(vs * (L::TILE_BYTES >> 4));
        const uint32_t pcol = tmem + t * 128;
        const uint32_t ocol = tmem + (t ? TM_O1 : TM_O0);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < TILE / 16; ++kk)
            umma_bf16_ts(ocol, pcol + kk * 8, dv + uint64_t(kk * (2048 >> 4)), idesc_pv,
                         (j > 0 || kk > 0) ? 1u : 0u);
        }
        __syncwarp();
      };
      auto commit = [&](int b) {
        if (elect_one()) umma_commit(bar(b));
        __syncwarp();
      };
      // prologue: S0(0), S1(0)
      F2_WAIT(bar(L::B_KFULL + ks), kph);
      tc_fence_after();
      issue_qk(0);
      issue_qk(1);
      commit(L::B_KEMPTY + ks);
      if (++ks == L::KST) { ks = 0; kph ^= 1; }
      for (int j = 0; j < n_tiles; ++j) {
        const bool more = j + 1 < n_tiles;
        F2_WAIT(bar(L::B_VFULL + vs), vph);
        TR(44, j);
        // ---- tile 0: PV0(j), QK0(j+1)
        F2_WAIT(bar(L::B_PFULL + 0), j & 1);
        tc_fence_after();
        TR(40, j);
        issue_pv(0, j);
        if (more) {
          F2_WAIT(bar(L::B_KFULL + ks), kph);
          tc_fence_after();
          issue_qk(0);
          TR(41, j);
        } else {
          commit(L::B_ODONE + 0);
        }
        // ---- tile 1: PV1(j), QK1(j+1)
        F2_WAIT(bar(L::B_PFULL + 1), j & 1);
        tc_fence_after();
        TR(42, j);
        issue_pv(1, j);
        commit(L::B_VEMPTY + vs);
        if (++vs == L::VST) { vs = 0; vph ^= 1; }
        if (more) {
          issue_qk(1);
          TR(43, j);
          commit(L::B_KEMPTY + ks);
          if (++ks == L::KST) { ks = 0; kph ^= 1; }
        } else {
          commit(L::B_ODONE + 1);
        }
      }
    }
  } else {
    regs_inc<200>();
    // ------------------------------------------------------------ softmax warps
    // CS = 1: warp w owns query tile t = (w-4)/4, all 128 key columns.
    // CS = 2: warp w owns column half h = (w-4)/4 of BOTH tiles (64 columns
    //         each), so every tile's exponentials run on two warps per SM
    //         sub-partition; the two halves of a row agree on the running max
    //         through shared memory and on the overflow re-base through
    //         barrier.red.or (named barrier 1 + quarter).
    constexpr int NC = TILE / CS;        // key columns of S per thread and tile
    constexpr int U = CS;                // tiles served by this warp
    const int sidx = warp - 4;
    const int quarter = warp & 3;
    const int h = CS == 1 ? 0 : (sidx >> 2);  // column half
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    const uint32_t xbar = 1 + quarter;
    const float sl2 = p.scale * kLog2e;
    const bool arr = p.q_map.mode == A2D_IDX_ARRAY;
    const int rot0 = n_tiles > 0 ? rot % n_tiles : 0;
    float m_run[U], l_run[U];
    uint32_t my_info[U];
    TileCursor cur[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      m_run[u] = -INFINITY;  // running max of scale*log2e*s (common to both halves)
      l_run[u] = 0.f;        // this half's share of the denominator
      my_info[u] = 0;
      if (arr) cur[u].start(kr, rot);
    }
    for (int j = 0; j < n_tiles; ++j) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = CS == 1 ? (sidx >> 2) : u;  // query tile of this unit
        const uint32_t s_addr = tmem + lane_addr + t * 128 + h * NC;
        const uint32_t p_addr = tmem + lane_addr + t * 128 + h * (NC / 2);
        const uint32_t o_addr = tmem + lane_addr + (t ? TM_O1 : TM_O0) + h * (HD / CS);
        float* xch = reinterpret_cast<float*>(smem + L::OFF_XCH) + t * 256;
        const bool present = (t == 0) || has1;
        const TileRef qt = t ? qt1 : qt0;
        // Per-tile mask classes for affine maps are computed 32 tiles at a
        // time, one tile per lane, and broadcast with one shuffle per tile;
        // explicit index arrays keep the per-tile binary-search path.
        bool partial;
        int lim = TILE - 1;  // last visible key column of this row (tile-relative)
        if (!present) {
          partial = true;
          lim = -1;
        } else if (arr) {
          const TileRef kt = tile_ref(p.k_map, p.nk, cur[u].row0(p.k_map));
          cur[u].next(kr);
          const PairMask pm = pair_mask(p.q_map, qt, kt, causal);
          partial = pm.partial;
          if (partial) lim = row_limit(p.q_map, p.k_map, qt, kt, pm, causal, row);
        } else {
          if ((j & 31) == 0) {
            const int f = j + lane;
            my_info[u] = 0;
            if (f < n_tiles) {
              const int g = rot0 + f < n_tiles ? rot0 + f : rot0 + f - n_tiles;
              const TileRef kt = tile_ref(p.k_map, p.nk, range_row0(kr, p.k_map, g));
              const PairMask q = pair_mask(p.q_map, qt, kt, causal);
              my_info[u] = uint32_t(q.thr + 512) | (uint32_t(q.kvalid) << 16) |
                           (q.partial ? 0x80000000u : 0u);
            }
          }
          const uint32_t inf = __shfl_sync(0xffffffffu, my_info[u], j & 31);
          partial = (inf >> 31) != 0;
          if (partial) {
            const int kvalid = int((inf >> 16) & 0xff);
            lim = causal ? min(row - (int(inf & 0xffff) - 512), kvalid - 1) : kvalid - 1;
          }
        }
        lim -= h * NC;  // relative to this half's first column
        mbar_wait(bar(L::B_SFULL + t), j & 1);
        tc_fence_after();
        TR(0 * 8 + t * 4 + quarter, j);
#ifdef F2X_NOSOFTMAX
        if (true) {
          tc_fence_before();
          mbar_arrive(bar(L::B_PFULL + t));
          continue;
        }
#endif
        float s[NC];
        auto load_s = [&]() {  // S_t(j) row from TMEM, causal / ragged columns masked
#pragma unroll
          for (int c = 0; c < NC / 32; ++c) tmem_ld32(s_addr + c * 32, s + c * 32);
          tmem_wait_ld();
          if (partial) {
#pragma unroll
            for (int jj = 0; jj < NC; ++jj)
              if (jj > lim) s[jj] = -INFINITY;
          }
        };
        load_s();
        TR(1 * 8 + t * 4 + quarter, j);
        float alpha = 1.f;
        uint32_t pk[NC / 2];
        const float2 sc = make_float2(sl2, sl2);
        // exponentials of this tile against the running max (P in pk, returns
        // the tile's share of the denominator)
        auto exps = [&](float mbase) -> float {
          float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
          const float2 nb = make_float2(-mbase, -mbase);
          if (partial) {  // masked entries are -inf: the exact MUFU path keeps them 0
#pragma unroll
            for (int jj = 0; jj < NC; jj += 2) {
              const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
              const float2 e = make_float2(XEX2(x.x), XEX2(x.y));
              acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
              pk[jj / 2] = pack_bf16(e.x, e.y);
            }
          } else {  // some exponentials on the FMA pipe (MUFU offload, F2_POLY)
#pragma unroll
            for (int jj = 0; jj < NC; jj += 2) {
              const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
              float2 e;
              if (F2_POLY(jj)) e = exp2_poly2(x);
              else e = make_float2(XEX2(x.x), XEX2(x.y));
              acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
              pk[jj / 2] = pack_bf16(e.x, e.y);
            }
          }
          const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
          const float2 a = fadd2(a01, a23);
          return a.x + a.y;
        };
        auto move_max = [&]() {  // exact running max of this tile (log2 domain)
          float mx = rowmax<NC>(s) * sl2;
          if constexpr (CS == 2) {
            // both halves of a row need one common max: exchange through smem
            // (slot (tile, half, row); the partner reads it before arriving on
            // PFULL(j) and it is rewritten only after S(j+1) is full)
            xch[h * 128 + row] = mx;
            named_bar_sync(xbar, 64);
            mx = fmaxf(mx, xch[(h ^ 1) * 128 + row]);
          }
          return mx;
        };
        // No row max in the steady state: P = 2^(x - m_run) with the max of the
        // row's first visible tile.  Values above 1 are exact in bf16 / fp32
        // (relative precision), so the max only has to move when a tile's sum
        // nears overflow (>= 2^64, or non-finite) — then it is recomputed
        // exactly and the tile redone.  (m_run is identical in both halves of
        // a row, so both warps of a pair take these branches together.)
        if (__any_sync(0xffffffffu, m_run[u] == -INFINITY)) {
          const float m_new = fmaxf(m_run[u], move_max());
          if (m_new > m_run[u]) {
            alpha = (m_run[u] == -INFINITY) ? 1.f : ex2(m_run[u] - m_new);
            m_run[u] = m_new;
          }
        }
        TR(2 * 8 + t * 4 + quarter, j);
        float tsum = exps(m_run[u] == -INFINITY ? 0.f : m_run[u]);
        bool ovf = __any_sync(0xffffffffu, !(tsum < 0x1p64f));
        if constexpr (CS == 2) ovf = bar_red_or(xbar, 64, ovf);  // one decision for both halves
        if (ovf) {  // rare: S is still in TMEM
          load_s();
          const float m_new = fmaxf(m_run[u], move_max());
          if (m_new > m_run[u]) {
            alpha *= (m_run[u] == -INFINITY) ? 1.f : ex2(m_run[u] - m_new);
            m_run[u] = m_new;
          }
          tsum = exps(m_run[u] == -INFINITY ? 0.f : m_run[u]);
        }
        l_run[u] = l_run[u] * alpha + tsum;
        if (l_run[u] > 0x1p96f) {  // keep the denominator far from fp32 overflow
          l_run[u] *= 0x1p-64f;
          alpha *= 0x1p-64f;
          m_run[u] += 64.f;
        }
        TR(3 * 8 + t * 4 + quarter, j);
        // P_t(j), this half's keys, over S_t columns already consumed (half 1
        // writes columns 32..63 of S, which half 0 loaded before it could
        // reach the P store: both halves passed this tile's barrier.red)
#pragma unroll
        for (int c = 0; c < NC / 64; ++c)
          tmem_st32(p_addr + c * 32, reinterpret_cast<const float*>(pk + c * 32));
        // O_t already holds PV_t(j-1) (its commit preceded S_t(j)'s): rescale
        // this half's columns in place when the running max moved
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < HD / CS / 32; ++c) {
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
        TR(4 * 8 + t * 4 + quarter, j);
        mbar_arrive(bar(L::B_PFULL + t));
      }
    }
    // ------------------------------------------------------------ epilogue
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = CS == 1 ? (sidx >> 2) : u;
      const uint32_t o_addr = tmem + lane_addr + (t ? TM_O1 : TM_O0) + h * (HD / CS);
      float* xch = reinterpret_cast<float*>(smem + L::OFF_XCH) + t * 256;
      const bool present = (t == 0) || has1;
      const TileRef qt = t ? qt1 : qt0;
      if (n_tiles > 0) {
        mbar_wait(bar(L::B_ODONE + t), 0);
        tc_fence_after();
      }
      float l = l_run[u];
      if constexpr (CS == 2) {  // the row's denominator is the sum of both halves
        xch[h * 128 + row] = l;
        named_bar_sync(xbar, 64);
        l += xch[(h ^ 1) * 128 + row];
      }
      if (present)
        f2_epilogue<HD, HD / CS>(p, o_addr, n_tiles > 0, bh, qt.row0 + row, row < qt.nvalid,
                                 m_run[u], l, h * (HD / CS), h == 0);
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

template <int HD, int CS>
int launch_fwd2_hd(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                   const CUtensorMap& tv, cudaStream_t stream) {
  using L = F2Layout<HD>;
  static bool configured[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(fwd2_kernel<HD, CS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(fwd2)");
    configured[dev & 63] = true;
  }
  const int q_tiles = (a.q_map.mode == A2D_IDX_AFFINE && a.q_map.nblocks > 1)
                          ? a.q_map.nblocks * (a.q_map.rows_per_block / TILE)
                          : (a.nq + TILE - 1) / TILE;
  dim3 grid((q_tiles + 1) / 2, a.bh);
  fwd2_kernel<HD, CS><<<grid, F2Threads<CS>::N, L::SMEM, stream>>>(tq, tk, tv, a, q_tiles);
  return check_launch("fwd2_kernel");
}

int launch_tile_fwd2(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                     const CUtensorMap& tv, cudaStream_t stream) {
  // CS = 2 (column-split softmax, 640 threads) measured slower on B200:
  // the SM sub-partitions are throughput-bound, not latency-bound, so the
  // extra warps only add the max exchange (kept for experiments: -DF2X_CS2)
#ifdef F2X_CS2
  constexpr int CS = 2;
#else
  constexpr int CS = 1;
#endif
  // tiles are 64 or 128 columns wide; columns past h are TMA zero fill
  if (a.h > 64) return launch_fwd2_hd<128, CS>(a, tq, tk, tv, stream);
  return launch_fwd2_hd<64, CS>(a, tq, tk, tv, stream);
}

}  // namespace a2d
