// tile_fwd2.cu — Attention2D tile forward on sm_100a, two query tiles per CTA.
//
// The streaming softmax of the reference's flash_forward
// (numpy_backend.py:24-43 / numba_backend.py:38-76), emitting the (O, LSE)
// partial that attn_fix merges (attention.py:194-214).  Each CTA owns TWO
// 128-row query tiles of one head and sweeps their common key range once, so
// the tensor pipe never waits for one softmax warpgroup.
//
// Warp roles (one CTA per SM, 384 threads):
//   warp 0       TMA producer: Q0/Q1 once, then K (3-stage) / V (2-stage) rings
//   warp 1       tcgen05 MMA issuer (whole warp, one elected lane issues)
//   warps 2-3    idle (complete the register-reallocation warpgroup)
//   warps 4-7    softmax warpgroup of query tile 0, warps 8-11 of tile 1;
//                warp w owns TMEM lanes 32*(w%4)..+31 (one query row per
//                thread, all 128 key columns).  A column-split softmax (two
//                threads per row, max exchange through shared memory) was
//                measured 5-10% slower: the sub-partitions are throughput-
//                bound, not latency-bound.
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
#include <atomic>
#include "sm100.cuh"
#include "tiles.cuh"
#include "kernels.h"

// one exponential pair in eight on the FMA-pipe polynomial (MUFU offload;
// measured best on B200 once the row-max tree is gone: 0, 1/4, 3/8 and 1/2
// were slower)
#define F2_POLY(jj) ((((jj) >> 1) & 7) == 7)

// clock64 instrumentation points; tools/mk_trace_lib.sh builds a traced copy
// of the library with -DA2D_TRACE (the product build compiles them away)
#ifdef A2D_TRACE
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

template <int HD>
struct F2Layout {
  static constexpr int SLAB = TILE * 128;  // one 128-row x 64-col bf16 slab
  static constexpr int SLABS = HD / 64;
  static constexpr int TILE_BYTES = SLAB * SLABS;
  static constexpr int KST = 3;  // 2 stages measured equal; the third is slack
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
  // the CTA's key-tile range, computed once by thread 0: every role reads it
  // from shared memory (a per-thread copy would live in local memory)
  static constexpr int OFF_RANGE = OFF_TMEMPTR + 16;
  static constexpr int SMEM = OFF_RANGE + (int(sizeof(TileRange)) + 15) / 16 * 16;
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
    } else {  // final O in bf16 or fp16
      uint16_t* dst = reinterpret_cast<uint16_t*>(p.o) + (long long)bh * p.o_stride_bh +
                      (long long)grow * p.o_stride_row + col0 + c * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        if (col0 + c * 32 + i >= p.h) continue;
        uint4 v;
        v.x = pack_out(p.o_dtype, o[i + 0] * w_new, o[i + 1] * w_new);
        v.y = pack_out(p.o_dtype, o[i + 2] * w_new, o[i + 3] * w_new);
        v.z = pack_out(p.o_dtype, o[i + 4] * w_new, o[i + 5] * w_new);
        v.w = pack_out(p.o_dtype, o[i + 6] * w_new, o[i + 7] * w_new);
        *reinterpret_cast<uint4*>(dst + i) = v;
      }
    }
  }
}

constexpr int F2_THREADS = 384;  // producer/MMA warpgroup + 8 softmax warps

// F16: fp16 Q/K/V and P (bf16 otherwise); everything else is shared
template <int HD, bool F16>
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
  const int bh_kv = p.kv_group > 1 ? bh / p.kv_group : bh;  // GQA / MQA: shared k/v head
  const int pair = gridDim.x - 1 - blockIdx.x;
  auto bar = [&](int i) { return sb + L::OFF_BAR + 8 * i; };
  const uint32_t TM_O0 = 256, TM_O1 = 256 + HD;

  const bool causal = p.causal != 0;
  const int t0 = 2 * pair, t1 = 2 * pair + 1;
  const bool has1 = t1 < q_tiles;
  const TileRef qt0 = tile_ref(p.q_map, p.nq, t0 * TILE);
  TileRef qt1 = qt0;
  if (has1) qt1 = tile_ref(p.q_map, p.nq, t1 * TILE);
  if (threadIdx.x == 0) {
    key_range(p.k_map, p.nk, causal, has1 ? max(qt0.gmax, qt1.gmax) : qt0.gmax,
              *reinterpret_cast<TileRange*>(smem + L::OFF_RANGE));
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

  const TileRange& kr = *reinterpret_cast<const TileRange*>(smem + L::OFF_RANGE);
  const int n_tiles = kr.total;
  const int rot = pair;  // rotated key sweep

  if (warp < 4) {
    regs_dec<80>();
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
        mbar_wait_sleep(bar(L::B_KEMPTY + ks), kph ^ 1);
        TR(45, j);
        mbar_expect_tx(bar(L::B_KFULL + ks), L::TILE_BYTES);
        for (int s = 0; s < L::SLABS; ++s)
          tma_load_3d(sb + L::OFF_K + ks * L::TILE_BYTES + s * L::SLAB, &tm_k,
                      bar(L::B_KFULL + ks), s * 64, krow, bh_kv);
        if (++ks == L::KST) { ks = 0; kph ^= 1; }
        mbar_wait_sleep(bar(L::B_VEMPTY + vs), vph ^ 1);
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
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0, 0, F16);
      const uint32_t idesc_pv = make_idesc_bf16(128, ksteps * 16, 0, 1, F16);
      int ks = 0, kph = 0, vs = 0, vph = 0;
      mbar_wait_sleep(bar(L::B_Q), 0);
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
      mbar_wait_sleep(bar(L::B_KFULL + ks), kph);
      tc_fence_after();
      issue_qk(0);
      issue_qk(1);
      commit(L::B_KEMPTY + ks);
      if (++ks == L::KST) { ks = 0; kph ^= 1; }
      for (int j = 0; j < n_tiles; ++j) {
        const bool more = j + 1 < n_tiles;
        mbar_wait_sleep(bar(L::B_VFULL + vs), vph);
        TR(44, j);
        // ---- tile 0: PV0(j), QK0(j+1)
        mbar_wait_sleep(bar(L::B_PFULL + 0), j & 1);
        tc_fence_after();
        TR(40, j);
        issue_pv(0, j);
        if (more) {
          mbar_wait_sleep(bar(L::B_KFULL + ks), kph);
          tc_fence_after();
          issue_qk(0);
          TR(41, j);
        } else {
          commit(L::B_ODONE + 0);
        }
        // ---- tile 1: PV1(j), QK1(j+1)
        mbar_wait_sleep(bar(L::B_PFULL + 1), j & 1);
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
    regs_inc<208>();
    // ------------------------------------------------------------ softmax warps
    // warp w owns query tile t = (w-4)/4, all 128 key columns
    constexpr int NC = TILE;  // key columns of S per thread and tile
    const int t = (warp - 4) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    const float sl2 = p.scale * kLog2e;
    const bool arr = p.q_map.mode == A2D_IDX_ARRAY;
    const int rot0 = n_tiles > 0 ? rot % n_tiles : 0;
    float m_run = -INFINITY;  // running max of scale*log2e*s
    float l_run = 0.f;        // running denominator
    uint32_t my_info = 0;
    TileCursor cur;
    if (arr) cur.start(kr, rot);
    const uint32_t s_addr = tmem + lane_addr + t * 128;
    const uint32_t o_addr = tmem + lane_addr + (t ? TM_O1 : TM_O0);
    const bool present = (t == 0) || has1;
    const TileRef qt = t ? qt1 : qt0;
    for (int j = 0; j < n_tiles; ++j) {
      // Per-tile mask classes for affine maps are computed 32 tiles at a
      // time, one tile per lane, and broadcast with one shuffle per tile;
      // explicit index arrays keep the per-tile binary-search path.
      bool partial;
      int lim = TILE - 1;  // last visible key column of this row (tile-relative)
      if (!present) {
        partial = true;
        lim = -1;
      } else if (arr) {
        const TileRef kt = tile_ref(p.k_map, p.nk, cur.row0(p.k_map));
        cur.next(kr);
        const PairMask pm = pair_mask(p.q_map, qt, kt, causal);
        partial = pm.partial;
        if (partial) lim = row_limit(p.q_map, p.k_map, qt, kt, pm, causal, row);
      } else {
        if ((j & 31) == 0) {
          const int f = j + lane;
          my_info = 0;
          if (f < n_tiles) {
            const int g = rot0 + f < n_tiles ? rot0 + f : rot0 + f - n_tiles;
            const TileRef kt = tile_ref(p.k_map, p.nk, range_row0(kr, p.k_map, g));
            const PairMask q = pair_mask(p.q_map, qt, kt, causal);
            my_info = uint32_t(q.thr + 512) | (uint32_t(q.kvalid) << 16) |
                      (q.partial ? 0x80000000u : 0u);
          }
        }
        const uint32_t inf = __shfl_sync(0xffffffffu, my_info, j & 31);
        partial = (inf >> 31) != 0;
        if (partial) {
          const int kvalid = int((inf >> 16) & 0xff);
          lim = causal ? min(row - (int(inf & 0xffff) - 512), kvalid - 1) : kvalid - 1;
        }
      }
      mbar_wait(bar(L::B_SFULL + t), j & 1);
      tc_fence_after();
      TR(0 * 8 + t * 4 + quarter, j);
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
            const float2 e = make_float2(ex2(x.x), ex2(x.y));
            acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
            pk[jj / 2] = pack2<F16>(e.x, e.y);
          }
        } else {  // some exponentials on the FMA pipe (MUFU offload, F2_POLY)
#pragma unroll
          for (int jj = 0; jj < NC; jj += 2) {
            const float2 x = ffma2(make_float2(s[jj], s[jj + 1]), sc, nb);
            float2 e;
            if (F2_POLY(jj)) e = exp2_poly2(x);
            else e = make_float2(ex2(x.x), ex2(x.y));
            acc[(jj >> 1) & 3] = fadd2(acc[(jj >> 1) & 3], e);
            pk[jj / 2] = pack2<F16>(e.x, e.y);
          }
        }
        const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
        const float2 a = fadd2(a01, a23);
        return a.x + a.y;
      };
      // No row max in the steady state: P = 2^(x - m_run) with the max of the
      // row's first visible tile.  Values above 1 are exact in bf16 / fp32
      // (relative precision), so the max only has to move when a tile's sum
      // nears overflow (>= 2^64, or non-finite) — then it is recomputed
      // exactly and the tile redone.  fp16 P has a 2^16 range, so there the
      // bound is a tile sum of 2^15 (every element then fits).
      if (__any_sync(0xffffffffu, m_run == -INFINITY)) {
        const float m_new = fmaxf(m_run, rowmax<NC>(s) * sl2);
        if (m_new > m_run) {
          alpha = (m_run == -INFINITY) ? 1.f : ex2(m_run - m_new);
          m_run = m_new;
        }
      }
      TR(2 * 8 + t * 4 + quarter, j);
      float tsum = exps(m_run == -INFINITY ? 0.f : m_run);
      if (__any_sync(0xffffffffu, !(tsum < (F16 ? 0x1p15f : 0x1p64f)))) {  // rare: S still in TMEM
        load_s();
        const float m_new = fmaxf(m_run, rowmax<NC>(s) * sl2);
        if (m_new > m_run) {
          alpha *= (m_run == -INFINITY) ? 1.f : ex2(m_run - m_new);
          m_run = m_new;
        }
        tsum = exps(m_run == -INFINITY ? 0.f : m_run);
      }
      // Every tile adds less than 2^64 (else it was re-based above, after
      // which its entries are <= 1), so l_run < 2^64 * n_tiles <= 2^88 for
      // any row count the ABI accepts: no denominator overflow guard is needed.
      l_run = l_run * alpha + tsum;
      TR(3 * 8 + t * 4 + quarter, j);
      // P_t(j) over the first 64 columns of S_t (already consumed)
#pragma unroll
      for (int c = 0; c < NC / 64; ++c)
        tmem_st32(s_addr + c * 32, reinterpret_cast<const float*>(pk + c * 32));
      // O_t already holds PV_t(j-1) (its commit preceded S_t(j)'s): rescale
      // it in place when the running max moved
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
      TR(4 * 8 + t * 4 + quarter, j);
      mbar_arrive(bar(L::B_PFULL + t));
    }
    // ------------------------------------------------------------ epilogue
    if (n_tiles > 0) {
      mbar_wait(bar(L::B_ODONE + t), 0);
      tc_fence_after();
    }
    if (present)
      f2_epilogue<HD, HD>(p, o_addr, n_tiles > 0, bh, qt.row0 + row, row < qt.nvalid, m_run,
                          l_run, 0, true);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace

template <int HD, bool F16>
int launch_fwd2_hd(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                   const CUtensorMap& tv, cudaStream_t stream) {
  using L = F2Layout<HD>;
  static std::atomic<bool> configured[64];  // see launch_tile_bwd
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(fwd2_kernel<HD, F16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(fwd2)");
    configured[dev & 63].store(true, std::memory_order_release);
  }
  const int q_tiles = (a.q_map.mode == A2D_IDX_AFFINE && a.q_map.nblocks > 1)
                          ? a.q_map.nblocks * (a.q_map.rows_per_block / TILE)
                          : (a.nq + TILE - 1) / TILE;
  dim3 grid((q_tiles + 1) / 2, a.bh);
  fwd2_kernel<HD, F16><<<grid, F2_THREADS, L::SMEM, stream>>>(tq, tk, tv, a, q_tiles);
  return check_launch("fwd2_kernel");
}

int launch_tile_fwd(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, cudaStream_t stream) {
  // tiles are 64 or 128 columns wide; columns past h are TMA zero fill
  const bool f16 = a.in_dtype == A2D_F16;
  if (a.h > 64)
    return f16 ? launch_fwd2_hd<128, true>(a, tq, tk, tv, stream)
               : launch_fwd2_hd<128, false>(a, tq, tk, tv, stream);
  return f16 ? launch_fwd2_hd<64, true>(a, tq, tk, tv, stream)
             : launch_fwd2_hd<64, false>(a, tq, tk, tv, stream);
}

}  // namespace a2d
