// tile_bwd128.cu — Attention2D tile backward on sm_100a (any head dim <= 128;
// the tiles are 128 wide and columns past h are TMA zero fill).
//
// The reference's flash_backward recurrence (numpy_backend.py:46-62), shaped
// so that EVERY tcgen05.mma has N = 128, the shape that runs at the full
// 8192 flop/clk/SM (tools/umma_rate.py: N = 64 shapes are shared-memory
// bound at 61-70%).
//
// One CTA = one 128-key tile of one head; it sweeps 128-query tiles:
//   S^T  = K Q_i^T            -> TMEM X      (SS, M128 N128)
//   dP^T = V dO_i^T           -> TMEM Y      (SS; needs no P, so it runs
//                                             while the exponentials are formed)
//   P^T  = exp2(S^T c - lse)  -> TMEM X (bf16, in place)          [P/dS warpgroups]
//   dV  += P^T dO_i           (TS: A from TMEM)                   -> TMEM dV
//   S_{i+1} -> X              (X is free once dV_i has read P_i: in-order pipe)
//   dS^T = P^T (dP^T - delta) -> smem (bf16, 128B swizzle)          [P/dS warpgroups]
//   dS^T (bf16) also -> TMEM Y (its first 32 columns per warpgroup)
//   dK  += dS^T Q_i           (TS: dS^T from Y)                    -> TMEM dK
//   dQ^T = K^T dS^T           (SS, both MN-major; after dK has read Y) -> TMEM Y
//   dQ   -> registers (Y free again) -> fp32 staging -> TMA bulk reduce-add
// Tensor-pipe order per tile: dP_i, dV_i, S_{i+1}, dK_i, dQ_i.  The P/dS
// warpgroups run P_i then dS_i back to back (dP_i is ready when P_i is), and
// P_{i+1} overlaps dK_i / dQ_i; the dQ drain empties Y while P_{i+1} is
// still being formed (dP_{i+1} waits for it, dV_{i+1} for P_{i+1}).
// dK reads dS^T from TMEM (TS) rather than shared memory: the kernel is
// bound by shared-memory traffic, and this saves 32 KB of
// operand reads per query tile (+1-2% measured).
//
// TMEM (512 cols): dV [0,128) dK [128,256) X [256,384) Y [384,512).
// SMEM (231.6 KB): K, V, 2 x Q, dO, dS^T (B operand of dQ^T), 4 x dQ staging,
// LSE/delta stats.
// Warps (512 threads, register budgets via setmaxnreg):
//   0 TMA producer, 1 MMA issuer, 2-3 idle                         (72 regs)
//   4-7 P/dS warpgroup A (query columns 0-63), 8-11 B (64-127)     (136 regs)
//   12-15 dQ drain: all 128 columns of Y in registers at once       (168 regs)
#include <atomic>
#include "sm100.cuh"
#include "tiles.cuh"
#include "kernels.h"

namespace a2d {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr int THREADS = 512;
constexpr int SLAB = 128 * 128;  // 128 rows x 128 B
constexpr int TILE_B = 2 * SLAB; // one 128 x 128 bf16 tile
constexpr int OFF_K = 0;
constexpr int OFF_V = OFF_K + TILE_B;
constexpr int OFF_Q = OFF_V + TILE_B;      // 2 stages
constexpr int OFF_DO = OFF_Q + 2 * TILE_B;
constexpr int OFF_DS = OFF_DO + TILE_B;
// dQ staging: DQ_BUFS buffers of DQ_ROWS query rows x 128 fp32 (32 KB in all),
// so up to DQ_BUFS TMA bulk reduce-adds are in flight per CTA.  The staging
// stores and the reduce's reads are a quarter of this kernel's shared-memory
// traffic, which is what bounds it: 4 x 16-row buffers
// measured 1-3% faster than 2 x 32, 8 x 8 16% slower; sending any share of
// the rows by red.global.add.v4 from registers instead (scalar, vector,
// coalesced through lane-quad transposes) measured 11-64% slower.
constexpr int DQ_BUFS = 4;
constexpr int DQ_ROWS = 64 / DQ_BUFS;
constexpr int DQ_ROUNDS = 128 / DQ_ROWS;
constexpr int DQ_BUF_BYTES = DQ_ROWS * 128 * 4;
constexpr int OFF_DQ = OFF_DS + TILE_B;
constexpr int OFF_STAT = OFF_DQ + DQ_BUFS * DQ_BUF_BYTES;  // [2][2][128] fp32
constexpr int OFF_BAR = OFF_STAT + 2 * 2 * 128 * 4;
enum {
  B_KV, B_QFULL0, B_QFULL1, B_QEMPTY0, B_QEMPTY1, B_DOFULL, B_DOEMPTY, B_SFULL, B_PREADY,
  B_DPFULL, B_DSREADY, B_DSFREE, B_DQFULL, B_DQFREE, B_DONE, NBAR
};
constexpr int OFF_TMEMPTR = OFF_BAR + NBAR * 8;
// the CTA's query-tile range, computed once by thread 0 and read by every
// role from shared memory (a per-thread copy would live in local memory)
constexpr int OFF_RANGE = OFF_TMEMPTR + 16;
constexpr int SMEM = OFF_RANGE + (int(sizeof(TileRange)) + 15) / 16 * 16;
static_assert(SMEM <= 232448, "shared memory budget");
constexpr uint32_t TM_DV = 0, TM_DK = 128, TM_X = 256, TM_Y = 384;

// F16: fp16 Q/K/V/dO, P and dS (bf16 otherwise)
template <bool F16>
__global__ void __launch_bounds__(THREADS, 1)
    bwd128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                  const __grid_constant__ CUtensorMap tm_dq,
                  const __grid_constant__ a2d_tile_bwd_args p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int bh_kv = p.kv_group > 1 ? bh / p.kv_group : bh;  // GQA / MQA: shared k/v head
  const int kt_idx = blockIdx.x;
  auto bar = [&](int i) { return sb + OFF_BAR + 8 * i; };
  float* stat = reinterpret_cast<float*>(smem + OFF_STAT);
  if ((sb & 1023) != 0) __trap();

  const bool causal = p.causal != 0;
  const TileRef kt = tile_ref(p.k_map, p.nk, kt_idx * TILE);
  if (threadIdx.x == 0) {
    query_range(p.q_map, p.nq, causal, kt.gmin, *reinterpret_cast<TileRange*>(smem + OFF_RANGE),
                TILE);
    mbar_init(bar(B_KV), 1);
    mbar_init(bar(B_QFULL0), 2);  // TMA bytes + the producer's stats arrival
    mbar_init(bar(B_QFULL1), 2);
    mbar_init(bar(B_QEMPTY0), 1);
    mbar_init(bar(B_QEMPTY1), 1);
    mbar_init(bar(B_DOFULL), 1);
    mbar_init(bar(B_DOEMPTY), 1);
    mbar_init(bar(B_SFULL), 1);
    mbar_init(bar(B_PREADY), 256);
    mbar_init(bar(B_DPFULL), 1);
    mbar_init(bar(B_DSREADY), 256);
    mbar_init(bar(B_DSFREE), 1);
    mbar_init(bar(B_DQFULL), 1);
    mbar_init(bar(B_DQFREE), 128);
    mbar_init(bar(B_DONE), 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_dq);
  }
  if (warp == 1) {
    tmem_alloc(sb + OFF_TMEMPTR, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + OFF_TMEMPTR);

  const TileRange& qr = *reinterpret_cast<const TileRange*>(smem + OFF_RANGE);
  const int n_tiles = qr.total;
  const int qrot = kt_idx;  // rotated q sweep: co-resident CTAs reduce into different dQ rows

  // ---------------------------------------------------------------- MMA issue
  // Warp-level helpers (one elected lane issues; whole warp converged):
  // h < 128: ceil(h/16) K steps for K Q^T / V dO^T and N = 16 ceil(h/16)
  // for dV / dK (the tiles' other head columns are zero fill)
  const int ksteps = (p.h + 15) / 16;
  constexpr uint32_t id_ss = make_idesc_bf16(128, 128, 0, 0, F16);   // K Q^T, V dO^T
  const uint32_t id_kmn = make_idesc_bf16(128, ksteps * 16, 0, 1, F16);  // P^T dO, dS^T Q
  constexpr uint32_t id_mnmn = make_idesc_bf16(128, 128, 1, 1, F16); // K^T dS^T
  // K-major SW128: +32 B per K16 step inside a slab, +SLAB per 64 columns;
  // MN-major SW128: +2048 B per K16 step (16 rows of 128 B)
  auto kofs = [](int kk) { return uint64_t(((kk >> 2) * SLAB + (kk & 3) * 32) >> 4); };
  auto mofs = [](int kk) { return uint64_t((kk * 2048) >> 4); };
  constexpr uint64_t QSTEP = TILE_B >> 4;
  auto commit = [&](int b) {
    if (elect_one()) umma_commit(bar(b));
    __syncwarp();
  };
  auto issue_s = [&](uint32_t col, uint64_t a, uint64_t b) {
    a = opaque64(a);
    b = opaque64(b);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        if (kk < ksteps) umma_bf16(tmem + col, a + kofs(kk), b + kofs(kk), id_ss, kk > 0);
    }
    __syncwarp();
  };
  auto issue_dv = [&](int i) {  // dV += P^T dO_i (P^T in TMEM: WG A's queries at X+0, B's at X+64)
    if (elect_one()) {
      const uint64_t dob = opaque64(make_sdesc(sb + OFF_DO, SLAB, 1024));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16_ts(tmem + TM_DV, tmem + TM_X + (kk >> 2) * 64 + (kk & 3) * 8,
                     dob + mofs(kk), id_kmn, (i > 0 || kk > 0));
    }
    __syncwarp();
  };
  // dQ^T = K^T dS^T -> Y, then dK += dS^T Q_i; commits DQFULL, QEMPTY, DSFREE
  auto issue_dq_dk = [&](int i) {
    const int qs = i & 1;
    if (elect_one()) {
      const uint64_t qb = opaque64(make_sdesc(sb + OFF_Q, SLAB, 1024) + qs * QSTEP);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16_ts(tmem + TM_DK, tmem + TM_Y + (kk >> 2) * 64 + (kk & 3) * 8, qb + mofs(kk),
                     id_kmn, (i > 0 || kk > 0));
      umma_commit(bar(B_QEMPTY0 + qs));
      const uint64_t kb = opaque64(make_sdesc(sb + OFF_K, SLAB, 1024));
      const uint64_t dsb = opaque64(make_sdesc(sb + OFF_DS, SLAB, 1024));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16(tmem + TM_Y, kb + mofs(kk), dsb + mofs(kk), id_mnmn, kk > 0);
      umma_commit(bar(B_DQFULL));
      umma_commit(bar(B_DSFREE));
    }
    __syncwarp();
  };
  const uint64_t k_k = make_sdesc(sb + OFF_K, 16, 1024);
  const uint64_t v_k = make_sdesc(sb + OFF_V, 16, 1024);
  const uint64_t do_k = make_sdesc(sb + OFF_DO, 16, 1024);
  const uint64_t q_k = make_sdesc(sb + OFF_Q, 16, 1024);

  if (warp < 4) {
    regs_dec<72>();
    if (warp == 0) {
      // ---------------------------------------------------------- producer
      if (n_tiles > 0) {
        if (lane == 0) {
          mbar_expect_tx(bar(B_KV), 2 * TILE_B);
          for (int s = 0; s < 2; ++s) {
            tma_load_3d(sb + OFF_K + s * SLAB, &tm_k, bar(B_KV), s * 64, kt.row0, bh_kv);
            tma_load_3d(sb + OFF_V + s * SLAB, &tm_v, bar(B_KV), s * 64, kt.row0, bh_kv);
          }
        }
        // the LSE / delta rows of tile i+1 are loaded into registers while tile i
        // is in flight, so their global-load latency never gates S_{i+1}
        TileCursor cur;
        cur.start(qr, qrot);
        float l2n[4], dln[4];
        auto load_stats = [&](int qrow) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int gr = qrow + lane + 32 * k;
            l2n[k] = INFINITY;
            dln[k] = 0.f;
            if (gr < p.nq) {
              const float l = p.lse[(long long)bh * p.nq + gr];
              l2n[k] = (l == -INFINITY) ? INFINITY : l * kLog2e;
              dln[k] = p.delta[(long long)bh * p.nq + gr];
            }
          }
        };
        load_stats(cur.row0(p.q_map));
        for (int i = 0; i < n_tiles; ++i) {
          const int qrow = cur.row0(p.q_map);
          const int qs = i & 1;
          mbar_wait(bar(B_QEMPTY0 + qs), ((i >> 1) & 1) ^ 1);
          if (lane == 0) {
            mbar_expect_tx(bar(B_QFULL0 + qs), TILE_B);
            for (int s = 0; s < 2; ++s)
              tma_load_3d(sb + OFF_Q + qs * TILE_B + s * SLAB, &tm_q, bar(B_QFULL0 + qs), s * 64,
                          qrow, bh);
          }
          float* s_lse = stat + qs * 256;
          float* s_del = s_lse + 128;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            s_lse[lane + 32 * k] = l2n[k];
            s_del[lane + 32 * k] = dln[k];
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(B_QFULL0 + qs));
          cur.next(qr);
          if (i + 1 < n_tiles) load_stats(cur.row0(p.q_map));
          if (lane == 0) {
            mbar_wait(bar(B_DOEMPTY), (i & 1) ^ 1);
            mbar_expect_tx(bar(B_DOFULL), TILE_B);
            for (int s = 0; s < 2; ++s)
              tma_load_3d(sb + OFF_DO + s * SLAB, &tm_do, bar(B_DOFULL), s * 64, qrow, bh);
          }
          __syncwarp();
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      // whole warp: warp-uniform control flow keeps descriptors in uniform
      // registers; one elected lane issues (the single-lane version issued
      // one MMA per ~70 cycles, slower than the 64-cycle N=128 MMA itself)
      if (n_tiles > 0) {
        mbar_wait(bar(B_KV), 0);
        mbar_wait(bar(B_QFULL0), 0);
        tc_fence_after();
        issue_s(TM_X, k_k, q_k);
        commit(B_SFULL);
        for (int i = 0; i < n_tiles; ++i) {
          const int qs = i & 1;
          // dP^T = V dO_i^T -> Y, once the drain has emptied dQ_{i-1} out of it
          mbar_wait(bar(B_DOFULL), i & 1);
          if (i > 0) mbar_wait(bar(B_DQFREE), (i - 1) & 1);
          tc_fence_after();
          issue_s(TM_Y, v_k, do_k);
          commit(B_DPFULL);
          mbar_wait(bar(B_PREADY), i & 1);
          tc_fence_after();
          issue_dv(i);
          commit(B_DOEMPTY);
          // S_{i+1} -> X: dV_i has read P_i out of X (in-order pipe)
          if (i + 1 < n_tiles) {
            mbar_wait(bar(B_QFULL0 + (qs ^ 1)), ((i + 1) >> 1) & 1);
            tc_fence_after();
            issue_s(TM_X, k_k, q_k + (qs ^ 1) * QSTEP);
            commit(B_SFULL);
          }
          // dQ^T = K^T dS^T -> Y (dP_i was read out of Y before dS_i was published),
          // then dK += dS^T Q_i while the drain empties Y
          mbar_wait(bar(B_DSREADY), i & 1);
          tc_fence_after();
          issue_dq_dk(i);
        }
        commit(B_DONE);
      }
    }
  } else if (warp < 12) {
    regs_inc<136>();
    // ------------------------------------------------------------ P / dS warpgroups
    const int wg = (warp - 4) >> 2;  // 0: query columns 0-63, 1: 64-127
    const int quarter = warp & 3;
    const int jj = quarter * 32 + lane;  // key row within the tile
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    const int c0 = wg * 64;
    const float sl2 = p.scale * kLog2e;
    const bool row_ok = jj < kt.nvalid;
    const bool affine = p.q_map.mode != A2D_IDX_ARRAY;
    // causal threshold of query block b against this key tile, ceil((kt.gmin -
    // base_b) / s): one division per block change instead of one per tile
    // Per-tile causal classes (threshold, valid query columns, full flag)
    // for affine maps are computed 32 tiles at a time, one tile per lane,
    // and broadcast with one shuffle per tile; explicit index arrays keep a
    // per-tile path.
    const int rot0 = n_tiles > 0 ? qrot % n_tiles : 0;
    uint32_t my_info = 0;
    TileCursor cur;
    if (!affine) cur.start(qr, qrot);
    for (int i = 0; i < n_tiles; ++i) {
      const int qs = i & 1;
      int first = 0;  // first visible query column of this key row
      bool full = true;
      if (!affine) {
        const int qrow0 = cur.row0(p.q_map);
        cur.next(qr);
        const int qvalid = min(TILE, p.nq - qrow0);
        if (causal) {
          const TileRef qt = tile_ref(p.q_map, p.nq, qrow0, TILE);
          PairMask pm;
          pm.partial = true;
          pm.thr = 0;
          pm.kvalid = kt.nvalid;
          first = col_first(p.q_map, p.k_map, qt, kt, pm, true, jj);
          full = false;
        }
        full = full && kt.nvalid == TILE && qvalid == TILE;
      } else {
        if ((i & 31) == 0) {
          const int f = i + lane;
          my_info = 0;
          if (f < n_tiles) {
            const int g = rot0 + f < n_tiles ? rot0 + f : rot0 + f - n_tiles;
            int b, t;
            range_pos(qr, g, b, t);
            const int rpb = p.q_map.nblocks == 1 ? 0 : p.q_map.rows_per_block;
            const int qrow0 = b * rpb + t * TILE;
            const int qend = p.q_map.nblocks == 1 ? p.nq : (b + 1) * rpb;
            const int qvalid = min(TILE, qend - qrow0);
            long long thr = -(long long)(2 * TILE);
            if (causal) {
              thr = ceil_div_s(kt.gmin - p.q_map.base[b], p.q_map.stride) - (long long)TILE * t;
              thr = max(-(long long)(2 * TILE), min((long long)(2 * TILE), thr));
            }
            const bool fl = thr <= -(TILE - 1) && kt.nvalid == TILE && qvalid == TILE;
            my_info = uint32_t(thr + 512) | (uint32_t(qvalid) << 16) | (fl ? 0x80000000u : 0u);
          }
        }
        const uint32_t inf = __shfl_sync(0xffffffffu, my_info, i & 31);
        full = (inf >> 31) != 0;
        first = causal ? jj + (int(inf & 0xffff) - 512) : 0;
      }
      if (!row_ok) first = TILE;
      const float* s_lse = stat + qs * 256 + c0;
      const float* s_del = s_lse + 128;
      mbar_wait(bar(B_QFULL0 + qs), (i >> 1) & 1);  // orders the producer's stats stores
      mbar_wait(bar(B_SFULL), i & 1);
      tc_fence_after();
      float pr[64];
      tmem_ld32(tmem + lane_addr + TM_X + c0, pr);
      tmem_ld32(tmem + lane_addr + TM_X + c0 + 32, pr + 32);
      tmem_wait_ld();
      uint32_t pk[32];
      const float2 sc = make_float2(sl2, sl2);
      if (full) {
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 x = ffma2(make_float2(pr[c], pr[c + 1]), sc,
                                 make_float2(-s_lse[c], -s_lse[c + 1]));
          // every exponential on MUFU: moving a quarter of them to the
          // FMA-pipe polynomial measured 1-2% slower (profiles/r2_ab.md)
          const float2 e = make_float2(ex2(x.x), ex2(x.y));
          pk[c >> 1] = pack2<F16>(e.x, e.y);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 x = ffma2(make_float2(pr[c], pr[c + 1]), sc,
                                 make_float2(-s_lse[c], -s_lse[c + 1]));
          const float e0 = (c0 + c >= first) ? ex2(x.x) : 0.f;
          const float e1 = (c0 + c + 1 >= first) ? ex2(x.y) : 0.f;
          pk[c >> 1] = pack2<F16>(e0, e1);
        }
      }
      // P^T (bf16 pairs) over the first 32 columns of this warpgroup's S slice
      tmem_st32(tmem + lane_addr + TM_X + c0, reinterpret_cast<const float*>(pk));
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(B_PREADY));

      mbar_wait(bar(B_DPFULL), i & 1);
      tc_fence_after();
      // dS = P (dP - delta), with P re-read from its 16-bit pairs (the same
      // rounded P that fed dV)
      float dpa[64];
      tmem_ld32(tmem + lane_addr + TM_Y + c0, dpa);
      tmem_ld32(tmem + lane_addr + TM_Y + c0 + 32, dpa + 32);
      tmem_wait_ld();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float* dp = dpa + 32 * h;
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const float2 d = fadd2(make_float2(dp[c], dp[c + 1]),
                                 make_float2(-s_del[32 * h + c], -s_del[32 * h + c + 1]));
          const float2 pf = unpack2<F16>(pk[(32 * h + c) >> 1]);
          const float2 ds = fmul2(pf, d);
          pk[(32 * h + c) >> 1] = pack2<F16>(ds.x, ds.y);
        }
      }
      // dS^T (bf16 pairs) into this warpgroup's first 32 columns of Y: the
      // A operand of dK (TS); the same layout as P^T in X
      tmem_st32(tmem + lane_addr + TM_Y + c0, reinterpret_cast<const float*>(pk));
      tmem_wait_st();
      tc_fence_before();  // the dP^T loads / dS^T stores are done before Y is handed back
      if (i > 0) mbar_wait(bar(B_DSFREE), (i - 1) & 1);
      // dS^T row jj -> K-major SW128 slab `wg` (64 queries = 128 B per row)
      const uint32_t drow = sb + OFF_DS + wg * SLAB + jj * 128;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
        st_shared_v4(drow + ((cc ^ (jj & 7)) << 4), pk[cc * 4], pk[cc * 4 + 1], pk[cc * 4 + 2],
                     pk[cc * 4 + 3]);
      fence_proxy_async_smem();
      mbar_arrive(bar(B_DSREADY));
    }
    // ------------------------------------------------------------ dV (A) / dK (B) epilogue
    if (n_tiles > 0) {
      mbar_wait(bar(B_DONE), 0);
      tc_fence_after();
    }
    const uint32_t col0 = wg == 0 ? TM_DV : TM_DK;
    void* base = wg == 0 ? p.dv : p.dk;
    const float mul = wg == 0 ? 1.f : p.scale;
    const long long grow = (long long)kt.row0 + jj;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float v[32];
      if (n_tiles > 0) {
        tmem_ld32(tmem + lane_addr + col0 + c * 32, v);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0.f;
      }
      if (!row_ok || c * 32 >= p.h) continue;  // columns past h are TMA zero fill
      const long long off = (long long)bh * p.dkv_stride_bh + grow * p.dkv_stride_row + c * 32;
      if (p.dkv_dtype == A2D_F32) {
        float* dst = reinterpret_cast<float*>(base) + off;
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          if (c * 32 + e >= p.h) continue;
          float4 w = make_float4(v[e] * mul, v[e + 1] * mul, v[e + 2] * mul, v[e + 3] * mul);
          if (p.accumulate_dkv) {
            const float4 o = *reinterpret_cast<const float4*>(dst + e);
            w.x += o.x; w.y += o.y; w.z += o.z; w.w += o.w;
          }
          *reinterpret_cast<float4*>(dst + e) = w;
        }
      } else {  // bf16 or fp16 dK / dV
        uint16_t* dst = reinterpret_cast<uint16_t*>(base) + off;
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          if (c * 32 + e >= p.h) continue;
          uint4 u;
          u.x = pack_out(p.dkv_dtype, v[e] * mul, v[e + 1] * mul);
          u.y = pack_out(p.dkv_dtype, v[e + 2] * mul, v[e + 3] * mul);
          u.z = pack_out(p.dkv_dtype, v[e + 4] * mul, v[e + 5] * mul);
          u.w = pack_out(p.dkv_dtype, v[e + 6] * mul, v[e + 7] * mul);
          *reinterpret_cast<uint4*>(dst + e) = u;
        }
      }
    }
  } else {
    regs_inc<168>();
    // ------------------------------------------------------------ dQ drain
    const int quarter = warp & 3;
    const int h = quarter * 32 + lane;  // TMEM lane = head dim of dQ^T
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    int round = 0;
    TileCursor cur;
    cur.start(qr, qrot);
    for (int i = 0; i < n_tiles; ++i, cur.next(qr)) {
      const int qrow = cur.row0(p.q_map);
      mbar_wait(bar(B_DQFULL), i & 1);
      tc_fence_after();
      // all 128 query columns at once: Y is handed back before any staging
      float v[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lane_addr + TM_Y + 32 * c, v + 32 * c);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(B_DQFREE));
#pragma unroll
      for (int r = 0; r < DQ_ROUNDS; ++r) {
        const uint32_t buf = sb + OFF_DQ + (round % DQ_BUFS) * DQ_BUF_BYTES;
        ++round;
        // this buffer's previous reduce has read it
        if (h == 0) bulk_wait_group_read<DQ_BUFS - 1>();
        named_bar_sync(1, 128);
        // row-major [DQ_ROWS q][128 h] fp32: a warp's 32 head dims are one 128 B row
#pragma unroll
        for (int q = 0; q < DQ_ROWS; ++q) {
          const uint32_t addr = buf + q * 512 + h * 4;
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v[DQ_ROWS * r + q]) : "memory");
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 128);
        if (h == 0) {
          tma_reduce_add_3d_g(&tm_dq, buf, 0, qrow + DQ_ROWS * r, bh);
          bulk_commit_group();
        }
      }
    }
    if (h == 0) bulk_wait_group_all();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

int bwd_q_tile_rows(int) { return TILE; }

int launch_tile_bwd(const a2d_tile_bwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                  const CUtensorMap& tv, const CUtensorMap& tdo, cudaStream_t stream) {
  // per (operand type, device): cudaFuncSetAttribute once (idempotent, so a
  // racing first call from two host threads is harmless; atomic for the flag)
  static std::atomic<bool> configured[2][64];
  const bool f16 = a.in_dtype == A2D_F16;
  auto kern = f16 ? bwd128_kernel<true> : bwd128_kernel<false>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[f16][dev & 63].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(bwd128)");
    configured[f16][dev & 63].store(true, std::memory_order_release);
  }
  CUtensorMap tdq;
  int rc = make_map_f32_dq_flat(&tdq, a.dq_acc, a.h, a.nq, a.bh, a.dq_stride_row, a.dq_stride_bh,
                                    DQ_ROWS, 128);
  if (rc) return rc;
  const int k_tiles = (a.k_map.mode == A2D_IDX_AFFINE && a.k_map.nblocks > 1)
                          ? a.k_map.nblocks * (a.k_map.rows_per_block / TILE)
                          : (a.nk + TILE - 1) / TILE;
  dim3 grid(k_tiles, a.bh);
  kern<<<grid, THREADS, SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
  return check_launch("bwd128_kernel");
}

}  // namespace a2d
