// tile_bwd.cu — Attention2D tile backward on sm_100a.
//
// The reference's flash_backward (pkg/src/attn2d/kernels/numpy_backend.py:46-62,
// numba_backend.py:79-102) recomputes P = exp(s - m)/d from the GLOBAL row
// statistics and accumulates
//     dV += P^T dO,  dS = P * (dO V^T - delta),  dQ += dS K scale,  dK += dS^T Q scale
// for whatever key subset it is given, so key-subset calls are exact partial
// sums (attention.py:225-257).  Here one CTA owns a 128-row key tile of one
// head (dK/dV accumulate in TMEM for the whole sweep) and walks the query
// sub-tiles that attend it:
//
//   S^T  = K Q_i^T      (M=128 keys, N=QT queries)        -> TMEM
//   dP^T = V dO_i^T                                        -> TMEM
//   P^T  = exp2(S^T scale log2e - lse_i log2e)   (softmax WG, bf16 -> smem)
//   dS^T = P^T (dP^T - delta_i)                   (softmax WG, bf16 -> smem)
//   dV  += P^T dO_i ;  dK += dS^T Q_i             (TMEM accumulators)
//   dQ_i: H=128: dQ^T = K^T dS^T (M=128 head dims, N=64) ; H=64: dQ = dS K
//         -> TMEM -> fp32 smem tile -> TMA bulk reduce-add into dq_acc.
//
// Warp roles (320 threads): warp 0 TMA producer (+ lse/delta staging),
// warp 1 MMA issuer + TMEM owner, warps 2-5 softmax/dS warpgroup (one key
// row per thread), warps 6-9 dQ drain warpgroup.
#include "sm100.cuh"
#include "tiles.cuh"
#include "kernels.h"

#ifdef A2D_X_MMA_ONLY
#define XWAIT(b, ph) ((void)0)
#define XLOOP 0
#else
#define XWAIT(b, ph) mbar_wait(b, ph)
#define XLOOP 1
#endif

namespace a2d {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr int BWD_THREADS = 320;
constexpr uint32_t TMEM_COLS = 512;

A2D_DEV void tma_reduce_add_3d(const void* map, uint32_t src, int c0, int c1, int c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group"
      " [%0, {%2, %3, %4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
A2D_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
A2D_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
A2D_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int HD>
struct BwdLayout {
  static constexpr int QT = (HD == 128) ? 64 : 128;  // query rows per sub-tile
  static constexpr bool DQ_T = (HD == 128);          // dQ^T = K^T dS^T
  static constexpr int HS = HD / 64;                  // 64-col slabs per head row
  static constexpr int KSLAB = 128 * 128;             // 128 rows x 128 B
  static constexpr int QSLAB = QT * 128;              // QT rows x 128 B
  static constexpr int KV_BYTES = HS * KSLAB;         // K (or V) tile
  static constexpr int Q_BYTES = HS * QSLAB;          // Q (or dO) sub-tile
  static constexpr int PS = QT / 64;                  // slabs of a [128 x QT] P / dS tile
  static constexpr int P_BYTES = PS * KSLAB;
  static constexpr int DQ_SLAB = QT * 128;            // QT rows x 32 fp32
  static constexpr int DQ_BYTES = (HD / 32) * DQ_SLAB;
  static constexpr int ST = (HD == 128) ? 3 : 2;      // Q/dO stages
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV_BYTES;
  static constexpr int OFF_Q = OFF_V + KV_BYTES;
  static constexpr int OFF_DO = OFF_Q + ST * Q_BYTES;
  static constexpr int OFF_P = OFF_DO + ST * Q_BYTES;
  static constexpr int OFF_DS = OFF_P + P_BYTES;
  static constexpr int OFF_DQ = OFF_DS + P_BYTES;
  static constexpr int OFF_STAT = OFF_DQ + DQ_BYTES;  // [ST][2][QT] fp32 (lse2, delta)
  static constexpr int OFF_BAR = OFF_STAT + ST * 2 * QT * 4;
  static constexpr int B_KV = 0;
  static constexpr int B_QFULL = 1;
  static constexpr int B_QEMPTY = B_QFULL + ST;
  static constexpr int B_SFULL = B_QEMPTY + ST;
  static constexpr int B_DPFULL = B_SFULL + 1;
  static constexpr int B_PREADY = B_DPFULL + 1;
  static constexpr int B_DSREADY = B_PREADY + 1;
  static constexpr int B_PFREE = B_DSREADY + 1;
  static constexpr int B_DSFREE = B_PFREE + 1;
  static constexpr int B_DQFULL = B_DSFREE + 1;
  static constexpr int B_DQFREE = B_DQFULL + 1;
  static constexpr int B_DONE = B_DQFREE + 1;
  static constexpr int NBAR = B_DONE + 1;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NBAR * 8;
  static constexpr int SMEM = OFF_TMEMPTR + 16 + 1024;
  // TMEM columns
  static constexpr uint32_t TM_DV = 0;
  static constexpr uint32_t TM_DK = HD;
  static constexpr uint32_t TM_S = 2 * HD;
  static constexpr uint32_t TM_DP = TM_S + QT;
  static constexpr uint32_t TM_DQ = TM_DP + QT;
  static_assert(TM_DQ + (DQ_T ? QT : HD) <= TMEM_COLS, "TMEM budget");
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <int HD>
__global__ void __launch_bounds__(BWD_THREADS, 1)
    bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ a2d_tile_bwd_args p) {
  using L = BwdLayout<HD>;
  constexpr int QT = L::QT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int bh_kv = p.kv_group > 1 ? bh / p.kv_group : bh;  // GQA / MQA: shared k/v head
  const int kt_idx = blockIdx.x;
  auto bar = [&](int i) { return sb + L::OFF_BAR + 8 * i; };
  float* stat = reinterpret_cast<float*>(smem + L::OFF_STAT);

  if (threadIdx.x == 0) {
    mbar_init(bar(L::B_KV), 1);
    for (int i = 0; i < L::ST; ++i) {
      mbar_init(bar(L::B_QFULL + i), 1);
      mbar_init(bar(L::B_QEMPTY + i), 1);
    }
    mbar_init(bar(L::B_SFULL), 1);
    mbar_init(bar(L::B_DPFULL), 1);
    mbar_init(bar(L::B_PREADY), 128);
    mbar_init(bar(L::B_DSREADY), 128);
    mbar_init(bar(L::B_PFREE), 1);
    mbar_init(bar(L::B_DSFREE), 1);
    mbar_init(bar(L::B_DQFULL), 1);
    mbar_init(bar(L::B_DQFREE), 128);
    mbar_init(bar(L::B_DONE), 1);
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
    tmem_alloc(sb + L::OFF_TMEMPTR, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + L::OFF_TMEMPTR);

  const bool causal = p.causal != 0;
  const TileRef kt = tile_ref(p.k_map, p.nk, kt_idx * TILE);
  TileRange qr;
  query_range(p.q_map, p.nq, causal, kt.gmin, qr, QT);
  const int n_tiles = qr.total;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (n_tiles > 0) {
      if (lane == 0) {
        mbar_expect_tx(bar(L::B_KV), 2 * L::KV_BYTES);
        for (int s = 0; s < L::HS; ++s) {
          tma_load_3d(sb + L::OFF_K + s * L::KSLAB, &tm_k, bar(L::B_KV), s * 64, kt.row0, bh_kv);
          tma_load_3d(sb + L::OFF_V + s * L::KSLAB, &tm_v, bar(L::B_KV), s * 64, kt.row0, bh_kv);
        }
      }
      TileCursor cur;
      cur.start(qr);
      int st = 0, ph = 0;
      for (int i = 0; i < n_tiles; ++i, cur.next(qr)) {
        const int qrow = cur.row0(p.q_map, QT);
        mbar_wait(bar(L::B_QEMPTY + st), ph ^ 1);
        // global row statistics of this sub-tile: lse*log2e and delta;
        // rows past the end (and empty rows) get lse2 = +inf so P = 0.
        float* s_lse = stat + st * 2 * QT;
        float* s_del = s_lse + QT;
        for (int r = lane; r < QT; r += 32) {
          const int gr = qrow + r;
          float l2 = INFINITY, dl = 0.f;
          if (gr < p.nq) {
            const float l = p.lse[(long long)bh * p.nq + gr];
            l2 = (l == -INFINITY) ? INFINITY : l * kLog2e;
            dl = p.delta[(long long)bh * p.nq + gr];
          }
          s_lse[r] = l2;
          s_del[r] = dl;
        }
        __syncwarp();
        if (lane == 0) {
          mbar_expect_tx(bar(L::B_QFULL + st), 2 * L::Q_BYTES);
          for (int s = 0; s < L::HS; ++s) {
            tma_load_3d(sb + L::OFF_Q + st * L::Q_BYTES + s * L::QSLAB, &tm_q,
                        bar(L::B_QFULL + st), s * 64, qrow, bh);
            tma_load_3d(sb + L::OFF_DO + st * L::Q_BYTES + s * L::QSLAB, &tm_do,
                        bar(L::B_QFULL + st), s * 64, qrow, bh);
          }
        }
        __syncwarp();
        if (++st == L::ST) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, QT, 0, 0);       // K Q^T, V dO^T
      constexpr uint32_t idesc_acc = make_idesc_bf16(128, HD, 0, 1);     // P^T dO, dS^T Q
      constexpr uint32_t idesc_dq = L::DQ_T ? make_idesc_bf16(128, QT, 1, 1)   // K^T dS^T
                                            : make_idesc_bf16(128, HD, 1, 1);  // dS K
      mbar_wait(bar(L::B_KV), 0);
      tc_fence_after();
      auto kmaj = [](uint32_t base, int kk, int slab_bytes) {
        return make_sdesc(base + (kk >> 2) * slab_bytes + (kk & 3) * 32, 16, 1024);
      };
      // S^T or dP^T for sub-tile in stage st: A = K or V (K-major), B = Q or dO (K-major)
      auto issue_s = [&](uint32_t d, uint32_t a_base, uint32_t b_base) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(d, kmaj(a_base, kk, L::KSLAB), kmaj(b_base, kk, L::QSLAB), idesc_s, kk > 0);
      };
      int st = 0, ph = 0;
      mbar_wait(bar(L::B_QFULL + st), ph);
      tc_fence_after();
      issue_s(tmem + L::TM_S, sb + L::OFF_K, sb + L::OFF_Q + st * L::Q_BYTES);
      umma_commit(bar(L::B_SFULL));
      issue_s(tmem + L::TM_DP, sb + L::OFF_V, sb + L::OFF_DO + st * L::Q_BYTES);
      umma_commit(bar(L::B_DPFULL));
      for (int i = 0; i < n_tiles; ++i) {
        const uint32_t sq = sb + L::OFF_Q + st * L::Q_BYTES;
        const uint32_t sdo = sb + L::OFF_DO + st * L::Q_BYTES;
        // dV += P^T dO_i : A = P^T [128 x QT] K-major, B = dO_i [QT x HD] MN-major
        XWAIT(bar(L::B_PREADY), i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)
          umma_bf16(tmem + L::TM_DV, kmaj(sb + L::OFF_P, kk, L::KSLAB),
                    make_sdesc(sdo + kk * 2048, L::QSLAB, 1024), idesc_acc, (i > 0 || kk > 0));
        umma_commit(bar(L::B_PFREE));
        // next S^T as soon as this one has been consumed
        int st1 = st + 1, ph1 = ph;
        if (st1 == L::ST) { st1 = 0; ph1 ^= 1; }
        const bool more = i + 1 < n_tiles;
        if (more) {
          mbar_wait(bar(L::B_QFULL + st1), ph1);
          tc_fence_after();
          issue_s(tmem + L::TM_S, sb + L::OFF_K, sb + L::OFF_Q + st1 * L::Q_BYTES);
          umma_commit(bar(L::B_SFULL));
        }
        // dK += dS^T Q_i : A = dS^T K-major, B = Q_i MN-major
        XWAIT(bar(L::B_DSREADY), i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < QT / 16; ++kk)
          umma_bf16(tmem + L::TM_DK, kmaj(sb + L::OFF_DS, kk, L::KSLAB),
                    make_sdesc(sq + kk * 2048, L::QSLAB, 1024), idesc_acc, (i > 0 || kk > 0));
        umma_commit(bar(L::B_QEMPTY + st));  // last reader of Q_i / dO_i
        // next dP^T (its TMEM was consumed when dS_i was produced)
        if (more) {
          issue_s(tmem + L::TM_DP, sb + L::OFF_V, sb + L::OFF_DO + st1 * L::Q_BYTES);
          umma_commit(bar(L::B_DPFULL));
        }
        // dQ of this sub-tile into TMEM once the drain warps have emptied it
        if (i > 0) {
          XWAIT(bar(L::B_DQFREE), (i - 1) & 1);
          tc_fence_after();
        }
        if constexpr (L::DQ_T) {
          // dQ^T [HD x QT] = K^T dS^T : A = K^T (MN-major view of K), B = dS^T (MN-major)
#pragma unroll
          for (int kk = 0; kk < TILE / 16; ++kk)
            umma_bf16(tmem + L::TM_DQ, make_sdesc(sb + L::OFF_K + kk * 2048, L::KSLAB, 1024),
                      make_sdesc(sb + L::OFF_DS + kk * 2048, L::KSLAB, 1024), idesc_dq, kk > 0);
        } else {
          // dQ [QT x HD] = dS K : A = dS (MN-major view of dS^T), B = K (MN-major)
#pragma unroll
          for (int kk = 0; kk < TILE / 16; ++kk)
            umma_bf16(tmem + L::TM_DQ, make_sdesc(sb + L::OFF_DS + kk * 2048, L::KSLAB, 1024),
                      make_sdesc(sb + L::OFF_K + kk * 2048, L::KSLAB, 1024), idesc_dq, kk > 0);
        }
        umma_commit(bar(L::B_DSFREE));
        umma_commit(bar(L::B_DQFULL));
        st = st1;
        ph = ph1;
      }
      umma_commit(bar(L::B_DONE));
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ softmax / dS WG
    const int quarter = warp & 3;
    const int jj = quarter * 32 + lane;  // key row within the tile
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    const float sl2 = p.scale * kLog2e;
    const bool row_ok = jj < kt.nvalid;
    TileCursor cur;
    cur.start(qr);
    int st = 0, sph = 0;
    for (int i = 0; i < (XLOOP ? n_tiles : 0); ++i, cur.next(qr)) {
      const TileRef qt = tile_ref(p.q_map, p.nq, cur.row0(p.q_map, QT), QT);
      mbar_wait(bar(L::B_QFULL + st), sph);  // orders the producer's lse/delta stores
      int first = 0;  // first visible query column of this key row
      if (causal) {
        if (p.q_map.mode == A2D_IDX_ARRAY) {
          PairMask pm;
          pm.partial = true;
          pm.thr = 0;
          pm.kvalid = kt.nvalid;
          first = col_first(p.q_map, p.k_map, qt, kt, pm, true, jj);
        } else {
          long long thr = ceil_div_s(kt.gmin - qt.gmin, p.q_map.stride);
          thr = max(-(long long)(2 * TILE), min((long long)(2 * TILE), thr));
          first = jj + (int)thr;
        }
      }
      if (!row_ok) first = QT;
      const float* s_lse = stat + st * 2 * QT;
      const float* s_del = s_lse + QT;

      mbar_wait(bar(L::B_SFULL), i & 1);
      tc_fence_after();
      float pr[QT];
#pragma unroll
      for (int c = 0; c < QT / 32; ++c) tmem_ld32(tmem + lane_addr + L::TM_S + c * 32, pr + c * 32);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < QT; ++c) {
#ifndef A2D_X_NO_EXP
        const float e = ex2(fmaf(pr[c], sl2, -s_lse[c]));
#else
        const float e = fmaf(pr[c], sl2, -s_lse[c]);
#endif
        pr[c] = (c >= first) ? e : 0.f;
      }
      uint32_t pk[QT / 2];
#pragma unroll
      for (int c = 0; c < QT; c += 2) pk[c / 2] = pack_bf16(pr[c], pr[c + 1]);
      if (i > 0) mbar_wait(bar(L::B_PFREE), (i - 1) & 1);
      // P^T row jj -> K-major SW128 [128 x QT]
#pragma unroll
      for (int cc = 0; cc < QT / 8; ++cc) {
        const uint32_t addr = sb + L::OFF_P + (cc >> 3) * L::KSLAB + jj * 128 +
                              (((cc & 7) ^ (jj & 7)) << 4);
        st_shared_v4(addr, pk[cc * 4 + 0], pk[cc * 4 + 1], pk[cc * 4 + 2], pk[cc * 4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(bar(L::B_PREADY));

      mbar_wait(bar(L::B_DPFULL), i & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < QT; c0 += 32) {
        float dp[32];
        tmem_ld32(tmem + lane_addr + L::TM_DP + c0, dp);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 32; c += 2)
          pk[(c0 + c) / 2] = pack_bf16(pr[c0 + c] * (dp[c] - s_del[c0 + c]),
                                       pr[c0 + c + 1] * (dp[c + 1] - s_del[c0 + c + 1]));
      }
      if (i > 0) mbar_wait(bar(L::B_DSFREE), (i - 1) & 1);
#pragma unroll
      for (int cc = 0; cc < QT / 8; ++cc) {
        const uint32_t addr = sb + L::OFF_DS + (cc >> 3) * L::KSLAB + jj * 128 +
                              (((cc & 7) ^ (jj & 7)) << 4);
        st_shared_v4(addr, pk[cc * 4 + 0], pk[cc * 4 + 1], pk[cc * 4 + 2], pk[cc * 4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(bar(L::B_DSREADY));
      if (++st == L::ST) { st = 0; sph ^= 1; }
    }
    // ------------------------------------------------------------ dK / dV epilogue
    if (n_tiles > 0) {
      mbar_wait(bar(L::B_DONE), 0);
      tc_fence_after();
    }
    const long long grow = (long long)kt.row0 + jj;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t col0 = which == 0 ? L::TM_DV : L::TM_DK;
      void* base = which == 0 ? p.dv : p.dk;
      const float mul = which == 0 ? 1.f : p.scale;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        float v[32];
        if (n_tiles > 0) {
          tmem_ld32(tmem + lane_addr + col0 + c * 32, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0.f;
        }
        if (!row_ok) continue;
        const long long off = (long long)bh * p.dkv_stride_bh + grow * p.dkv_stride_row + c * 32;
        if (p.dkv_dtype == A2D_F32) {
          float* dst = reinterpret_cast<float*>(base) + off;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + e) =
                make_float4(v[e] * mul, v[e + 1] * mul, v[e + 2] * mul, v[e + 3] * mul);
        } else {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(base) + off;
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 u;
            u.x = pack_bf16(v[e] * mul, v[e + 1] * mul);
            u.y = pack_bf16(v[e + 2] * mul, v[e + 3] * mul);
            u.z = pack_bf16(v[e + 4] * mul, v[e + 5] * mul);
            u.w = pack_bf16(v[e + 6] * mul, v[e + 7] * mul);
            *reinterpret_cast<uint4*>(dst + e) = u;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ dQ drain WG
    const int quarter = warp & 3;
    const int t = quarter * 32 + lane;  // TMEM lane: head dim (dQ^T) or query row (dQ)
    const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
    TileCursor cur;
    cur.start(qr);
    for (int i = 0; i < (XLOOP ? n_tiles : 0); ++i, cur.next(qr)) {
      const int qrow = cur.row0(p.q_map, QT);
      mbar_wait(bar(L::B_DQFULL), i & 1);
      tc_fence_after();
      constexpr int NC = L::DQ_T ? QT : HD;  // TMEM columns of this lane
      float v[NC];
#pragma unroll
      for (int c = 0; c < NC / 32; ++c) tmem_ld32(tmem + lane_addr + L::TM_DQ + c * 32, v + c * 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(L::B_DQFREE));
      // previous reduce must have finished reading the staging tile
      if (t == 0) bulk_wait_read0();
      named_bar_sync(1, 128);
      if constexpr (L::DQ_T) {
        // lane t = head dim h; v[q] = dQ[q][h].  Tile [QT][HD] fp32 in HD/32
        // slabs of [QT][32] with 128B swizzle.
        const int h = t;
        const uint32_t slab = sb + L::OFF_DQ + (h >> 5) * L::DQ_SLAB;
        const int hc = (h & 31) >> 2, he = (h & 3) * 4;
#pragma unroll
        for (int q = 0; q < QT; ++q) {
          const uint32_t addr = slab + q * 128 + ((hc ^ (q & 7)) << 4) + he;
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v[q]) : "memory");
        }
      } else {
        // lane t = query row; v[h] = dQ[t][h]
        const int q = t;
#pragma unroll
        for (int c = 0; c < HD / 4; ++c) {
          const uint32_t addr = sb + L::OFF_DQ + (c >> 3) * L::DQ_SLAB + q * 128 +
                                (((c & 7) ^ (q & 7)) << 4);
          st_shared_v4(addr, __float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]),
                       __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3]));
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
#ifndef A2D_X_NO_DQ_REDUCE
      if (t == 0) {
#else
      if (false) {
#endif
#pragma unroll
        for (int s = 0; s < HD / 32; ++s)
          tma_reduce_add_3d(&tm_dq, sb + L::OFF_DQ + s * L::DQ_SLAB, s * 32, qrow, bh);
        bulk_commit();
      }
    }
    if (t == 0) bulk_wait0();
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
int launch_bwd_hd(const a2d_tile_bwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                  const CUtensorMap& tv, const CUtensorMap& tdo, cudaStream_t stream) {
  using L = BwdLayout<HD>;
  static bool configured[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(bwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         L::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(bwd)");
    configured[dev & 63] = true;
  }
  CUtensorMap tdq;
  int rc = make_map_f32_dq(&tdq, a.dq_acc, HD, a.nq, a.bh, a.dq_stride_row, a.dq_stride_bh, L::QT);
  if (rc) return rc;
  const int k_tiles = (a.k_map.mode == A2D_IDX_AFFINE && a.k_map.nblocks > 1)
                          ? a.k_map.nblocks * (a.k_map.rows_per_block / TILE)
                          : (a.nk + TILE - 1) / TILE;
  dim3 grid(k_tiles, a.bh);
  bwd_kernel<HD><<<grid, BWD_THREADS, L::SMEM, stream>>>(tq, tk, tv, tdo, tdq, a);
  return check_launch("bwd_kernel");
}

// H = 128 runs the N=128-shaped kernel (tile_bwd128.cu); A2D_BWD_V1=1 selects
// this file's 64-query design instead (kept for A/B measurement).
static bool use_v1_for_128() {
  static const bool v1 = [] {
    const char* e = getenv("A2D_BWD_V1");
    return e != nullptr && e[0] == '1';
  }();
  return v1;
}

// Every head dim runs the N=128-shaped kernel (tile_bwd128.cu): columns past
// h are TMA zero fill, which for h = 64 still beats this file's 64-column
// kernel by ~2x.  A2D_BWD_V1=1 selects the 64-query design for h in {64, 128}.
int launch_tile_bwd(const a2d_tile_bwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, const CUtensorMap& tdo, cudaStream_t stream) {
  if (use_v1_for_128() && a.h == 128) return launch_bwd_hd<128>(a, tq, tk, tv, tdo, stream);
  if (use_v1_for_128() && a.h == 64) return launch_bwd_hd<64>(a, tq, tk, tv, tdo, stream);
  return launch_bwd128(a, tq, tk, tv, tdo, stream);
}

int bwd_q_tile_rows(int h) {
  if (use_v1_for_128() && h == 128) return BwdLayout<128>::QT;
  if (use_v1_for_128() && h == 64) return BwdLayout<64>::QT;
  return TILE;
}

}  // namespace a2d
