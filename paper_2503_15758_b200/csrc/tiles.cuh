// tiles.cuh — global-index bookkeeping shared by the tile kernels.
//
// The reference masks by GLOBAL token index (q_idx >= k_idx,
// numpy_backend.py:31, numba_backend.py:51), with indices carried by each
// TokenShard (attention.py:50-72).  Here a shard's indices are an
// a2d_index_map; every kernel role evaluates tile classes arithmetically so
// that producer, MMA issuer and softmax warps enumerate the same tile list
// without exchanging it.
#pragma once
#include <stdint.h>
#include "../../include/attn2d_b200.h"

namespace a2d {

constexpr int TILE = 128;

__host__ __device__ __forceinline__ long long ceil_div_s(long long a, long long s) {
  return a >= 0 ? (a + s - 1) / s : -((-a) / s);
}

// Rows in block b of a map over n rows.
__device__ __forceinline__ int blk_rows(const a2d_index_map& m, int n, int b) {
  return m.nblocks == 1 ? n : m.rows_per_block;
}

// Global index of local row `row` (row < n).
__device__ __forceinline__ long long gidx(const a2d_index_map& m, int row) {
  if (m.mode == A2D_IDX_ARRAY) return m.idx[row];
  if (m.nblocks == 1) return m.base[0] + m.stride * row;
  const int b = row / m.rows_per_block;
  return m.base[b] + m.stride * (row - b * m.rows_per_block);
}

// Number of elements among sorted a[0..n) that are <= x.
__device__ __forceinline__ int upper_bound_i64(const int64_t* a, int n, long long x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// A 128-row tile of one side (query or key) of a call.
struct TileRef {
  int row0;        // first local row
  int nvalid;      // valid rows in the tile (<= 128)
  long long gmin;  // global index of the first row
  long long gmax;  // global index of the last valid row
};

__device__ __forceinline__ TileRef tile_ref(const a2d_index_map& m, int n, int t_flat_row0,
                                           int T = TILE) {
  TileRef r;
  r.row0 = t_flat_row0;
  int end;
  if (m.mode == A2D_IDX_ARRAY || m.nblocks == 1) {
    end = n;
  } else {
    const int b = t_flat_row0 / m.rows_per_block;
    end = (b + 1) * m.rows_per_block;
  }
  r.nvalid = min(T, end - t_flat_row0);
  r.gmin = gidx(m, t_flat_row0);
  r.gmax = gidx(m, t_flat_row0 + r.nvalid - 1);
  return r;
}

// Enumerates, for one query tile, the key tiles it attends (forward), or
// for one key tile, the query tiles that attend it (backward).  Within each
// block of the enumerated side, global indices increase with the local row,
// so under causal masking the attended tiles form a prefix (keys) or a
// suffix (queries) of every block.
struct TileRange {
  int nblk;
  int first[A2D_MAX_BLOCKS];  // first tile (within block) to visit
  int last[A2D_MAX_BLOCKS];   // one past the last tile (within block)
  int total;
};

// Key tiles attended by a query tile whose global indices span [qmin, qmax].
__device__ __forceinline__ void key_range(const a2d_index_map& km, int nk, bool causal,
                                          long long qmax, TileRange& r) {
  r.total = 0;
  r.nblk = (km.mode == A2D_IDX_ARRAY) ? 1 : km.nblocks;
  for (int b = 0; b < r.nblk; ++b) {
    const int rows = (km.mode == A2D_IDX_ARRAY) ? nk : blk_rows(km, nk, b);
    const int ntiles = (rows + TILE - 1) / TILE;
    int cnt = ntiles;
    if (causal) {
      if (km.mode == A2D_IDX_ARRAY) {
        // count tiles whose first key index is <= qmax (sorted keys)
        int lo = 0, hi = ntiles;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (km.idx[mid * TILE] <= qmax) lo = mid + 1; else hi = mid;
        }
        cnt = lo;
      } else {
        const long long base = km.base[b];
        if (qmax < base) cnt = 0;
        else cnt = (int)min((long long)ntiles, (qmax - base) / (km.stride * TILE) + 1);
      }
    }
    r.first[b] = 0;
    r.last[b] = cnt;
    r.total += cnt;
  }
}

// Query tiles that attend a key tile whose first global index is kmin.
__device__ __forceinline__ void query_range(const a2d_index_map& qm, int nq, bool causal,
                                            long long kmin, TileRange& r, int T = TILE) {
  r.total = 0;
  r.nblk = (qm.mode == A2D_IDX_ARRAY) ? 1 : qm.nblocks;
  for (int b = 0; b < r.nblk; ++b) {
    const int rows = (qm.mode == A2D_IDX_ARRAY) ? nq : blk_rows(qm, nq, b);
    const int ntiles = (rows + T - 1) / T;
    int first = 0;
    if (causal) {
      if (qm.mode == A2D_IDX_ARRAY) {
        // first tile whose last query index is >= kmin
        int lo = 0, hi = ntiles;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const int lastrow = min(rows, (mid + 1) * T) - 1;
          if (qm.idx[lastrow] < kmin) lo = mid + 1; else hi = mid;
        }
        first = lo;
      } else {
        const long long base = qm.base[b];
        const long long s = qm.stride;
        // tile t covers base + s*(T t .. T t + T-1); need its max >= kmin
        const long long need = kmin - base - s * (T - 1);
        first = need <= 0 ? 0 : (int)min((long long)ntiles, ceil_div_s(need, s * T));
        // a short tail tile has a smaller maximum than the formula assumes
        if (first < ntiles) {
          const int lastrow = min(rows, (first + 1) * T) - 1;
          if (base + s * lastrow < kmin) first += 1;
        }
      }
    }
    r.first[b] = first;
    r.last[b] = ntiles;
    r.total += ntiles - first;
  }
}

// Cursor over a TileRange; yields the local row0 of each tile, cyclically
// starting at flat position `rot` (callers iterate exactly `total` tiles).
// Rotating the start per CTA keeps co-resident CTAs of one head on
// different tiles, so their loads and dQ reduce-adds do not pile onto the
// same L2 lines at the same time.
struct TileCursor {
  int b, t;
  __device__ __forceinline__ void start(const TileRange& r, int rot = 0) {
    b = 0;
    t = r.first[0];
    skip(r);
    if (r.total > 0 && rot > 0) {
      rot %= r.total;
      while (rot > 0) {  // jump whole blocks, then within the block
        const int left = r.last[b] - t;
        if (rot < left) {
          t += rot;
          rot = 0;
        } else {
          rot -= left;
          t = r.last[b];
          skip(r);
        }
      }
    }
  }
  __device__ __forceinline__ void skip(const TileRange& r) {
    while (t >= r.last[b]) {
      ++b;
      if (b >= r.nblk) b = 0;
      t = r.first[b];
      if (r.total == 0) return;
    }
  }
  __device__ __forceinline__ void next(const TileRange& r) {
    ++t;
    skip(r);
  }
  __device__ __forceinline__ int row0(const a2d_index_map& m, int T = TILE) const {
    const int rpb = (m.mode == A2D_IDX_ARRAY || m.nblocks == 1) ? 0 : m.rows_per_block;
    return b * rpb + t * T;
  }
};

// Block and tile (within the block) at flat position f (0 <= f < r.total).
__device__ __forceinline__ void range_pos(const TileRange& r, int f, int& b, int& t) {
  b = 0;
  for (; b < r.nblk - 1; ++b) {
    const int cnt = r.last[b] - r.first[b];
    if (f < cnt) break;
    f -= cnt;
  }
  t = r.first[b] + f;
}

// Local row0 of the tile at flat position f (0 <= f < r.total) of a
// TileRange in block-major order (random access twin of TileCursor).
__device__ __forceinline__ int range_row0(const TileRange& r, const a2d_index_map& m, int f,
                                          int T = TILE) {
  int b = 0;
  for (; b < r.nblk - 1; ++b) {
    const int cnt = r.last[b] - r.first[b];
    if (f < cnt) break;
    f -= cnt;
  }
  const int rpb = (m.mode == A2D_IDX_ARRAY || m.nblocks == 1) ? 0 : m.rows_per_block;
  return b * rpb + (r.first[b] + f) * T;
}

// Causal visibility inside a (query tile, key tile) pair: query row ii
// (0..127) sees key columns 0..lim(ii).  Returns whether any masking is
// needed.  Affine maps share one stride s, so q_g >= k_g  <=>
// ii - jj >= thr with thr = ceil((kmin - qmin) / s).
struct PairMask {
  bool partial;
  int thr;       // affine causal threshold (clamped)
  int kvalid;    // valid key columns
};

__device__ __forceinline__ PairMask pair_mask(const a2d_index_map& qm, const TileRef& qt,
                                              const TileRef& kt, bool causal) {
  PairMask pm;
  pm.kvalid = kt.nvalid;
  pm.thr = -TILE;
  if (!causal) {
    pm.partial = kt.nvalid < TILE;
    return pm;
  }
  if (qm.mode == A2D_IDX_ARRAY) {
    pm.partial = true;  // per-row binary search
    return pm;
  }
  long long thr = qm.stride == 1 ? kt.gmin - qt.gmin : ceil_div_s(kt.gmin - qt.gmin, qm.stride);
  thr = max(-(long long)TILE, min((long long)(2 * TILE), thr));
  pm.thr = (int)thr;
  pm.partial = (kt.nvalid < TILE) || (pm.thr > -(TILE - 1));
  return pm;
}

// Last visible key column of query row ii (may be < 0: row sees nothing).
__device__ __forceinline__ int row_limit(const a2d_index_map& qm, const a2d_index_map& km,
                                         const TileRef& qt, const TileRef& kt,
                                         const PairMask& pm, bool causal, int ii) {
  if (!causal) return pm.kvalid - 1;
  if (qm.mode == A2D_IDX_ARRAY) {
    if (ii >= qt.nvalid) return -1;
    const long long g = qm.idx[qt.row0 + ii];
    return upper_bound_i64(km.idx + kt.row0, kt.nvalid, g) - 1;
  }
  return min(ii - pm.thr, pm.kvalid - 1);
}

// For the backward (key rows in TMEM lanes): key row jj sees query columns
// ii >= first(jj).  Returns the first visible query column (may be > 127).
__device__ __forceinline__ int col_first(const a2d_index_map& qm, const a2d_index_map& km,
                                         const TileRef& qt, const TileRef& kt,
                                         const PairMask& pm, bool causal, int jj) {
  if (!causal) return 0;
  if (qm.mode == A2D_IDX_ARRAY) {
    if (jj >= kt.nvalid) return TILE;
    const long long g = km.idx[kt.row0 + jj];
    // first query with index >= g: count of queries < g
    int lo = 0, hi = qt.nvalid;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (qm.idx[qt.row0 + mid] < g) lo = mid + 1; else hi = mid;
    }
    return lo;
  }
  return jj + pm.thr;
}

}  // namespace a2d
