/*
 * attn2d_b200 — C ABI of the B200-native Attention2D hot path.
 *
 * Drop-in boundary for the reference's kernel layer
 * (reference pkg/src/attn2d/kernels/__init__.py:60-92):
 *
 *   reference                                   this ABI
 *   -----------------------------------------   ---------------------------------
 *   kernels.flash_forward   (__init__.py:70-78) a2d_tile_fwd      (partial O + LSE)
 *   kernels.flash_backward  (__init__.py:81-92) a2d_bwd_preprocess + a2d_tile_bwd
 *                                               + a2d_bwd_finalize
 *   attention.attn_fix      (attention.py:194)  a2d_lse_merge     (k-way, fused finalize)
 *   attention.finalize      (attention.py:217)  fused into a2d_tile_fwd / a2d_lse_merge
 *
 * Conventions (all calls):
 *   - every pointer is a DEVICE pointer owned by the caller; the caller
 *     allocates every output (same ownership rule as the reference kernels);
 *   - calls are stream-ordered and asynchronous on `stream`;
 *   - no C++ exceptions cross the boundary; return codes:
 *       A2D_OK = 0, A2D_EINVAL = 1 (bad argument / shape),
 *       A2D_EUNSUPPORTED = 2 (valid but unsupported: head dim not a multiple
 *       of 8 in [8, 128], index map),
 *       A2D_ECUDA = 3 (CUDA launch / runtime error).
 *     a2d_last_error() returns a thread-local message for the last failure.
 *   - tensors are [bh, rows, h] with unit stride along h; strides in elements.
 *   - a call with no work (zero heads, or zero rows on the side that owns the
 *     outputs' rows) returns A2D_OK before any pointer is checked or
 *     dereferenced: empty framework tensors may carry null data pointers.
 *   - the partial state of one query row is (O, LSE): O normalised by its own
 *     denominator and LSE = m + log(d) (natural log, -inf for a row that has
 *     attended nothing).  This is the reference's (m, n, d) triple
 *     (attention.py:75-110) in its unique form: n = O * d, m + log d = LSE.
 */
#ifndef ATTN2D_B200_H
#define ATTN2D_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define A2D_ABI_VERSION 4
#define A2D_MAX_BLOCKS 16

enum { A2D_OK = 0, A2D_EINVAL = 1, A2D_EUNSUPPORTED = 2, A2D_ECUDA = 3 };
enum { A2D_IDX_AFFINE = 0, A2D_IDX_ARRAY = 1 };
enum { A2D_F32 = 0, A2D_BF16 = 1, A2D_F16 = 2 };

/* Global token index of every local row — the reference's TokenShard.indices
 * (attention.py:50-72) in a form the kernel can evaluate without memory
 * traffic.
 *   A2D_IDX_AFFINE: rows are split into `nblocks` blocks of `rows_per_block`
 *     rows; row i of block b has global index base[b] + stride * i.
 *     nblocks > 1 requires rows_per_block % 128 == 0.  This covers every
 *     layout the strategies produce: a contiguous shard (1 block, stride 1),
 *     the cyclic 2D gathers (Pc or Pr blocks, stride P; layouts.py:53-65) and
 *     the ring's mirrored halves (2 blocks, stride 1; ring.py:27-38).
 *   A2D_IDX_ARRAY: `idx` points to one int64 global index per row, strictly
 *     increasing (the TokenShard contract); slow path for arbitrary subsets.
 * Query and key maps of one call must use the same mode; affine maps must
 * share the same stride. */
typedef struct {
  int32_t mode;
  int32_t nblocks;
  int32_t rows_per_block;
  int32_t reserved;
  int64_t stride;
  int64_t base[A2D_MAX_BLOCKS];
  const int64_t* idx;
} a2d_index_map;

/* Tile forward: kernels.flash_forward (reference kernels/__init__.py:70-78,
 * numpy_backend.py:24-43) for bh independent heads.
 *   q [bh, nq, h], k/v [bh, nk, h]: in_dtype A2D_BF16 (0 reads as bf16) or
 *   A2D_F16, all three alike.
 *   o [bh, nq, h] (o_dtype A2D_F32: normalised partial O; A2D_BF16 or
 *   A2D_F16: final O),
 *   lse [bh, nq] fp32 natural-log LSE (-inf: row attended nothing here).
 *   accumulate = 1 continues from the (o, lse) state already in the buffers
 *   (requires A2D_F32): the streaming continuation of the reference kernel
 *   (kernels/__init__.py:73-77, test_kernels.py:124-137).
 *   kv_group (GQA / MQA): query head b reads k/v head
 *   b / kv_group; k/v hold bh / kv_group heads.  0 or 1 = one k/v head per
 *   query head. */
typedef struct {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  float* lse;
  int64_t q_stride_bh, q_stride_row;
  int64_t k_stride_bh, k_stride_row;
  int64_t v_stride_bh, v_stride_row;
  int64_t o_stride_bh, o_stride_row;
  int32_t bh, nq, nk, h;
  int32_t causal;
  float scale;
  int32_t o_dtype;
  int32_t accumulate;
  a2d_index_map q_map;
  a2d_index_map k_map;
  int32_t kv_group;
  int32_t in_dtype;
} a2d_tile_fwd_args;

int a2d_tile_fwd(const a2d_tile_fwd_args* args, void* stream);

/* delta[bh, n] = rowsum(dO * O) in fp32 — the first line of the reference's
 * backward recurrence (numpy_backend.py:49, numba_backend.py:84-86).
 * o, dout are [bh, n, h] of in_dtype (A2D_BF16 or A2D_F16) with the given
 * strides. */
int a2d_bwd_preprocess(const void* o, const void* dout, float* delta,
                       int64_t o_stride_bh, int64_t o_stride_row,
                       int64_t do_stride_bh, int64_t do_stride_row,
                       int32_t bh, int32_t n, int32_t h, int32_t in_dtype, void* stream);

/* Tile backward: kernels.flash_backward (kernels/__init__.py:81-92,
 * numpy_backend.py:46-62).  lse / delta are the GLOBAL row statistics of q's
 * rows (after every merge), so the gradients are exact partial sums over
 * this key subset (attention.py:225-257).
 *   dq_acc [bh, nq, h] fp32 (strides dq_stride_*, multiples of 4 elements):
 *   dS K (unscaled) is ADDED to it with TMA reduce-add (caller zeroes);
 *   q, k, v, dout: in_dtype (A2D_BF16, 0 reads as bf16, or A2D_F16).
 *   dk, dv [bh, nk, h]: written (dkv_dtype A2D_F32, A2D_BF16 or A2D_F16); dk is
 *   already multiplied by scale.  accumulate_dkv = 1 ADDS the contributions
 *   to the fp32 dk / dv already in the buffers instead (the ring's and the
 *   overlapped schedule's per-hop accumulation, reference ring.py:118-143).
 *   nq == 0 writes zero dk / dv (nothing attends these keys).
 *   kv_group: as for a2d_tile_fwd (k/v hold bh / kv_group heads); dk / dv
 *   stay per QUERY head, the caller sums each group. */
typedef struct {
  const void* q;
  const void* k;
  const void* v;
  const void* dout;
  const float* lse;
  const float* delta;
  float* dq_acc;
  void* dk;
  void* dv;
  int64_t q_stride_bh, q_stride_row;
  int64_t k_stride_bh, k_stride_row;
  int64_t v_stride_bh, v_stride_row;
  int64_t do_stride_bh, do_stride_row;
  int64_t dq_stride_bh, dq_stride_row;
  int64_t dkv_stride_bh, dkv_stride_row;
  int32_t bh, nq, nk, h;
  int32_t causal;
  float scale;
  int32_t dkv_dtype;
  int32_t accumulate_dkv;
  a2d_index_map q_map;
  a2d_index_map k_map;
  int32_t kv_group;
  int32_t in_dtype;
} a2d_tile_bwd_args;

int a2d_tile_bwd(const a2d_tile_bwd_args* args, void* stream);

/* dq = scale * dq_acc, converted to out_dtype (A2D_F32, A2D_BF16 or
 * A2D_F16); both [bh, n, h] with the given strides (unit stride along h). */
int a2d_bwd_finalize(const float* dq_acc, int64_t acc_stride_bh, int64_t acc_stride_row,
                     void* dq, int32_t out_dtype, int64_t dq_stride_bh, int64_t dq_stride_row,
                     int32_t bh, int32_t n, int32_t h, float scale, void* stream);

/* k-way log-sum-exp merge of partial (O, LSE) over disjoint key sets —
 * attn_fix folded over k parts (attention.py:194-214) fused with finalize
 * (attention.py:217-222).  Part i lives at o_parts + i*part_stride_o
 * (fp32 [rows, h] rows of `row_stride` elements) and
 * lse_parts + i*part_stride_lse.  Writes o_out (out_dtype A2D_F32, A2D_BF16
 * or A2D_F16, [rows, h] with
 * out_row_stride) and lse_out (fp32 [rows]); rows whose every part is empty
 * get O = 0 and LSE = -inf (the caller raises FullyMaskedRowError). */
int a2d_lse_merge(const float* o_parts, const float* lse_parts, int32_t k_parts,
                  int64_t part_stride_o, int64_t part_stride_lse,
                  int64_t rows, int32_t h, int64_t row_stride,
                  void* o_out, int32_t out_dtype, int64_t out_row_stride,
                  float* lse_out, void* stream);

/* Diagnostic: tcgen05 descriptor self-test.  d[128 x n] fp32 = A B with
 * A [128 x 128] bf16 row-major (K-major) and B given as [128(k) x n] bf16
 * row-major (MN-major, b_mn_major=1) or [n x 128(k)] (K-major, 0).
 * n in {64, 128}. */
int a2d_selftest_umma(const void* a, const void* b, float* d, int32_t n,
                      int32_t b_mn_major, void* stream);

/* Diagnostic: tcgen05 issue-rate probe; cycles_out[ctas] receives the cycles
 * one CTA spent issuing `iters` K=128 units of MMA shape `variant`. */
int a2d_bench_umma(int32_t variant, int32_t iters, int64_t* cycles_out, int32_t ctas,
                   void* stream);

/* Diagnostic: fill shared memory (mode bit 0) and TMEM (bit 1) of every SM
 * with NaN patterns, to prove the kernels never consume on-chip memory they
 * did not write. */
int a2d_debug_poison(int32_t mode, void* stream);

int a2d_abi_version(void);
const char* a2d_last_error(void);
int a2d_num_sms(void);

#ifdef __cplusplus
}
#endif
#endif /* ATTN2D_B200_H */
