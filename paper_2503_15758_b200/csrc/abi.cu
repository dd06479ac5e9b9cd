// abi.cu — the extern "C" boundary (include/attn2d_b200.h): argument
// validation with the reference's error taxonomy (errors.py:4-21 — shape
// errors -> A2D_EINVAL, unsupported-but-valid -> A2D_EUNSUPPORTED), TMA
// descriptor construction, and dispatch to the sm_100a kernels.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <mutex>
#include "kernels.h"

namespace a2d {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(cudaError_t e, const char* what) {
  return set_error(A2D_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  return A2D_OK;
}

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3-D map over a bf16 [bh, rows, h] tensor (unit stride along h), box 64 x 128 x 1,
// 128-byte swizzle: one box is one K-major SW128 slab of a 128-row tile.
int make_map(CUtensorMap* m, const void* ptr, int h, int rows, int bh, long long s_row,
             long long s_bh, const char* name, int box_rows = 128, bool f16 = false) {
  if (ptr == nullptr) return set_error(A2D_EINVAL, "%s is null", name);
  if (reinterpret_cast<uintptr_t>(ptr) % 16)
    return set_error(A2D_EINVAL, "%s must be 16-byte aligned", name);
  if ((s_row * 2) % 16 || (s_bh * 2) % 16)
    return set_error(A2D_EINVAL, "%s strides must be multiples of 8 elements", name);
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(A2D_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)h, (cuuint64_t)rows, (cuuint64_t)bh};
  cuuint64_t strides[2] = {(cuuint64_t)(s_row * 2), (cuuint64_t)(s_bh * 2)};
  if (bh == 1) strides[1] = (cuuint64_t)((long long)rows * s_row * 2);
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(A2D_ECUDA, "cuTensorMapEncodeTiled(%s) failed: %d", name, (int)r);
  return A2D_OK;
}

}  // namespace

int make_map_bf16(CUtensorMap* m, const void* ptr, int h, int rows, int bh, long long s_row,
                  long long s_bh, const char* name, int box_rows) {
  return make_map(m, ptr, h, rows, bh, s_row, s_bh, name, box_rows);
}

// 16-bit operand type of a tile call: 0 (the v3 reserved field) reads as bf16
static int in_type(int32_t in_dtype, bool* f16) {
  if (in_dtype != 0 && in_dtype != A2D_BF16 && in_dtype != A2D_F16)
    return set_error(A2D_EUNSUPPORTED, "in_dtype %d: inputs must be bf16 or fp16", in_dtype);
  *f16 = in_dtype == A2D_F16;
  return A2D_OK;
}

static bool out16_ok(int32_t dt) { return dt == A2D_F32 || dt == A2D_BF16 || dt == A2D_F16; }

// fp32 [bh, rows, h] contiguous accumulator, box 32 x box_rows x 1, 128B swizzle
// (the backward's dQ reduce-add target).
int make_map_f32_dq(CUtensorMap* m, const float* ptr, int h, int rows, int bh, long long s_row,
                    long long s_bh, int box_rows) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return set_error(A2D_EINVAL, "dq_acc must be 16-byte aligned");
  if ((s_row * 4) % 16 || (s_bh * 4) % 16)
    return set_error(A2D_EINVAL, "dq_acc strides must be multiples of 4 elements");
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(A2D_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)h, (cuuint64_t)rows, (cuuint64_t)bh};
  cuuint64_t strides[2] = {(cuuint64_t)(s_row * 4), (cuuint64_t)(s_bh * 4)};
  if (bh == 1) strides[1] = (cuuint64_t)((long long)rows * s_row * 4);
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(A2D_ECUDA, "cuTensorMapEncodeTiled(dq_acc) failed: %d", (int)r);
  return A2D_OK;
}

// Same accumulator, box h x box_rows x 1 without swizzle (row-major staging).
int make_map_f32_dq_flat(CUtensorMap* m, const float* ptr, int h, int rows, int bh,
                         long long s_row, long long s_bh, int box_rows, int box_cols) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16) return set_error(A2D_EINVAL, "dq_acc must be 16-byte aligned");
  if ((s_row * 4) % 16 || (s_bh * 4) % 16)
    return set_error(A2D_EINVAL, "dq_acc strides must be multiples of 4 elements");
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(A2D_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)h, (cuuint64_t)rows, (cuuint64_t)bh};
  cuuint64_t strides[2] = {(cuuint64_t)(s_row * 4), (cuuint64_t)(s_bh * 4)};
  if (bh == 1) strides[1] = (cuuint64_t)((long long)rows * s_row * 4);
  // box_cols may exceed h: the reduce clips the columns past the tensor
  cuuint32_t box[3] = {(cuuint32_t)(box_cols > 0 ? box_cols : h), (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(A2D_ECUDA, "cuTensorMapEncodeTiled(dq_acc flat) failed: %d", (int)r);
  return A2D_OK;
}

namespace {

int check_map(const a2d_index_map& m, int n, const char* name) {
  if (m.mode == A2D_IDX_ARRAY) {
    if (m.idx == nullptr && n > 0) return set_error(A2D_EINVAL, "%s.idx is null", name);
    return A2D_OK;
  }
  if (m.mode != A2D_IDX_AFFINE) return set_error(A2D_EINVAL, "%s.mode invalid", name);
  if (m.nblocks < 1 || m.nblocks > A2D_MAX_BLOCKS)
    return set_error(A2D_EINVAL, "%s.nblocks must be in [1, %d]", name, A2D_MAX_BLOCKS);
  if (m.stride < 1) return set_error(A2D_EUNSUPPORTED, "%s.stride must be >= 1", name);
  if (m.nblocks > 1) {
    if (m.rows_per_block <= 0 || m.rows_per_block % 128)
      return set_error(A2D_EUNSUPPORTED, "%s: multi-block maps need rows_per_block %% 128 == 0",
                       name);
    if ((long long)m.nblocks * m.rows_per_block != n)
      return set_error(A2D_EINVAL, "%s: nblocks * rows_per_block != rows", name);
  }
  return A2D_OK;
}

int check_common(int bh, int nq, int nk, int h, int causal, float scale,
                 const a2d_index_map& qm, const a2d_index_map& km) {
  if (bh < 0 || nq < 0 || nk < 0) return set_error(A2D_EINVAL, "negative sizes");
  // any head dim up to 128 in steps of 8 (16-byte rows): the tiles are 64 or
  // 128 columns wide and the TMA zero-fills the columns past h, so the extra
  // MMA columns add nothing and the epilogues write only h columns
  if (h < 8 || h > 128 || h % 8)
    return set_error(A2D_EUNSUPPORTED, "head dim %d not a multiple of 8 in [8, 128]", h);
  if (!(scale > 0.f)) return set_error(A2D_EUNSUPPORTED, "scale must be positive");
  int rc;
  if ((rc = check_map(qm, nq, "q_map"))) return rc;
  if ((rc = check_map(km, nk, "k_map"))) return rc;
  if (qm.mode != km.mode) return set_error(A2D_EUNSUPPORTED, "q_map and k_map modes differ");
  if (causal && qm.mode == A2D_IDX_AFFINE && qm.stride != km.stride)
    return set_error(A2D_EUNSUPPORTED, "affine q/k maps must share one stride");
  return A2D_OK;
}

}  // namespace
}  // namespace a2d

using namespace a2d;

extern "C" {

int a2d_abi_version(void) { return A2D_ABI_VERSION; }

const char* a2d_last_error(void) { return g_err; }

int a2d_num_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int a2d_tile_fwd(const a2d_tile_fwd_args* a, void* stream) {
  if (!a) return set_error(A2D_EINVAL, "args is null");
  int rc = check_common(a->bh, a->nq, a->nk, a->h, a->causal, a->scale, a->q_map, a->k_map);
  if (rc) return rc;
  const int g = a->kv_group > 1 ? a->kv_group : 1;
  if (a->kv_group < 0 || a->bh % g) return set_error(A2D_EINVAL, "kv_group %d must divide bh %d", a->kv_group, a->bh);
  if (!out16_ok(a->o_dtype)) return set_error(A2D_EINVAL, "o_dtype invalid");
  bool f16 = false;
  if ((rc = in_type(a->in_dtype, &f16))) return rc;
  if (a->accumulate && a->o_dtype != A2D_F32)
    return set_error(A2D_EINVAL, "accumulate requires an fp32 partial O");
  if (a->bh == 0 || a->nq == 0) return A2D_OK;  // empty outputs may have null pointers
  if (!a->o || !a->lse) return set_error(A2D_EINVAL, "o / lse are null");
  if (a->nk == 0) {  // nothing to attend: the empty partial (attention.py:91-97)
    if (a->accumulate) return A2D_OK;
    return set_error(A2D_EINVAL, "nk == 0 without accumulate");
  }
  if (a->o_stride_row % 4 || a->o_stride_bh % 4)
    return set_error(A2D_EINVAL, "o strides must be multiples of 4 elements");
  CUtensorMap tq, tk, tv;
  if ((rc = make_map(&tq, a->q, a->h, a->nq, a->bh, a->q_stride_row, a->q_stride_bh, "q", 128, f16)))
    return rc;
  if ((rc = make_map(&tk, a->k, a->h, a->nk, a->bh / g, a->k_stride_row, a->k_stride_bh, "k", 128,
                     f16)))
    return rc;
  if ((rc = make_map(&tv, a->v, a->h, a->nk, a->bh / g, a->v_stride_row, a->v_stride_bh, "v", 128,
                     f16)))
    return rc;
  return launch_tile_fwd(*a, tq, tk, tv, static_cast<cudaStream_t>(stream));
}

int a2d_bwd_preprocess(const void* o, const void* dout, float* delta, int64_t o_stride_bh,
                       int64_t o_stride_row, int64_t do_stride_bh, int64_t do_stride_row,
                       int32_t bh, int32_t n, int32_t h, int32_t in_dtype, void* stream) {
  bool f16 = false;
  int rc = in_type(in_dtype, &f16);
  if (rc) return rc;
  if (h < 8 || h > 128 || h % 8)
    return set_error(A2D_EUNSUPPORTED, "head dim %d not a multiple of 8 in [8, 128]", h);
  if (bh < 0 || n < 0) return set_error(A2D_EINVAL, "negative sizes");
  if (bh == 0 || n == 0) return A2D_OK;
  if (!o || !dout || !delta) return set_error(A2D_EINVAL, "null pointer");
  return launch_bwd_preprocess(o, dout, delta, o_stride_bh, o_stride_row, do_stride_bh,
                               do_stride_row, bh, n, h, f16, static_cast<cudaStream_t>(stream));
}

int a2d_tile_bwd(const a2d_tile_bwd_args* a, void* stream) {
  if (!a) return set_error(A2D_EINVAL, "args is null");
  int rc = check_common(a->bh, a->nq, a->nk, a->h, a->causal, a->scale, a->q_map, a->k_map);
  if (rc) return rc;
  const int g = a->kv_group > 1 ? a->kv_group : 1;
  if (a->kv_group < 0 || a->bh % g) return set_error(A2D_EINVAL, "kv_group %d must divide bh %d", a->kv_group, a->bh);
  if (!out16_ok(a->dkv_dtype)) return set_error(A2D_EINVAL, "dkv_dtype invalid");
  bool f16 = false;
  if ((rc = in_type(a->in_dtype, &f16))) return rc;
  if (a->accumulate_dkv && a->dkv_dtype != A2D_F32)
    return set_error(A2D_EINVAL, "accumulate_dkv requires fp32 dk / dv");
  if (a->bh == 0 || a->nk == 0) return A2D_OK;  // empty outputs may have null pointers
  if (!a->dk || !a->dv) return set_error(A2D_EINVAL, "null dk / dv pointer");
  if (a->nq > 0 && (!a->lse || !a->delta || !a->dq_acc))
    return set_error(A2D_EINVAL, "null dq_acc / statistics pointer");
  if (a->nq == 0) {  // no query rows: zero gradients (reference attention.py:250-252)
    if (a->accumulate_dkv) return A2D_OK;
    if ((a->dkv_stride_bh | a->dkv_stride_row) % 4)
      return set_error(A2D_EINVAL, "dk / dv strides must be multiples of 4 elements");
    int r = launch_bwd_finalize(nullptr, 0, 0, a->dk, a->dkv_dtype, a->dkv_stride_bh,
                                a->dkv_stride_row, a->bh, a->nk, a->h, 0.f,
                                static_cast<cudaStream_t>(stream));
    if (r) return r;
    return launch_bwd_finalize(nullptr, 0, 0, a->dv, a->dkv_dtype, a->dkv_stride_bh,
                               a->dkv_stride_row, a->bh, a->nk, a->h, 0.f,
                               static_cast<cudaStream_t>(stream));
  }
  CUtensorMap tq, tk, tv, tdo;
  const int qt = bwd_q_tile_rows(a->h);
  if ((rc = make_map(&tq, a->q, a->h, a->nq, a->bh, a->q_stride_row, a->q_stride_bh, "q", qt,
                     f16)))
    return rc;
  if ((rc = make_map(&tk, a->k, a->h, a->nk, a->bh / g, a->k_stride_row, a->k_stride_bh, "k", 128,
                     f16)))
    return rc;
  if ((rc = make_map(&tv, a->v, a->h, a->nk, a->bh / g, a->v_stride_row, a->v_stride_bh, "v", 128,
                     f16)))
    return rc;
  if ((rc = make_map(&tdo, a->dout, a->h, a->nq, a->bh, a->do_stride_row, a->do_stride_bh, "dout",
                     qt, f16)))
    return rc;
  return launch_tile_bwd(*a, tq, tk, tv, tdo, static_cast<cudaStream_t>(stream));
}

int a2d_bwd_finalize(const float* dq_acc, int64_t acc_stride_bh, int64_t acc_stride_row, void* dq,
                     int32_t out_dtype, int64_t dq_stride_bh, int64_t dq_stride_row, int32_t bh,
                     int32_t n, int32_t h, float scale, void* stream) {
  if (bh < 0 || n < 0) return set_error(A2D_EINVAL, "negative sizes");
  if (bh == 0 || n == 0) return A2D_OK;
  if (!dq_acc || !dq) return set_error(A2D_EINVAL, "null pointer");
  if (h % 4 || acc_stride_bh % 4 || acc_stride_row % 4 || dq_stride_bh % 4 || dq_stride_row % 4)
    return set_error(A2D_EINVAL, "h and strides must be multiples of 4");
  if (!out16_ok(out_dtype)) return set_error(A2D_EINVAL, "out_dtype invalid");
  return launch_bwd_finalize(dq_acc, acc_stride_bh, acc_stride_row, dq, out_dtype, dq_stride_bh,
                             dq_stride_row, bh, n, h, scale, static_cast<cudaStream_t>(stream));
}

int a2d_lse_merge(const float* o_parts, const float* lse_parts, int32_t k_parts,
                  int64_t part_stride_o, int64_t part_stride_lse, int64_t rows, int32_t h,
                  int64_t row_stride, void* o_out, int32_t out_dtype, int64_t out_row_stride,
                  float* lse_out, void* stream) {
  if (k_parts < 1 || k_parts > 16) return set_error(A2D_EUNSUPPORTED, "k_parts must be in [1, 16]");
  if (h % 4 || row_stride % 4 || part_stride_o % 4)
    return set_error(A2D_EINVAL, "h and strides must be multiples of 4");
  if (rows < 0) return set_error(A2D_EINVAL, "negative sizes");
  if (rows == 0) return A2D_OK;
  if (!o_parts || !lse_parts || !o_out || !lse_out) return set_error(A2D_EINVAL, "null pointer");
  if (!out16_ok(out_dtype)) return set_error(A2D_EINVAL, "out_dtype invalid");
  return launch_lse_merge(o_parts, lse_parts, k_parts, part_stride_o, part_stride_lse, rows, h,
                          row_stride, o_out, out_dtype, out_row_stride, lse_out,
                          static_cast<cudaStream_t>(stream));
}

int a2d_debug_poison(int32_t mode, void* stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return launch_poison(mode, sms, static_cast<cudaStream_t>(stream));
}

int a2d_bench_umma(int32_t variant, int32_t iters, int64_t* cycles_out, int32_t ctas, void* stream) {
  return launch_bench_umma(variant, iters, reinterpret_cast<long long*>(cycles_out), ctas,
                           static_cast<cudaStream_t>(stream));
}

int a2d_selftest_umma(const void* a, const void* b, float* d, int32_t n, int32_t b_mn_major,
                      void* stream) {
  if (n != 64 && n != 128) return set_error(A2D_EUNSUPPORTED, "n must be 64 or 128");
  return launch_selftest_umma(a, b, d, n, b_mn_major, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
