// kernels.h — internal launcher declarations shared by the .cu files.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../include/attn2d_b200.h"

namespace a2d {

// error plumbing (abi.cu)
int set_error(int code, const char* fmt, ...);
int set_cuda_error(cudaError_t e, const char* what);
int check_launch(const char* what);

int launch_tile_fwd(const a2d_tile_fwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, cudaStream_t stream);
int launch_tile_bwd(const a2d_tile_bwd_args& a, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, const CUtensorMap& tdo, cudaStream_t stream);
int launch_lse_merge(const float* o_parts, const float* lse_parts, int k_parts,
                     long long part_stride_o, long long part_stride_lse, long long rows, int h,
                     long long row_stride, void* o_out, int out_dtype, long long out_row_stride,
                     float* lse_out, cudaStream_t stream);
int launch_bwd_preprocess(const void* o, const void* dout, float* delta, long long o_sbh,
                          long long o_srow, long long do_sbh, long long do_srow, int bh, int n,
                          int h, bool f16, cudaStream_t stream);
int launch_bwd_finalize(const float* dq_acc, long long asbh, long long asrow, void* dq,
                        int out_dtype, long long sbh, long long srow, int bh, int n, int h,
                        float scale, cudaStream_t stream);
int make_map_bf16(CUtensorMap* m, const void* ptr, int h, int rows, int bh, long long s_row,
                  long long s_bh, const char* name, int box_rows);
int make_map_f32_dq(CUtensorMap* m, const float* ptr, int h, int rows, int bh, long long s_row,
                    long long s_bh, int box_rows);
int make_map_f32_dq_flat(CUtensorMap* m, const float* ptr, int h, int rows, int bh,
                         long long s_row, long long s_bh, int box_rows, int box_cols = 0);
int bwd_q_tile_rows(int h);
int launch_poison(int mode, int num_sms, cudaStream_t stream);
int launch_bench_umma(int variant, int iters, long long* out, int ctas, cudaStream_t stream);
int launch_selftest_umma(const void* a, const void* b, float* d, int n, int b_mn_major,
                         cudaStream_t stream);

}  // namespace a2d
