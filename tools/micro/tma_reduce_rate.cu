// Micro-benchmark: throughput of the fp32 reduce-add paths the backward's
// dQ drain can use, one CTA per SM (148), from a 32 KB staging area in
// shared memory (4 x 8 KB buffers, up to DEPTH reduce groups in flight) into
// a large fp32 accumulator (rows rotated per CTA, like the drain's query sweep):
//   mode 0: cp.reduce.async.bulk.tensor.3d (TMA tensor reduce, 16 x 128 fp32 box)
//   mode 1: cp.reduce.async.bulk (1-D bulk reduce of the same 8 KB, contiguous rows)
//   mode 2: cp.async.bulk.tensor store (no reduction) of the same box
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_15758_b200/csrc
//   -o /tmp/tma_reduce_rate tools/micro/tma_reduce_rate.cu -lcuda && /tmp/tma_reduce_rate
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace a2d;

constexpr int ROWS_PER_BOX = 16, COLS = 128, BOX_BYTES = ROWS_PER_BOX * COLS * 4;

template <int MODE, int DEPTH, int REQ = BOX_BYTES>
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tm, float* acc,
                                            int rows, int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  float* s = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < 4 * BOX_BYTES / 4; i += blockDim.x) s[i] = 1e-3f;
  fence_proxy_async_smem();
  __syncthreads();
  __shared__ __align__(8) uint64_t lbar[4];
  if (threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&lbar[i]), 1);
  fence_mbar_init();
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nbox = rows / ROWS_PER_BOX;
  if (MODE >= 5) {  // 5: TMA tensor loads only; 6: loads and reduce-adds alternating
    long long t0 = clock64();
    int use[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
      const int box = (blockIdx.x * 37 + it) % nbox;
      const int b = it & 3;
      const uint32_t buf = sb + b * BOX_BYTES;
      const bool load = MODE == 5 || (it & 1);
      if (load) {
        if (use[b] > 0) mbar_wait(smem_u32(&lbar[b]), (use[b] - 1) & 1);
        bulk_wait_group_read<0>();
        mbar_expect_tx(smem_u32(&lbar[b]), BOX_BYTES);
        tma_load_3d(buf, &tm, smem_u32(&lbar[b]), 0, box * ROWS_PER_BOX, 0);
        ++use[b];
      } else {
        if (use[b] > 0) mbar_wait(smem_u32(&lbar[b]), (use[b] - 1) & 1);
        bulk_wait_group_read<1>();
        tma_reduce_add_3d_g(&tm, buf, 0, box * ROWS_PER_BOX, 0);
        bulk_commit_group();
      }
    }
    for (int b = 0; b < 4; ++b)
      if (use[b] > 0) mbar_wait(smem_u32(&lbar[b]), (use[b] - 1) & 1);
    bulk_wait_group_all();
    cyc[blockIdx.x] = clock64() - t0;
    return;
  }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int box = (blockIdx.x * 37 + it) % nbox;
    const uint32_t buf = sb + (it & 3) * BOX_BYTES;
    bulk_wait_group_read<DEPTH - 1>();
    if (MODE == 0) {
      tma_reduce_add_3d_g(&tm, buf, 0, box * ROWS_PER_BOX, 0);
    } else if (MODE == 1) {
      float* dst = acc + (long long)box * ROWS_PER_BOX * COLS;
      // REQ-byte requests from a ring of 32 KB / REQ buffers
      const int nb = 4 * BOX_BYTES / REQ;
      const uint32_t b2 = sb + (it % nb) * REQ;
      float* d2 = acc + ((long long)box * ROWS_PER_BOX * COLS) % ((long long)rows * COLS - REQ / 4);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                   ::"l"(d2), "r"(b2), "r"(REQ) : "memory");
      (void)dst;
    } else {
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group"
                   " [%0, {%2, %3, %4}], [%1];" ::"l"(reinterpret_cast<uint64_t>(&tm)),
                   "r"(buf), "r"(0), "r"(box * ROWS_PER_BOX), "r"(0) : "memory");
    }
    bulk_commit_group();
  }
  bulk_wait_group_all();
  cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

template <int MODE, int DEPTH, int REQ = BOX_BYTES>
void run(const CUtensorMap& tm, float* acc, int rows, long long* dcyc, const char* name,
         int ctas = 148) {
  const int iters = 2048;
  auto kern = k<MODE, DEPTH, REQ>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * BOX_BYTES);
  for (int rep = 0; rep < 2; ++rep) kern<<<ctas, 128, 4 * BOX_BYTES>>>(tm, acc, rows, iters, dcyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, dcyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < ctas; ++i) mean += h[i];
  mean /= ctas;
  printf("%-42s depth %d, %3d CTAs, %4d MB target: %6.1f B/clk per SM (%s)\n", name, DEPTH, ctas,
         int((long long)rows * COLS * 4 >> 20), (double)iters * (MODE == 1 ? REQ : BOX_BYTES) / mean,
         e == cudaSuccess ? "ok" : cudaGetErrorString(e));
}

int main() {
  const int rows = 32 * 131072;  // 2 GiB fp32 accumulator, like dQ_acc at the metric point
  float* acc;
  long long* dcyc;
  cudaMalloc(&acc, (size_t)rows * COLS * 4);
  cudaMemset(acc, 0, (size_t)rows * COLS * 4);
  cudaMalloc(&dcyc, 148 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {COLS, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {COLS * 4, (cuuint64_t)rows * COLS * 4};
  cuuint32_t box[3] = {COLS, ROWS_PER_BOX, 1}, es[3] = {1, 1, 1};
  CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, acc, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  run<0, 4>(tm, acc, rows, dcyc, "TMA tensor reduce-add (8 KB boxes)");
  run<0, 2>(tm, acc, rows, dcyc, "TMA tensor reduce-add (8 KB boxes)");
  run<0, 1>(tm, acc, rows, dcyc, "TMA tensor reduce-add (8 KB boxes)");
  run<1, 4>(tm, acc, rows, dcyc, "1-D bulk reduce-add (8 KB)");
  run<2, 4>(tm, acc, rows, dcyc, "TMA tensor store (8 KB boxes, no reduction)");
  // L2-resident target (32 MB: one head's dQ accumulator at N = 64K), and one SM alone
  CUtensorMap tms;
  const int rows_s = 65536;
  cuuint64_t dims_s[3] = {COLS, (cuuint64_t)rows_s, 1};
  cuuint64_t strides_s[2] = {COLS * 4, (cuuint64_t)rows_s * COLS * 4};
  r = ((EncodeFn)fn)(&tms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, acc, dims_s, strides_s, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  run<0, 4>(tms, acc, rows_s, dcyc, "TMA tensor reduce-add (8 KB boxes)");
  run<0, 4>(tms, acc, rows_s, dcyc, "TMA tensor reduce-add (8 KB boxes)", 1);
  run<0, 4>(tms, acc, rows_s, dcyc, "TMA tensor reduce-add (8 KB boxes)", 16);
  run<2, 4>(tms, acc, rows_s, dcyc, "TMA tensor store (8 KB boxes, no reduction)");
  run<2, 4>(tms, acc, rows_s, dcyc, "TMA tensor store (8 KB boxes, no reduction)", 1);
  run<1, 4, 2048>(tms, acc, rows_s, dcyc, "1-D bulk reduce-add, 2 KB requests");
  run<1, 4, 4096>(tms, acc, rows_s, dcyc, "1-D bulk reduce-add, 4 KB requests");
  run<1, 2, 16384>(tms, acc, rows_s, dcyc, "1-D bulk reduce-add, 16 KB requests");
  run<1, 1, 32768>(tms, acc, rows_s, dcyc, "1-D bulk reduce-add, 32 KB requests");
  run<1, 8, 4096>(tms, acc, rows_s, dcyc, "1-D bulk reduce-add, 4 KB requests");
  run<5, 4>(tms, acc, rows_s, dcyc, "TMA tensor load (8 KB boxes)");
  run<5, 4>(tms, acc, rows_s, dcyc, "TMA tensor load (8 KB boxes)", 1);
  run<6, 4>(tms, acc, rows_s, dcyc, "TMA loads + reduce-adds alternating (8 KB)");
  return 0;
}
