// Microbenchmark (tuning aid, not part of the library): stream a 2 GiB bf16 weight matrix
// [R rows, K = 1024 cols] from HBM into shared memory with TMA, one CTA per SM, 8-stage ring of
// 128-row x 64-col (16 KB) boxes, no math -- the expert FFN's B-operand pattern.  Layout A: plain
// row-major (each box = 128 row segments of 128 B at a 2 KB stride); layout P: packed so that
// every box is 16 KB contiguous ([R/128][K/64][128][64]).  Work per CTA: contiguous row blocks, all
// 16 k-blocks of a row block in order (the GEMM's order).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cstdlib>

constexpr int K = 1024, BK = 64, BR = 128, STAGES = 8, BOX = BR * BK * 2;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(sa(b)), "r"(ph) : "memory");
}

template <int PACKED>
__global__ void __launch_bounds__(64, 1) stream_k(const __grid_constant__ CUtensorMap m, int nrb, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int rb0 = (int)((int64_t)blockIdx.x * nrb / gridDim.x), rb1 = (int)((int64_t)(blockIdx.x + 1) * nrb / gridDim.x);
  const int total = (rb1 - rb0) * (K / BK);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      wait(&empty[s], ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(BOX) : "memory");
      const int rb = rb0 + i / (K / BK), kb = i % (K / BK);
      if (PACKED)
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                     ::"r"(sa(sm + s * BOX)), "l"(&m), "r"(sa(&full[s])), "r"(0), "r"(0), "r"(kb), "r"(rb) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(sa(sm + s * BOX)), "l"(&m), "r"(sa(&full[s])), "r"(kb * BK), "r"(rb * BR) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    int acc = 0;
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      wait(&full[s], (i / STAGES) & 1);
      acc += sm[s * BOX + (i & 1023)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
    if (acc == 0x7fffffff) sink[0] = acc;
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  Enc enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int64_t R = 1 << 20;                       // 1M rows x 1024 cols x 2 B = 2 GiB
  const int nrb = (int)(R / BR);
  void* w; cudaMalloc(&w, R * K * 2); cudaMemset(w, 1, R * K * 2);
  int* sink; cudaMalloc(&sink, 4);
  CUtensorMap m2, m4;
  { cuuint64_t dims[2] = {K, (cuuint64_t)R}, str[1] = {K * 2}; cuuint32_t box[2] = {BK, BR}, es[2] = {1, 1};
    enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  { cuuint64_t dims[4] = {BK, BR, K / BK, (cuuint64_t)nrb};
    cuuint64_t str[3] = {BK * 2, (cuuint64_t)BOX, (cuuint64_t)BOX * (K / BK)};
    cuuint32_t box[4] = {BK, BR, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode4 failed %d\n", (int)r); }
  const int smem = STAGES * BOX;
  cudaFuncSetAttribute(stream_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<int> grids = {148, 296};
  if (argc > 1) { grids.clear(); for (int i = 1; i < argc; ++i) grids.push_back(atoi(argv[i])); }
  for (int grid : grids) {
    for (int v = 0; v < 2; ++v) {
      std::vector<float> ts;
      for (int it = 0; it < 7; ++it) {
        cudaEventRecord(a);
        if (v == 0) stream_k<0><<<grid, 64, smem>>>(m2, nrb, sink);
        else stream_k<1><<<grid, 64, smem>>>(m4, nrb, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ts.push_back(ms);
      }
      std::sort(ts.begin(), ts.end());
      printf("grid %d layout %s: %.3f ms  %.0f GB/s\n", grid, v ? "packed" : "row-major", ts[3], R * K * 2 / ts[3] / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
