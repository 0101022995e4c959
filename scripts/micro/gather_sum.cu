// Microbenchmark (tuning aid, not part of the library): gather-and-sum of n random bf16 rows
// (d = 768) into per-warp sums, the memory pattern of the centroid phase.  Variants:
//   0: register loads, one row per iteration      1: register loads, 4 rows in flight
//   2: cp.async ring (per-warp, 10 rows deep)
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

constexpr int D = 768, RB = D * 2, NC = RB / 16;   // 96 chunks

__device__ __forceinline__ void add16(float* a, uint4 r) {
  const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[2 * i] += __uint_as_float(u[i] << 16); a[2 * i + 1] += __uint_as_float(u[i] & 0xFFFF0000u); }
}

template <int V>
__global__ void __launch_bounds__(256, 1) k(const uint8_t* x, const int* tok, int n, float* out) {
  const int lane = threadIdx.x % 32, gw = blockIdx.x * 8 + threadIdx.x / 32, GW = gridDim.x * 8;
  const int b = (int)((int64_t)gw * n / GW), e = (int)((int64_t)(gw + 1) * n / GW);
  float acc[3][8] = {};
  if (V == 3) { if (n < 0) out[0] = 1; return; }
  if (V == 0) {
    for (int p = b; p < e; ++p) {
      const uint4* src = reinterpret_cast<const uint4*>(x + (int64_t)tok[p] * RB);
#pragma unroll
      for (int t = 0; t < 3; ++t) add16(acc[t], __ldg(src + lane + 32 * t));
    }
  } else if (V == 1) {
    int p = b;
    for (; p + 4 <= e; p += 4) {
      uint4 v[4][3];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint4* src = reinterpret_cast<const uint4*>(x + (int64_t)tok[p + r] * RB);
#pragma unroll
        for (int t = 0; t < 3; ++t) v[r][t] = __ldg(src + lane + 32 * t);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int t = 0; t < 3; ++t) add16(acc[t], v[r][t]);
    }
    for (; p < e; ++p) {
      const uint4* src = reinterpret_cast<const uint4*>(x + (int64_t)tok[p] * RB);
#pragma unroll
      for (int t = 0; t < 3; ++t) add16(acc[t], __ldg(src + lane + 32 * t));
    }
  } else {
    extern __shared__ __align__(16) uint8_t sm[];
    uint8_t* ring = sm + (threadIdx.x / 32) * 10 * RB;
    auto issue = [&](int p) {
      if (p < e) {
        const uint8_t* src = x + (int64_t)tok[p] * RB;
        uint8_t* dst = ring + ((p - b) % 10) * RB;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int c = lane + 32 * t;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst + 16 * c)), "l"(src + 16 * c) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int i = 0; i < 9; ++i) issue(b + i);
    for (int p = b; p < e; ++p) {
      issue(p + 9);
      asm volatile("cp.async.wait_group 9;" ::: "memory");
      const uint8_t* st = ring + ((p - b) % 10) * RB;
#pragma unroll
      for (int t = 0; t < 3; ++t) add16(acc[t], *reinterpret_cast<const uint4*>(st + 16 * (lane + 32 * t)));
    }
  }
  float s = 0;
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[t][i];
  out[gw * 32 + lane] = s;
}

int main() {
  const int n = 16384;
  uint8_t* x; int* tok; float* out; int* flush;
  cudaMalloc(&x, (size_t)n * RB); cudaMalloc(&tok, n * 4); cudaMalloc(&out, 148 * 8 * 8 * 32 * 4);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(x, 0x3f, (size_t)n * RB);
  std::vector<int> h(n); for (int i = 0; i < n; ++i) h[i] = i;
  std::shuffle(h.begin(), h.end(), std::mt19937(1));
  cudaMemcpy(tok, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 10 * RB);
  cudaEvent_t a, c; cudaEventCreate(&a); cudaEventCreate(&c);
  for (int flushit = 0; flushit < 2; ++flushit)
  for (int v = 0; v < 7; ++v) {
    std::vector<float> ts;
    for (int it = 0; it < 20; ++it) {
      if (flushit) cudaMemsetAsync(flush, it, 256 << 20);
      cudaEventRecord(a);
      if (v == 0) k<0><<<148, 256>>>(x, tok, n, out);
      if (v == 1) k<1><<<148, 256>>>(x, tok, n, out);
      if (v == 2) k<2><<<148, 256, 8 * 10 * RB>>>(x, tok, n, out);
      if (v == 3) k<0><<<148 * 4, 256>>>(x, tok, n, out);
      if (v == 4) k<1><<<148 * 4, 256>>>(x, tok, n, out);
      if (v == 5) k<0><<<148 * 8, 256>>>(x, tok, n, out);
      if (v == 6) k<3><<<148, 256>>>(x, tok, n, out);
      cudaEventRecord(c); cudaEventSynchronize(c);
      float ms; cudaEventElapsedTime(&ms, a, c); ts.push_back(ms * 1e3f);
    }
    std::sort(ts.begin(), ts.end());
    printf("variant %d flush %d: median %.1f us  (%.0f GB/s)\n", v, flushit, ts[10], (double)n * RB / ts[10] / 1e3);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
