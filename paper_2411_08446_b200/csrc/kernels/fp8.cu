// NEXT-2's fp8 option (reading R28): per-token power-of-two scaling of x to e4m3.
// Eq. 3's argmax is invariant to a positive scale of the token, so each row is scaled
// by the largest 2^k with max|x| * 2^k <= 448 (exact in fp32) and rounded to e4m3 (RNE,
// __nv_cvt_float_to_fp8); lshmoe_hash_e4m3 then hashes the e4m3 values on kind::f8f6f4 tensor
// cores.  One warp per row; 128-bit loads, 64-bit stores.
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../abi/lshmoe_internal.h"

namespace lshmoe {
namespace {

__global__ void __launch_bounds__(256) quantize_e4m3_kernel(const __nv_bfloat16* __restrict__ x, int64_t n, int d,
                                                            uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int cpr = d / 8;                        // 16-byte chunks (8 bf16) per row
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x / 32) + threadIdx.x / 32; t < n; t += warps) {
    const uint4* row = reinterpret_cast<const uint4*>(x + t * d);
    float vmax = 0.0f;
    for (int ch = lane; ch < cpr; ch += 32) {
      const uint4 v = __ldg(row + ch);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
        vmax = fmaxf(vmax, fmaxf(fabsf(__uint_as_float(w[i] << 16)), fabsf(__uint_as_float(w[i] & 0xFFFF0000u))));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xFFFFFFFFu, vmax, off));
    float scale = 1.0f;
    if (vmax > 0.0f) {                          // largest 2^k with vmax * 2^k <= 448 = 0.875 * 2^9
      int e;
      const float f = frexpf(vmax, &e);         // vmax = f * 2^e, f in [0.5, 1)
      scale = ldexpf(1.0f, f <= 0.875f ? 9 - e : 8 - e);
    }
    uint2* orow = reinterpret_cast<uint2*>(out + t * d);
    for (int ch = lane; ch < cpr; ch += 32) {
      const uint4 v = __ldg(row + ch);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      uint32_t packed[2] = {0, 0};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = __uint_as_float(w[i] << 16) * scale, b = __uint_as_float(w[i] & 0xFFFF0000u) * scale;
        const uint32_t qa = __nv_cvt_float_to_fp8(a, __NV_SATFINITE, __NV_E4M3);
        const uint32_t qb = __nv_cvt_float_to_fp8(b, __NV_SATFINITE, __NV_E4M3);
        packed[i / 2] |= (qa | (qb << 8)) << (16 * (i % 2));
      }
      orow[ch] = make_uint2(packed[0], packed[1]);
    }
  }
}

}  // namespace

int launch_quantize_e4m3(const void* x, int64_t n, int d, uint8_t* out, void* stream) {
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, 16 * int64_t(device_sm_count()))));
  quantize_e4m3_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const __nv_bfloat16*>(x), n,
                                                                          d, out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lshmoe
