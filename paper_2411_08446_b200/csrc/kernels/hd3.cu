// NEXT-4: cross-polytope hash (Eq. 3) under a structured pseudo-random
// rotation in place of the dense random R of P:L228 — reading R30: x zero-padded to d' = 1024,
// y = H D3 H D2 H D1 x with H the unnormalised Sylvester Hadamard matrix and D_r random +-1
// diagonals, code = sign(y_i*) (i* + 1), i* = argmax_i |y_i| over the d' outputs (ties to the
// smallest i, a zero winner is '+').  Three fast Walsh-Hadamard transforms per hash instead of a
// d x d contraction: O(d' log d') adds on the CUDA cores, no tensor cores.
//
// One warp per token at a time; the 1024-vector lives in registers, 32 fp32 per lane.  Index
// i = 32a + b; layout A: lane a holds b = 0..31 in its registers; layout B: lane b holds a = 0..31.
// H_1024 = H_32(a) (x) H_32(b), so an FWHT is a 32-point transform over the registers, a transpose
// through a warp-private padded 32 x 33 shared tile (conflict-free: bank (a + b) mod 32), and a
// second 32-point transform over the registers.  The two halves commute, so consecutive FWHTs
// alternate A -> B -> A -> B with one transpose each.  The in-register butterflies run on packed
// fp32 pairs (add/sub.rn.f32x2, FADD2 on sm_100a): every stage except the one inside a register
// pair.  The D signs are XORs on the fp32 sign bit.  The final argmax (layout B, i = 32 reg + lane)
// is a per-lane scan plus a 5-step shuffle reduction ordered by (|y| desc, i asc).  The token's x
// for the next iteration is prefetched while the q hashes of the current one run.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../abi/lshmoe_internal.h"

namespace lshmoe {
namespace {

constexpr int kHd3Threads = 256;
constexpr int kHd3Warps = kHd3Threads / 32;
constexpr int kHd3MaxQ = 16;             // LSHMOE_MAX_Q
constexpr int kTile = 32 * 33;           // floats per warp transpose tile

__device__ __forceinline__ void bfly2(float& a0, float& a1, float& b0, float& b1) {
  // (a, b) <- (a + b, a - b) on the pairs (a0, a1), (b0, b1): one FADD2 each way
  unsigned long long A, B, S, D;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(S) : "l"(A), "l"(B));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(S));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(b0), "=f"(b1) : "l"(D));
}

// 32-point unnormalised Walsh-Hadamard transform over the registers (index = register number).
// Registers pair as (r, r + 16): stages h = 1, 2, 4, 8 act on whole pairs (FADD2); stage 16 is the
// butterfly inside each pair (scalar).
__device__ __forceinline__ void wht32(float (&v)[32]) {
#pragma unroll
  for (int h = 1; h < 16; h <<= 1)
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (!(r & h)) bfly2(v[r], v[r + 16], v[r + h], v[r + h + 16]);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const float a = v[r], b = v[r + 16];
    v[r] = a + b;
    v[r + 16] = a - b;
  }
}

// v[r] *= (bit r of m) ? -1 : +1
__device__ __forceinline__ void apply_signs(float (&v)[32], uint32_t m) {
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = __uint_as_float(__float_as_uint(v[r]) ^ ((m << (31 - r)) & 0x80000000u));
}

// Warp transpose through tile[a * 33 + b]: the element a lane holds in register r moves to the lane
// numbered r, register (old lane).  Works for A -> B and B -> A.
__device__ __forceinline__ void transpose(float (&v)[32], float* tile, int lane) {
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) tile[lane * 33 + r] = v[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = tile[r * 33 + lane];
}

template <typename T>
__device__ __forceinline__ void load_row(const T* x, int64_t t, int d, int lane, uint4 (&raw)[8]);

template <>
__device__ __forceinline__ void load_row<__nv_bfloat16>(const __nv_bfloat16* x, int64_t t, int d, int lane,
                                                        uint4 (&raw)[8]) {
  const uint4* row = reinterpret_cast<const uint4*>(x + t * d);   // d % 8 == 0: 16-byte chunks
  const int nch = d / 8;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int ch = 4 * lane + c;                                    // elements 32 lane + 8c ..
    raw[c] = ch < nch ? __ldg(row + ch) : make_uint4(0, 0, 0, 0);
  }
}
template <>
__device__ __forceinline__ void load_row<float>(const float* x, int64_t t, int d, int lane, uint4 (&raw)[8]) {
  const uint4* row = reinterpret_cast<const uint4*>(x + t * d);   // d % 4 == 0
  const int nch = d / 4;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int ch = 8 * lane + c;
    raw[c] = ch < nch ? __ldg(row + ch) : make_uint4(0, 0, 0, 0);
  }
}

template <typename T>
__device__ __forceinline__ void unpack_row(const uint4 (&raw)[8], float (&x)[32]) {
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t w[4] = {raw[c].x, raw[c].y, raw[c].z, raw[c].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[8 * c + 2 * i] = __uint_as_float(w[i] << 16);
        x[8 * c + 2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      x[4 * c + 0] = __uint_as_float(raw[c].x);
      x[4 * c + 1] = __uint_as_float(raw[c].y);
      x[4 * c + 2] = __uint_as_float(raw[c].z);
      x[4 * c + 3] = __uint_as_float(raw[c].w);
    }
  }
}

// signs: [q][3][32] words, bit b of word a = 1 iff D_r[32a + b] = -1 (lshmoe_hd3_signs).
template <typename T>
__global__ void __launch_bounds__(kHd3Threads, 2) hd3_hash_kernel(const T* __restrict__ x, int64_t n, int d,
                                                                  const uint32_t* __restrict__ signs, int q,
                                                                  int16_t* __restrict__ codes) {
  __shared__ float s_tile[kHd3Warps * kTile];
  __shared__ uint32_t s_mA[kHd3MaxQ][3][32];   // layout-A words (D1, D3; D2 unused)
  __shared__ uint32_t s_mB[kHd3MaxQ][32];      // D2 in layout B: bit a of word b = sign of 32a + b
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < q * 3 * 32; i += kHd3Threads) (&s_mA[0][0][0])[i] = signs[i];
  __syncthreads();
  for (int i = threadIdx.x; i < q * 32; i += kHd3Threads) {
    const int j = i / 32, b = i % 32;
    uint32_t w = 0;
    for (int a = 0; a < 32; ++a) w |= ((s_mA[j][1][a] >> b) & 1u) << a;
    s_mB[j][b] = w;
  }
  __syncthreads();
  float* tile = s_tile + warp * kTile;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kHd3Warps + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kHd3Warps;
  uint4 raw[8];
  if (gw < n) load_row<T>(x, gw, d, lane, raw);
  for (int64_t t = gw; t < n; t += nw) {
    float xa[32];
    unpack_row<T>(raw, xa);
    if (t + nw < n) load_row<T>(x, t + nw, d, lane, raw);          // next token in flight
    int my_code = 0;
#pragma unroll 1
    for (int j = 0; j < q; ++j) {
      float v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = xa[r];
      apply_signs(v, s_mA[j][0][lane]);                              // D1 (layout A)
      wht32(v);                                                      // FWHT 1: H over b
      transpose(v, tile, lane);                                      //   -> layout B
      wht32(v);                                                      //   H over a
      apply_signs(v, s_mB[j][lane]);                                 // D2 (layout B)
      wht32(v);                                                      // FWHT 2: H over a
      transpose(v, tile, lane);                                      //   -> layout A
      wht32(v);                                                      //   H over b
      apply_signs(v, s_mA[j][2][lane]);                              // D3 (layout A)
      wht32(v);                                                      // FWHT 3: H over b
      transpose(v, tile, lane);                                      //   -> layout B
      wht32(v);                                                      //   H over a
      // argmax over i = 32 r + lane: registers ascend in i, so strict '>' keeps the smallest i
      float best = fabsf(v[0]), val = v[0];
      int bi = 0;
#pragma unroll
      for (int r = 1; r < 32; ++r)
        if (fabsf(v[r]) > best) {
          best = fabsf(v[r]);
          val = v[r];
          bi = r;
        }
      int idx = 32 * bi + lane;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const float ob = __shfl_xor_sync(0xFFFFFFFFu, best, off);
        const float ov = __shfl_xor_sync(0xFFFFFFFFu, val, off);
        const int oi = __shfl_xor_sync(0xFFFFFFFFu, idx, off);
        if (ob > best || (ob == best && oi < idx)) {
          best = ob;
          val = ov;
          idx = oi;
        }
      }
      const int code = val < 0.0f ? -(idx + 1) : idx + 1;
      if (lane == j) my_code = code;
    }
    if (lane < q) codes[t * q + lane] = static_cast<int16_t>(my_code);
  }
}

}  // namespace

int launch_hd3_hash(const void* x, int is_bf16, int64_t n, int d, const uint32_t* signs, int q, int16_t* codes,
                    void* stream) {
  if (q > kHd3MaxQ || d > 1024) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t warps_needed = n;
  int grid = 2 * device_sm_count();                                   // two 8-warp CTAs per SM
  if (warps_needed < static_cast<int64_t>(grid) * kHd3Warps) grid = static_cast<int>((warps_needed + kHd3Warps - 1) / kHd3Warps);
  if (grid < 1) return 0;
  if (is_bf16)
    hd3_hash_kernel<__nv_bfloat16><<<grid, kHd3Threads, 0, st>>>(static_cast<const __nv_bfloat16*>(x), n, d, signs, q,
                                                                 codes);
  else
    hd3_hash_kernel<float><<<grid, kHd3Threads, 0, st>>>(static_cast<const float*>(x), n, d, signs, q, codes);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lshmoe
