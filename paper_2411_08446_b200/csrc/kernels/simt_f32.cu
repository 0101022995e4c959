// fp32 (SIMT) kernels for the f32 configuration (BASELINE.json configs[0], d = 64):
//  * hash_f32_kernel — Eq. 3 with fp32 FMA accumulation over k in ascending order.
//    Not tf32 tensor cores: tf32 rounding (~5e-4 relative) would exceed the 1e-5 near-tie band
//    of BASELINE.json's tier 1 (reading R19).
//  * ffn_f32_kernel — E(x) = W2 relu(W1 x + b1) + b2 for the received rows.
#include <cuda_runtime.h>

#include "../abi/lshmoe_internal.h"
#include "common.cuh"

namespace lshmoe {
namespace {

constexpr int kTok = 128;     // tokens per CTA (one per thread)
constexpr int kRowsR = 32;    // rotation rows staged per step
constexpr int kXs = kTok + 1; // padded smem pitch of the transposed x tile (no bank conflicts)

// grid (ceil(n / 128), q), 128 x kRG threads: thread (g, t) scans rotation rows i = g (mod kRG) for
// token t in ascending i, then the kRG partial winners meet in shared memory (larger |y|, ties to
// the smaller index: the same winner as one ascending scan).  smem: x tile transposed [d][128] +
// R rows [32][d] + the partial winners.
constexpr int kRG = 4;
__global__ void __launch_bounds__(kTok * kRG) hash_f32_kernel(const float* __restrict__ x, int n, int d,
                                                              const float* __restrict__ R, int q,
                                                              int16_t* __restrict__ codes) {
  extern __shared__ float sm[];
  float* xs = sm;                      // [d][kXs]
  float* rs = sm + d * kXs;            // [kRowsR][d]
  __shared__ float s_best[kRG][kTok];
  __shared__ int s_idx[kRG][kTok];
  const int tl = threadIdx.x % kTok, grp = threadIdx.x / kTok;
  const int t0 = blockIdx.x * kTok;
  const int j = blockIdx.y;
  const float* Rj = R + static_cast<int64_t>(j) * d * d;
#pragma unroll 8   // several loads in flight per thread (the tile is one dependent round trip, not 16)
  for (int i = threadIdx.x; i < d * kTok; i += kTok * kRG) {
    const int tt = i / d, k = i - tt * d;                // coalesced read of x rows
    const int t = t0 + tt;
    xs[k * kXs + tt] = t < n ? x[static_cast<int64_t>(t) * d + k] : 0.0f;
  }
  float best = -1.0f;
  int bidx = 0;
  bool bneg = false;
  for (int i0 = 0; i0 < d; i0 += kRowsR) {
    const int rows = min(kRowsR, d - i0);
    __syncthreads();
#pragma unroll 8
    for (int i = threadIdx.x; i < rows * d; i += kTok * kRG) rs[i] = Rj[static_cast<int64_t>(i0) * d + i];
    __syncthreads();
    for (int ii = grp; ii < rows; ii += kRG) {
      const float* rrow = rs + ii * d;
      float y = 0.0f;
#pragma unroll 8   // the shared-memory loads of 8 steps issue together; the FMA chain keeps ascending k
      for (int k = 0; k < d; ++k) y = fmaf(rrow[k], xs[k * kXs + tl], y);
      const float a = fabsf(y);
      if (a > best) {          // ties keep the smaller index; a zero winner is '+' (R2)
        best = a;
        bidx = i0 + ii;
        bneg = y < 0.0f;
      }
    }
  }
  s_best[grp][tl] = best;
  s_idx[grp][tl] = bneg ? -(bidx + 1) : (bidx + 1);
  __syncthreads();
  const int t = t0 + tl;
  if (grp == 0 && t < n) {
    float b = s_best[0][tl];
    int c = s_idx[0][tl];
    for (int g2 = 1; g2 < kRG; ++g2) {
      const float a = s_best[g2][tl];
      const int c2 = s_idx[g2][tl];
      if (a > b || (a == b && abs(c2) < abs(c))) {
        b = a;
        c = c2;
      }
    }
    codes[static_cast<int64_t>(t) * q + j] = static_cast<int16_t>(c);
  }
}

// NEXT-3 SP hash, fp32: grid ceil(n / 128) CTAs, one token per thread, the q*b normals staged 32
// rows at a time; bit i of hash j = (n_{j*b+i} . x >= 0), fp32 FMA in ascending k (reading R26).
__global__ void __launch_bounds__(kTok) sp_hash_f32_kernel(const float* __restrict__ x, int n, int d,
                                                           const float* __restrict__ N, int q, int b,
                                                           int16_t* __restrict__ codes) {
  extern __shared__ float sm[];
  float* xs = sm;                      // [d][kXs]
  float* rs = sm + d * kXs;            // [kRowsR][d]
  const int t0 = blockIdx.x * kTok;
  for (int i = threadIdx.x; i < d * kTok; i += kTok) {
    const int tt = i / d, k = i - tt * d;
    const int t = t0 + tt;
    xs[k * kXs + tt] = t < n ? x[static_cast<int64_t>(t) * d + k] : 0.0f;
  }
  const int nb = q * b;
  uint32_t bits[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // up to 256 sign bits
  for (int i0 = 0; i0 < nb; i0 += kRowsR) {
    const int rows = min(kRowsR, nb - i0);
    __syncthreads();
    for (int i = threadIdx.x; i < rows * d; i += kTok) rs[i] = N[static_cast<int64_t>(i0) * d + i];
    __syncthreads();
    uint32_t m = 0;
    for (int ii = 0; ii < rows; ++ii) {
      const float* rrow = rs + ii * d;
      float y = 0.0f;
      for (int k = 0; k < d; ++k) y = fmaf(rrow[k], xs[k * kXs + threadIdx.x], y);
      m |= (y >= 0.0f ? 1u : 0u) << ii;
    }
#pragma unroll
    for (int w = 0; w < 8; ++w)
      if (w == i0 / kRowsR) bits[w] = m;
  }
  const int t = t0 + threadIdx.x;
  if (t >= n) return;
  for (int j = 0; j < q; ++j) {
    const int c0 = j * b, wi = c0 >> 5, sh = c0 & 31;
    uint64_t v = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      if (w == wi) v |= bits[w];
      if (w == wi + 1) v |= static_cast<uint64_t>(bits[w]) << 32;
    }
    codes[static_cast<int64_t>(t) * q + j] = static_cast<int16_t>((v >> sh) & ((1u << b) - 1u));
  }
}

// One thread per output element of one GEMM layer over rows segmented by expert:
// out[r][o] = act(sum_i W[e][o][i] * in[r][i] + b[e][o]).  Segment table recomputed per CTA.
// b nullable (no bias); mask nullable: out *= [mask[r][o] > 0] (NEXT-1: relu' from the forward's
// saved hidden activations).
__global__ void ffn_f32_layer_kernel(const float* __restrict__ in, int K, int N, const int32_t* __restrict__ recv_rows,
                                     int E_local, int world, const float* __restrict__ W, const float* __restrict__ b,
                                     float* __restrict__ out, int64_t capacity, int relu,
                                     const float* __restrict__ mask = nullptr) {
  __shared__ int seg_end[257];
  if (threadIdx.x == 0) {
    int rows = 0;
    for (int e = 0; e < E_local; ++e) {
      for (int s = 0; s < world; ++s) rows += recv_rows[e * world + s];
      seg_end[e] = rows;
    }
  }
  __syncthreads();
  const int64_t total = static_cast<int64_t>(seg_end[E_local - 1]) * N;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total; idx += int64_t(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx / N), o = static_cast<int>(idx - int64_t(r) * N);
    int e = 0;
    while (seg_end[e] <= r) ++e;
    const float* w = W + (static_cast<int64_t>(e) * N + o) * K;
    const float* xi = in + static_cast<int64_t>(r) * K;
    float acc = 0.0f;
    for (int i = 0; i < K; ++i) acc = fmaf(w[i], xi[i], acc);
    if (b) acc += b[static_cast<int64_t>(e) * N + o];
    if (mask && !(mask[static_cast<int64_t>(r) * N + o] > 0.0f)) acc = 0.0f;
    out[static_cast<int64_t>(r) * N + o] = relu ? fmaxf(acc, 0.0f) : acc;
  }
}

}  // namespace

int launch_sp_hash_f32(const float* x, int64_t n, int d, const float* N, int q, int b, int16_t* codes,
                       void* stream) {
  const int smem = (d * kXs + kRowsR * d) * 4;
  if (smem > 48 * 1024) {
    const int err = cudaFuncSetAttribute(sp_hash_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err) return err;
  }
  sp_hash_f32_kernel<<<static_cast<int>((n + kTok - 1) / kTok), kTok, smem, static_cast<cudaStream_t>(stream)>>>(
      x, static_cast<int>(n), d, N, q, b, codes);
  count_launches(1);
  return cudaGetLastError();
}

int launch_hash_f32(const float* x, int64_t n, int d, const float* R, int q, int16_t* codes, void* stream) {
  const size_t smem = sizeof(float) * (static_cast<size_t>(d) * kXs + kRowsR * d);
  static int configured_smem = 0;
  if (static_cast<int>(smem) > configured_smem) {
    int err = cudaFuncSetAttribute(hash_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (err) return err;
    configured_smem = static_cast<int>(smem);
  }
  dim3 grid(static_cast<unsigned>((n + kTok - 1) / kTok), q);
  hash_f32_kernel<<<grid, kTok * kRG, smem, static_cast<cudaStream_t>(stream)>>>(x, static_cast<int>(n), d, R, q,
                                                                                 codes);
  count_launches(1);
  return cudaGetLastError();
}

int launch_ffn_bf16(const void* in, int d, int d_ffn, const int32_t* recv_rows, int E_local, int world, const void* W1,
                    const void* b1, const void* W2, const void* b2, void* hidden, int64_t capacity, void* out,
                    void* stream);

int launch_expert_ffn(const void* in, lshmoe_dtype dtype, int d, int d_ffn, const int32_t* recv_rows, int E_local,
                      int world, const void* W1, const void* b1, const void* W2, const void* b2, void* hidden,
                      int64_t capacity, void* out, void* stream) {
  if (dtype == LSHMOE_BF16)
    return launch_ffn_bf16(in, d, d_ffn, recv_rows, E_local, world, W1, b1, W2, b2, hidden, capacity, out, stream);
  if (E_local > 256) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = 4 * device_sm_count();
  ffn_f32_layer_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(in), d, d_ffn, recv_rows, E_local, world,
                                            static_cast<const float*>(W1), static_cast<const float*>(b1),
                                            static_cast<float*>(hidden), capacity, 1);
  int err = cudaGetLastError();
  if (err) return err;
  ffn_f32_layer_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(hidden), d_ffn, d, recv_rows, E_local, world,
                                            static_cast<const float*>(W2), static_cast<const float*>(b2),
                                            static_cast<float*>(out), capacity, 0);
  count_launches(2);
  return cudaGetLastError();
}

int launch_expert_ffn_backward(const void* grad_out, lshmoe_dtype dtype, int d, int d_ffn, const int32_t* recv_rows,
                               int E_local, int world, const void* W2T, const void* W1T, const void* hidden,
                               void* dhidden, int64_t capacity, void* grad_in, void* stream) {
  if (dtype == LSHMOE_BF16)
    return launch_ffn_bwd_bf16(grad_out, d, d_ffn, recv_rows, E_local, world, W2T, W1T, hidden, dhidden, capacity,
                               grad_in, stream);
  if (E_local > 256) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = 4 * device_sm_count();
  // dh = (G W2) * [h > 0]  (W2T = W2^T per expert, [d_ffn, d]);  H = dh W1  (W1T = W1^T, [d, d_ffn])
  ffn_f32_layer_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(grad_out), d, d_ffn, recv_rows, E_local, world,
                                            static_cast<const float*>(W2T), nullptr, static_cast<float*>(dhidden),
                                            capacity, 0, static_cast<const float*>(hidden));
  int err = cudaGetLastError();
  if (err) return err;
  ffn_f32_layer_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(dhidden), d_ffn, d, recv_rows, E_local, world,
                                            static_cast<const float*>(W1T), nullptr, static_cast<float*>(grad_in),
                                            capacity, 0, nullptr);
  count_launches(2);
  return cudaGetLastError();
}

}  // namespace lshmoe
