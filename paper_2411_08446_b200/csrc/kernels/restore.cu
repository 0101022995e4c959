// a9: residual-based error compensation (Eq. 4-5; Alg. 1 L17-19,
// P:L536-538) summed over the k gated experts as in Eq. 2:
//     y_t = sum_s g_ts * (E(c~)[b_ts] + (x_t - c~[b_ts]))
// The residual x - c~ is never materialised: it is recomputed here from x and the transmitted
// centroid (reading R11), saving a write + read of n*k*d elements.  Default kernel (k <= 4, rows
// <= 2 KB): restore_stage_kernel, each token's x row and its c~ / E(c~) rows staged in shared memory
// by cp.async.bulk into per-warp mbarrier rings; the two-row warp kernel and the flat thread-per-
// 16-byte-chunk kernel cover the rest.  All variants evaluate the same expression in the same order
// (bit-identical outputs).  Also: the baseline un-permute and the world == 1 local exchange.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "../abi/lshmoe_internal.h"
#include "common.cuh"
#include "sm100.cuh"

namespace lshmoe {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) restore_kernel(const T* x /* y may alias x */, const T* __restrict__ ct,
                                                      const T* __restrict__ ret, int64_t n, int d,
                                                      const int32_t* __restrict__ bucket, int k,
                                                      const float* __restrict__ g, T* y) {
  constexpr int VN = Vec<T>::N;
  const int cpr = d / VN;
  const int64_t total = n * cpr;
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: the combined rows are complete
  asm volatile("griddepcontrol.launch_dependents;" :::);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / cpr;
    const int ch = static_cast<int>(i - t * cpr);
    float xv[VN], acc[VN];
    Vec<T>::load(x + t * d + ch * VN, xv);
    for (int s = 0; s < k; ++s) {
      const int64_t b = bucket[t * k + s];
      float cv[VN], rv[VN];
      Vec<T>::load(ct + b * d + ch * VN, cv);
      Vec<T>::load(ret + b * d + ch * VN, rv);
      const float gw = g ? g[t * k + s] : 1.0f;
#pragma unroll
      for (int v = 0; v < VN; ++v) {
        float term = rv[v] + (xv[v] - cv[v]);       // E(c~) + Delta  (Eq. 5)
        if (g) term = gw * term;
        acc[v] = (s == 0) ? term : acc[v] + term;   // Eq. 2 sum over the k experts
      }
    }
    Vec<T>::store(y + t * d + ch * VN, acc);
  }
}

// Warp per token row: lanes over the row's 16-byte chunks, the row's k bucket ids loaded once, and
// the next row's bucket id and x chunks fetched before the current row's c~ / E(c~) gathers are
// combined, so the dependent bucket -> gather chain of the next row overlaps this row's.  Measured
// (C2, graph-replayed, clean cold L2): 14.3 us against 18.4 us for the flat thread-per-chunk kernel;
// at d = 1024 (C3, C4) the flat kernel stays ahead.  Superseded for k = 1 rows of <= 96 chunks by
// restore_row2_kernel (below); LSHMOE_RESTORE_VAR: 0 forces the flat kernel, 2 / 4 this kernel
// with 2 / 4 CTAs per SM, 12 / 14 the two-row kernel.
template <typename T, int CPL>
__global__ void __launch_bounds__(256) restore_row_kernel(const T* x, const T* __restrict__ ct,
                                                          const T* __restrict__ ret, int64_t n, int d, int cpr,
                                                          const int32_t* __restrict__ bucket, int k,
                                                          const float* __restrict__ g, T* y) {
  constexpr int VN = Vec<T>::N;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x) >> 5;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * 8;
  uint4 xr[CPL];
  int32_t bn = 0;
  auto fetch = [&](int64_t t) {
    bn = __ldg(bucket + t * k);
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c = lane + 32 * j;
      if (c < cpr) xr[j] = __ldg(reinterpret_cast<const uint4*>(x + t * d) + c);
    }
  };
  if (w0 < n) fetch(w0);
  for (int64_t t = w0; t < n; t += nw) {
    float acc[CPL][VN];
    const int32_t b0 = bn;
    float xv[CPL][VN];
#pragma unroll
    for (int j = 0; j < CPL; ++j) Vec<T>::load(&xr[j], xv[j]);
    if (t + nw < n) fetch(t + nw);
    for (int s = 0; s < k; ++s) {
      const int64_t b = s == 0 ? b0 : __ldg(bucket + t * k + s);
      const float gw = g ? g[t * k + s] : 1.0f;
      uint4 cr[CPL], rr[CPL];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int c = lane + 32 * j;
        if (c < cpr) {
          cr[j] = __ldg(reinterpret_cast<const uint4*>(ct + b * d) + c);
          rr[j] = __ldg(reinterpret_cast<const uint4*>(ret + b * d) + c);
        }
      }
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        float cv[VN], rv[VN];
        Vec<T>::load(&cr[j], cv);
        Vec<T>::load(&rr[j], rv);
#pragma unroll
        for (int v = 0; v < VN; ++v) {
          float term = rv[v] + (xv[j][v] - cv[v]);
          if (g) term = gw * term;
          acc[j][v] = (s == 0) ? term : acc[j][v] + term;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c = lane + 32 * j;
      if (c < cpr) Vec<T>::store(y + t * d + c * VN, acc[j]);
    }
  }
}

// k = 1, two consecutive token rows per warp iteration: the pair's c~ / E(c~) gathers (6 KB per
// warp) are in flight together with the next pair's x rows and bucket ids (3 KB), twice the bytes
// in flight of restore_row_kernel per warp.
template <typename T, int CPL>
__global__ void __launch_bounds__(256) restore_row2_kernel(const T* x, const T* __restrict__ ct,
                                                           const T* __restrict__ ret, int64_t n, int d, int cpr,
                                                           const int32_t* __restrict__ bucket,
                                                           const float* __restrict__ g, T* y) {
  constexpr int VN = Vec<T>::N;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x) >> 5;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * 8;
  uint4 xr[2][CPL];
  int32_t bn[2] = {0, 0};
  auto fetch = [&](int64_t t) {               // rows t, t + 1
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = t + h;
      if (r < n) {
        bn[h] = __ldg(bucket + r);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int c = lane + 32 * j;
          if (c < cpr) xr[h][j] = __ldg(reinterpret_cast<const uint4*>(x + r * d) + c);
        }
      }
    }
  };
  if (2 * w0 < n) fetch(2 * w0);
  for (int64_t t = 2 * w0; t < n; t += 2 * nw) {
    uint4 xc[2][CPL];
    int32_t b[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      b[h] = bn[h];
#pragma unroll
      for (int j = 0; j < CPL; ++j) xc[h][j] = xr[h][j];
    }
    uint4 cr[2][CPL], rr[2][CPL];
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (t + h < n)
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          const int c = lane + 32 * j;
          if (c < cpr) {
            cr[h][j] = __ldg(reinterpret_cast<const uint4*>(ct + static_cast<int64_t>(b[h]) * d) + c);
            rr[h][j] = __ldg(reinterpret_cast<const uint4*>(ret + static_cast<int64_t>(b[h]) * d) + c);
          }
        }
    if (t + 2 * nw < n) fetch(t + 2 * nw);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (t + h >= n) break;
      const float gw = g ? g[t + h] : 1.0f;
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int c = lane + 32 * j;
        if (c >= cpr) continue;
        float xv[VN], cv[VN], rv[VN], acc[VN];
        Vec<T>::load(&xc[h][j], xv);
        Vec<T>::load(&cr[h][j], cv);
        Vec<T>::load(&rr[h][j], rv);
#pragma unroll
        for (int v = 0; v < VN; ++v) {
          const float term = rv[v] + (xv[v] - cv[v]);
          acc[v] = g ? gw * term : term;
        }
        Vec<T>::store(y + (t + h) * d + c * VN, acc);
      }
    }
  }
}

// Rows staged in shared memory by the bulk-copy engine (k <= 4): 16 warps per CTA (one CTA per SM),
// each warp owns a ring of `slots` slots, a slot = one token's x row followed by the c~ and E(c~)
// rows of its k copies, filled by one lane with 1 + 2k cp.async.bulk copies completing on the
// slot's mbarrier.  The x copy is issued at once, the gathers as soon as the token's bucket ids are
// known (the ids of a warp's next 32 / k tokens are loaded together, one batch ahead).  At d = 768
// bf16, k = 1, three tokens per warp (13.5 KB) are in flight without holding registers, against two
// rows in registers for restore_row2_kernel.  The arithmetic is restore_kernel's, term by term in
// slot order (same bits as every other restore kernel).
#ifndef LSHMOE_RSTAGE_WARPS
#define LSHMOE_RSTAGE_WARPS 16   // experiment knob (compile-time): warps per CTA of the staged restore
#endif
constexpr int kStageWarps = LSHMOE_RSTAGE_WARPS;
constexpr int kStageSmem = 216 * 1024;
constexpr int kStageMaxK = 4;

template <typename T, int KK>   // KK = 1: k == 1 at compile time; KK = 0: runtime k <= kStageMaxK
__global__ void __launch_bounds__(kStageWarps * 32, 1) restore_stage_kernel(const T* x, const T* __restrict__ ct,
                                                                            const T* __restrict__ ret, int64_t n,
                                                                            int d, int cpr, int k_arg, int slots, int pf,
                                                                            int prex,
                                                                            const int32_t* __restrict__ bucket,
                                                                            const float* __restrict__ g, T* y) {
  using namespace sm100;
  constexpr int VN = Vec<T>::N;
  constexpr int kMaxSlots = 8;
  constexpr int kKMax = KK ? KK : kStageMaxK;
  const int k = KK ? KK : k_arg;
  __shared__ __align__(8) uint64_t s_bar[kStageWarps][kMaxSlots];
  extern __shared__ __align__(128) uint8_t s_ring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t rb = static_cast<uint32_t>(cpr) * 16u;     // row bytes
  const uint32_t sb = (1u + 2u * k) * rb;                   // slot bytes
  const int tb = 32 / k;                                     // tokens per id batch
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kStageWarps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kStageWarps + warp;
  const int64_t cnt = gw < n ? (n - 1 - gw) / nw + 1 : 0;    // tokens t = gw + i * nw of this warp
  uint8_t* ring = s_ring + static_cast<size_t>(warp) * slots * sb;
  uint64_t* bar = s_bar[warp];
  if (lane < slots) mbar_init(&bar[lane], 1);
  fence_mbarrier_init();
  __syncwarp();
  // x is an input of the step: warm L2 with the x rows of this warp's first `slots` tokens while the
  // predecessor (the FFN's second GEMM, whose last wave leaves SMs free) finishes.  A prefetch is only
  // a hint, so it is safe even if a predecessor were still writing x.
  if (prex && lane == 0)
    for (int s2 = 0; s2 < slots && s2 < cnt; ++s2)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (gw + s2 * nw) * d), "r"(rb) : "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");   // PDL: the combined rows are complete
  asm volatile("griddepcontrol.launch_dependents;" :::);
  auto bulk = [&](uint8_t* dst, const void* src, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(rb), "r"(smem_u32(b))
                 : "memory");
  };
  // bucket ids of tokens [i0, i0 + tb): lane j < tb * k holds copy j % k of token i0 + j / k
  auto load_ids = [&](int64_t i0) {
    const int64_t i = i0 + lane / k;
    return lane < tb * k && i < cnt ? __ldg(bucket + (gw + i * nw) * k + lane % k) : 0;
  };
  // lane 0 issues the c~ / E(c~) copies of the token at batch position bpos into `slot`
  auto gathers = [&](uint8_t* slot, uint64_t* sbar, int ids, int bpos) {
    for (int s2 = 0; s2 < k; ++s2) {
      const int64_t b = __shfl_sync(0xFFFFFFFFu, ids, bpos * k + s2);
      if (lane == 0) {
        bulk(slot + (1 + 2 * s2) * rb, ct + b * d, sbar);
        bulk(slot + (2 + 2 * s2) * rb, ret + b * d, sbar);
      }
    }
  };
  // optional L2 prefetch of the x rows `pf` tokens beyond the ring (more DRAM reads in flight
  // without shared memory)
  auto prefetch_x = [&](int64_t i) {
    if (pf && lane == 0 && i < cnt)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (gw + i * nw) * d), "r"(rb) : "memory");
  };
  int ids = load_ids(0), ids_next = 0;
  if (lane == 0)                             // x rows of the first `slots` tokens: no dependency
    for (int s2 = 0; s2 < slots && s2 < cnt; ++s2) {
      mbar_arrive_expect_tx(&bar[s2], sb);
      bulk(ring + s2 * sb, x + (gw + s2 * nw) * d, &bar[s2]);
    }
  for (int u = 0; u < pf; ++u) prefetch_x(slots + u);
  if (cnt > tb) ids_next = load_ids(tb);
  for (int s2 = 0; s2 < slots && s2 < cnt; ++s2) gathers(ring + s2 * sb, &bar[s2], ids, s2);   // slots <= tb
  // counters instead of 64-bit divisions: slot s and its phase for token i; batch position of the
  // refill token i + slots
  int s = 0, nbp = slots == tb ? 0 : slots;
  uint32_t ph = 0;
  for (int64_t i = 0; i < cnt; ++i) {
    const int64_t t = gw + i * nw;
    float gwv[kKMax];
#pragma unroll
    for (int s2 = 0; s2 < kKMax; ++s2) gwv[s2] = g && s2 < k ? __ldg(g + t * k + s2) : 1.0f;
    mbar_wait(&bar[s], ph);
    const uint8_t* sx = ring + s * sb;
    for (int c = lane; c < cpr; c += 32) {
      float xv[VN], acc[VN];
      Vec<T>::load(sx + 16 * c, xv);
#pragma unroll
      for (int s2 = 0; s2 < kKMax; ++s2) {
        if (s2 >= k) break;
        float cv[VN], rv[VN];
        Vec<T>::load(sx + (1 + 2 * s2) * rb + 16 * c, cv);
        Vec<T>::load(sx + (2 + 2 * s2) * rb + 16 * c, rv);
#pragma unroll
        for (int v = 0; v < VN; ++v) {
          float term = rv[v] + (xv[v] - cv[v]);       // E(c~) + Delta  (Eq. 5)
          if (g) term = gwv[s2] * term;
          acc[v] = (s2 == 0) ? term : acc[v] + term;   // Eq. 2 sum over the k experts
        }
      }
      Vec<T>::store(y + t * d + c * VN, acc);
    }
    __syncwarp();                            // every lane has read the slot: refill it
    const int64_t nx = i + slots;
    if (nx < cnt) {
      if (nbp == 0) {                        // next batch of ids (loaded one batch ahead)
        ids = ids_next;
        ids_next = nx + tb < cnt ? load_ids(nx + tb) : 0;
      }
      if (lane == 0) {
        mbar_arrive_expect_tx(&bar[s], sb);
        bulk(ring + s * sb, x + (gw + nx * nw) * d, &bar[s]);
      }
      prefetch_x(nx + pf);
      gathers(ring + s * sb, &bar[s], ids, nbp);
    }
    if (++nbp == tb) nbp = 0;
    if (++s == slots) {
      s = 0;
      ph ^= 1u;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) unpermute_kernel(const T* __restrict__ ret, int64_t n, int d,
                                                        const int32_t* __restrict__ slot, int k,
                                                        const float* __restrict__ g, T* __restrict__ y) {
  constexpr int VN = Vec<T>::N;
  const int cpr = d / VN;
  const int64_t total = n * cpr;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / cpr;
    const int ch = static_cast<int>(i - t * cpr);
    float acc[VN];
    for (int s = 0; s < k; ++s) {
      const int64_t b = slot[t * k + s];
      float rv[VN];
      Vec<T>::load(ret + b * d + ch * VN, rv);
      const float gw = g ? g[t * k + s] : 1.0f;
#pragma unroll
      for (int v = 0; v < VN; ++v) {
        const float term = g ? gw * rv[v] : rv[v];
        acc[v] = (s == 0) ? term : acc[v] + term;
      }
    }
    Vec<T>::store(y + t * d + ch * VN, acc);
  }
}

// ---- NEXT-1 grad_restore (reading R27), two kernels:
//   grad_x_kernel     one thread per 16-byte chunk of dX (flat, like restore_kernel):
//                     dX_t = sum_s [ g_ts dY_t + (H_b - G_b) / n_b ],  n_b from the forward's row_start
//   grad_gate_kernel  (only when dgate is requested) one warp per token row: dg_ts = dY_t . (o_b + x_t - c~_b),
//                     lane partials over the row's chunks (all loads of a 32-chunk block issued
//                     first), then a warp reduction — a fixed order, so the result is deterministic.
template <typename T>
__global__ void __launch_bounds__(256) grad_x_kernel(const T* __restrict__ dy, const T* __restrict__ G,
                                                     const T* __restrict__ H, int64_t n, int d,
                                                     const int32_t* __restrict__ bucket,
                                                     const int32_t* __restrict__ row_start, int k,
                                                     const float* __restrict__ g, T* __restrict__ dx) {
  constexpr int VN = Vec<T>::N;
  const int cpr = d / VN;
  const int64_t total = n * cpr;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / cpr;
    const int ch = static_cast<int>(i - t * cpr);
    float dyv[VN], acc[VN];
    Vec<T>::load(dy + t * d + ch * VN, dyv);
    float gsum = 0.0f;
#pragma unroll
    for (int v = 0; v < VN; ++v) acc[v] = 0.0f;
    for (int s = 0; s < k; ++s) {
      const int64_t b = __ldg(bucket + t * k + s);
      const float inv_n = 1.0f / static_cast<float>(__ldg(row_start + b + 1) - __ldg(row_start + b));
      gsum += g ? __ldg(g + t * k + s) : 1.0f;
      float gv[VN], hv[VN];
      Vec<T>::load(G + b * d + ch * VN, gv);
      Vec<T>::load(H + b * d + ch * VN, hv);
#pragma unroll
      for (int v = 0; v < VN; ++v) acc[v] += (hv[v] - gv[v]) * inv_n;
    }
#pragma unroll
    for (int v = 0; v < VN; ++v) acc[v] += gsum * dyv[v];     // sum_s g_ts dY_t
    Vec<T>::store(dx + t * d + ch * VN, acc);
  }
}

constexpr int kGC = 4;   // 16-byte chunks per lane per column block (grad_gate_kernel)

template <typename T>
__global__ void __launch_bounds__(256) grad_gate_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                        const T* __restrict__ ct, const T* __restrict__ ret,
                                                        int64_t n, int d, const int32_t* __restrict__ bucket, int k,
                                                        float* __restrict__ dg) {
  constexpr int VN = Vec<T>::N;
  const int cpr = d / VN;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x / 32) + threadIdx.x / 32; t < n; t += warps) {
    for (int s = 0; s < k; ++s) {
      const int64_t b = __ldg(bucket + t * k + s);
      float dot = 0.0f;
      for (int c0 = 0; c0 < cpr; c0 += 32 * kGC) {
        uint4 dr[kGC], xr[kGC], cr[kGC], rr[kGC];
#pragma unroll
        for (int j = 0; j < kGC; ++j) {
          const int ch = c0 + j * 32 + lane;
          if (ch < cpr) {
            dr[j] = __ldg(reinterpret_cast<const uint4*>(dy + t * d) + ch);
            xr[j] = __ldg(reinterpret_cast<const uint4*>(x + t * d) + ch);
            cr[j] = __ldg(reinterpret_cast<const uint4*>(ct + b * d) + ch);
            rr[j] = __ldg(reinterpret_cast<const uint4*>(ret + b * d) + ch);
          }
        }
#pragma unroll
        for (int j = 0; j < kGC; ++j) {
          const int ch = c0 + j * 32 + lane;
          if (ch >= cpr) continue;
          float dv[VN], xv[VN], cv[VN], rv[VN];
          Vec<T>::load(&dr[j], dv);
          Vec<T>::load(&xr[j], xv);
          Vec<T>::load(&cr[j], cv);
          Vec<T>::load(&rr[j], rv);
#pragma unroll
          for (int v = 0; v < VN; ++v) dot = fmaf(dv[v], rv[v] + (xv[v] - cv[v]), dot);
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xFFFFFFFFu, dot, off);
      if (lane == 0) dg[t * k + s] = dot;
    }
  }
}

// world == 1 "all-to-all": copy the sum(counts) valid rows (device count) and the counts.
__global__ void __launch_bounds__(256) local_exchange_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                             int64_t capacity_rows, int row_bytes,
                                                             const int32_t* __restrict__ counts, int E,
                                                             int32_t* __restrict__ counts_out) {
  __shared__ int64_t rows_s;
  if (threadIdx.x == 0) {
    int64_t r = 0;
    for (int e = 0; e < E; ++e) r += counts[e];
    rows_s = r < capacity_rows ? r : capacity_rows;
  }
  if (counts_out && blockIdx.x == 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x) counts_out[e] = counts[e];
  __syncthreads();
  if (!dst) return;
  const int64_t total = rows_s * (row_bytes / 16);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int grid_for(int64_t work) {
  const int64_t g = (work + 255) / 256;
  const int64_t cap = 16 * static_cast<int64_t>(device_sm_count());
  return static_cast<int>(std::max<int64_t>(1, std::min(g, cap)));
}

}  // namespace

int restore_variant() {   // -1: the measured default (see restore_row_kernel)
  const char* v = getenv("LSHMOE_RESTORE_VAR");
  return v ? atoi(v) : -1;
}

int restore_prex() {   // LSHMOE_RESTORE_PREX: L2 warm-up of the first x rows before the dependency wait
  const char* v = getenv("LSHMOE_RESTORE_PREX");
  return v ? (atoi(v) != 0) : 0;   // measured: step C2 neutral, C5 -2 us; T_dc +1.4 us: off
}

int restore_prefetch() {   // LSHMOE_RESTORE_PF: x rows prefetched to L2 beyond the staged ring
  const char* v = getenv("LSHMOE_RESTORE_PF");
  return v ? std::max(0, std::min(8, atoi(v))) : 0;
}

template <typename T>
int launch_restore_pdl(const void* x, const void* ct, const void* ret, int64_t n, int d, const int32_t* bucket, int k,
                       const float* g, void* y, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  const int cpr = d / Vec<T>::N;
  const int64_t total = n * cpr;
  cfg.gridDim = dim3(grid_for(total));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  static bool carve = [] {   // full shared-memory carveout like the step's other kernels (no re-partition)
    const char* e = getenv("LSHMOE_CARVEOUT");
    if (e && e[0] == '0') return false;
    cudaFuncSetAttribute(restore_kernel<T>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(restore_row_kernel<T, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(restore_row_kernel<T, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(restore_row_kernel<T, 3>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(restore_row_kernel<T, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    return true;
  }();
  (void)carve;
  // k = 1 rows of <= 128 chunks: two rows per warp iteration, 2 CTAs per SM (graph-timed over cycled
  // token copies, scripts/restore_ab2.py: C2 13.45 vs 14.50 us for one row per warp, C5 18.9 vs 21.9,
  // C4 (d = 1024) 64.1 vs 75.4 us for the flat kernel); k > 1 keeps the flat kernel (C3 50.1 us vs
  // 59-69 for the row kernels)
  int var = restore_variant();
  const bool stage_ok = k <= kStageMaxK && cpr <= 128 && kStageSmem / (kStageWarps * (1 + 2 * k) * cpr * 16) >= 1;
  if (var < 0) var = stage_ok ? 20 : (k == 1 && cpr >= 32 && cpr <= 128) ? 12 : 0;
  if (var == 20 && stage_ok) {                  // staged: slots per warp from the smem budget
    static bool staged_cfg = [] {
      cudaFuncSetAttribute(restore_stage_kernel<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageSmem);
      cudaFuncSetAttribute(restore_stage_kernel<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageSmem);
      return true;
    }();
    (void)staged_cfg;
    const int rb = cpr * 16;
    const int slots = std::min(8, kStageSmem / (kStageWarps * (1 + 2 * k) * rb));
    const int64_t warps_needed = (n + 1) / 2;
    cfg.gridDim = dim3(static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>(device_sm_count(), (warps_needed + kStageWarps - 1) / kStageWarps))));
    cfg.blockDim = dim3(kStageWarps * 32);
    cfg.dynamicSmemBytes = static_cast<size_t>(kStageWarps) * slots * (1 + 2 * k) * rb;
    return cudaLaunchKernelEx(&cfg, k == 1 ? restore_stage_kernel<T, 1> : restore_stage_kernel<T, 0>,
                              static_cast<const T*>(x), static_cast<const T*>(ct),
                              static_cast<const T*>(ret), n, d, cpr, k, slots, restore_prefetch(), restore_prex(),
                              bucket, g, static_cast<T*>(y));
  }
  if (var >= 12 && k == 1 && cpr >= 32 && cpr <= 128) {   // 10 + CTAs per SM, two rows per warp
    const int64_t pairs = (n + 1) / 2;
    const int warps = static_cast<int>(std::min<int64_t>(pairs, int64_t(var - 10) * 8 * device_sm_count()));
    cfg.gridDim = dim3(std::max(1, (warps + 7) / 8));
    const int cpl = (cpr + 31) / 32;
    const T* xp2 = static_cast<const T*>(x);
    const T* cp2 = static_cast<const T*>(ct);
    const T* rp2 = static_cast<const T*>(ret);
    T* yp2 = static_cast<T*>(y);
    if (cpl == 1) return cudaLaunchKernelEx(&cfg, restore_row2_kernel<T, 1>, xp2, cp2, rp2, n, d, cpr, bucket, g, yp2);
    if (cpl == 2) return cudaLaunchKernelEx(&cfg, restore_row2_kernel<T, 2>, xp2, cp2, rp2, n, d, cpr, bucket, g, yp2);
    if (cpl == 3) return cudaLaunchKernelEx(&cfg, restore_row2_kernel<T, 3>, xp2, cp2, rp2, n, d, cpr, bucket, g, yp2);
    return cudaLaunchKernelEx(&cfg, restore_row2_kernel<T, 4>, xp2, cp2, rp2, n, d, cpr, bucket, g, yp2);
  }
  const T* xp = static_cast<const T*>(x);
  const T* cp = static_cast<const T*>(ct);
  const T* rp = static_cast<const T*>(ret);
  T* yp = static_cast<T*>(y);
  if (var >= 2 && cpr >= 32 && cpr <= 128) {
    const int warps = static_cast<int>(std::min<int64_t>(n, int64_t(var) * 8 * device_sm_count()));
    cfg.gridDim = dim3(std::max(1, (warps + 7) / 8));
    const int cpl = (cpr + 31) / 32;
    if (cpl == 1) return cudaLaunchKernelEx(&cfg, restore_row_kernel<T, 1>, xp, cp, rp, n, d, cpr, bucket, k, g, yp);
    if (cpl == 2) return cudaLaunchKernelEx(&cfg, restore_row_kernel<T, 2>, xp, cp, rp, n, d, cpr, bucket, k, g, yp);
    if (cpl == 3) return cudaLaunchKernelEx(&cfg, restore_row_kernel<T, 3>, xp, cp, rp, n, d, cpr, bucket, k, g, yp);
    return cudaLaunchKernelEx(&cfg, restore_row_kernel<T, 4>, xp, cp, rp, n, d, cpr, bucket, k, g, yp);
  }
  return cudaLaunchKernelEx(&cfg, restore_kernel<T>, xp, cp, rp, n, d, bucket, k, g, yp);
}

int launch_restore(const void* x, const void* ct, const void* ret, lshmoe_dtype dtype, int64_t n, int d,
                   const int32_t* bucket, int k, const float* g, void* y, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int err = dtype == LSHMOE_BF16 ? launch_restore_pdl<__nv_bfloat16>(x, ct, ret, n, d, bucket, k, g, y, st)
                                       : launch_restore_pdl<float>(x, ct, ret, n, d, bucket, k, g, y, st);
  count_launches(1);
  return err ? err : cudaGetLastError();
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* env = getenv("LSHMOE_PDL");
    return !(env && env[0] == '0');
  }();
  return on;
}

int launch_grad_restore(const void* dy, const void* x, const void* ct, const void* ret, const void* G, const void* H,
                        lshmoe_dtype dtype, int64_t n, int d, const int32_t* bucket, const int32_t* row_start, int k,
                        const float* g, void* dx, float* dg, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t items = n * (d / (dtype == LSHMOE_BF16 ? 8 : 4));
  const int rgrid = static_cast<int>(std::max<int64_t>(1, (n + 7) / 8));   // one warp per row
  if (dtype == LSHMOE_BF16) {
    using T = __nv_bfloat16;
    grad_x_kernel<T><<<grid_for(items), 256, 0, st>>>(static_cast<const T*>(dy), static_cast<const T*>(G),
                                                       static_cast<const T*>(H), n, d, bucket, row_start, k, g,
                                                       static_cast<T*>(dx));
    if (dg)
      grad_gate_kernel<T><<<rgrid, 256, 0, st>>>(static_cast<const T*>(dy), static_cast<const T*>(x),
                                                 static_cast<const T*>(ct), static_cast<const T*>(ret), n, d, bucket,
                                                 k, dg);
  } else {
    grad_x_kernel<float><<<grid_for(items), 256, 0, st>>>(static_cast<const float*>(dy), static_cast<const float*>(G),
                                                           static_cast<const float*>(H), n, d, bucket, row_start, k,
                                                           g, static_cast<float*>(dx));
    if (dg)
      grad_gate_kernel<float><<<rgrid, 256, 0, st>>>(static_cast<const float*>(dy), static_cast<const float*>(x),
                                                     static_cast<const float*>(ct), static_cast<const float*>(ret), n,
                                                     d, bucket, k, dg);
  }
  count_launches(dg ? 2 : 1);
  return cudaGetLastError();
}

int launch_unpermute(const void* ret, lshmoe_dtype dtype, int64_t n, int d, const int32_t* slot, int k, const float* g,
                     void* y, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == LSHMOE_BF16) {
    using T = __nv_bfloat16;
    unpermute_kernel<T><<<grid_for(n * (d / 8)), 256, 0, st>>>(static_cast<const T*>(ret), n, d, slot, k, g,
                                                               static_cast<T*>(y));
  } else {
    unpermute_kernel<float><<<grid_for(n * (d / 4)), 256, 0, st>>>(static_cast<const float*>(ret), n, d, slot, k, g,
                                                                   static_cast<float*>(y));
  }
  count_launches(1);
  return cudaGetLastError();
}

int launch_local_exchange(const void* src, void* dst, int64_t capacity_rows, int row_bytes, const int32_t* counts,
                          int E, int32_t* counts_out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!dst && !counts_out) return 0;                  // aliased exchange at world 1: nothing to move
  const int grid = dst ? 8 * device_sm_count() : 1;
  local_exchange_kernel<<<grid, 256, 0, st>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), capacity_rows,
                                              row_bytes, counts, E, counts_out);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lshmoe
