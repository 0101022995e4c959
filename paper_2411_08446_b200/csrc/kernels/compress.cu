// a3-a5: group the routed copies by expert, bucket them by their composite LSH key, and reduce
// each bucket to its centroid (Alg. 1 L3, L5-L8: P:L520; §2.3).
//
// Pipeline (all device-side, no host synchronisation):
//   1. insert  : global open-addressing hash table keyed by (expert, q-tuple of codes); the value
//                converges (atomicMin) to the smallest copy id c = t*k+s with that key = the first
//                appearance of the bucket in its expert group (reading R7).
//   2. lookup  : rep[c] = table value; a copy is a "first" iff rep[c] == c.
//   3. radix   : one stable LSD pass over key = expert (firsts) / E (others) puts the firsts in
//                (expert, first position) order: that position IS the global centroid row
//                (expert-major, first-appearance local ids); the pass's histogram scan gives
//                m_e and m.
//   4. radix   : stable LSD sort of all copies by row = rowid[rep[c]] (2 passes of 8 bits for
//                n*k <= 65536) -> perm (ascending copy id within a row, reading R8); bucket[c].
//   5. centroid: fixed 32-entry chunks of perm, one warp each, fp32 sums in perm order with
//                128-bit loads; rows spanning chunks leave partials that a fix-up warp adds in
//                chunk order (deterministic), then one IEEE division by the count (reading R10)
//                and RNE to the wire dtype.
// Stable ranking inside a radix tile uses __match_any_sync + per-warp digit counters in shared
// memory (rounds processed in order => stability), warp prefixes combined per digit.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../abi/lshmoe_internal.h"
#include "common.cuh"

namespace lshmoe {
namespace {

constexpr int kRadix = 256;
constexpr int kRT = 256;                 // threads per radix CTA
constexpr int kRItems = 4;               // items per thread
constexpr int kRTile = kRT * kRItems;    // 1024
constexpr int kRWarps = kRT / 32;
constexpr int kChunk = 32;               // perm entries per centroid work item
constexpr int kMaxE = 255;               // single-pass expert sort (E + sentinel <= 256 digits)

// Device error word (read by lshmoe_check_device_error).  Bit 0: expert id outside [0, E)
// (S:L312).  Only this translation unit validates expert ids.
__device__ int g_device_error = 0;

__device__ __forceinline__ void raise_device_error(int bit) { atomicOr(&g_device_error, bit); }

__device__ __forceinline__ int load_expert(const int32_t* experts, int c, int E) {
  int e = experts[c];
  if (static_cast<unsigned>(e) >= static_cast<unsigned>(E)) {
    raise_device_error(1);
    e = 0;                                // keep every index in bounds; the result is flagged
  }
  return e;
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ uint32_t key_hash(int e, const int16_t* c, int q) {
  uint32_t h = fmix32(static_cast<uint32_t>(e) + 0x9E3779B9u);
  for (int i = 0; i < q; ++i) h = fmix32(h ^ (static_cast<uint32_t>(static_cast<uint16_t>(c[i])) + (i << 16)));
  return h;
}

__device__ __forceinline__ bool codes_equal(const int16_t* a, const int16_t* b, int q) {
  for (int i = 0; i < q; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

__global__ void insert_kernel(const int16_t* __restrict__ codes, int q, const int32_t* __restrict__ experts, int k,
                              int E, int nk, int32_t* table, uint32_t mask) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nk; c += gridDim.x * blockDim.x) {
    const int e = load_expert(experts, c, E);
    const int16_t* mc = codes + static_cast<int64_t>(c / k) * q;
    uint32_t slot = key_hash(e, mc, q) & mask;
    while (true) {
      int cur = *reinterpret_cast<volatile int32_t*>(&table[slot]);
      if (cur < 0) {
        const int old = atomicCAS(&table[slot], -1, c);
        if (old < 0) break;              // claimed an empty slot
        cur = old;
      }
      // cur is some copy with this slot's key (the key of a slot never changes once claimed)
      int ec = experts[cur];
      if (static_cast<unsigned>(ec) >= static_cast<unsigned>(E)) ec = 0;
      if (ec == e && codes_equal(codes + static_cast<int64_t>(cur / k) * q, mc, q)) {
        if (c < cur) atomicMin(&table[slot], c);   // skip the atomic once a smaller id is in
        break;
      }
      slot = (slot + 1) & mask;
    }
  }
}

__global__ void lookup_kernel(const int16_t* __restrict__ codes, int q, const int32_t* __restrict__ experts, int k,
                              int E, int nk, const int32_t* __restrict__ table, uint32_t mask, int32_t* __restrict__ rep,
                              uint32_t* __restrict__ key_out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nk; c += gridDim.x * blockDim.x) {
    int e = experts[c];
    if (static_cast<unsigned>(e) >= static_cast<unsigned>(E)) e = 0;
    const int16_t* mc = codes + static_cast<int64_t>(c / k) * q;
    uint32_t slot = key_hash(e, mc, q) & mask;
    int r;
    while (true) {
      r = table[slot];
      int er = experts[r];
      if (static_cast<unsigned>(er) >= static_cast<unsigned>(E)) er = 0;
      if (er == e && codes_equal(codes + static_cast<int64_t>(r / k) * q, mc, q)) break;
      slot = (slot + 1) & mask;
    }
    rep[c] = r;
    key_out[c] = (r == c) ? static_cast<uint32_t>(e) : static_cast<uint32_t>(E);
  }
}

// ---- stable LSD radix pass ------------------------------------------------------------------
enum KeyMode { KEY_DIRECT = 0, KEY_ROW = 1, KEY_EXPERT = 2 };
enum OutMode { OUT_WRITE = 0, OUT_ROWID = 1, OUT_SLOT = 2 };

struct RadixIO {
  const uint32_t* keys_in;   // KEY_DIRECT
  const int32_t* vals_in;    // KEY_DIRECT (nullptr = identity)
  const int32_t* rep;        // KEY_ROW
  const int32_t* rowid;      // KEY_ROW
  const int32_t* experts;    // KEY_EXPERT: key = validated expert id of copy i
  int32_t* bucket;           // KEY_ROW: bucket[c] = row written by the downsweep
  uint32_t* keys_out;        // OUT_WRITE / OUT_SLOT
  int32_t* vals_out;         // OUT_WRITE / OUT_SLOT
  int32_t* rowid_out;        // OUT_ROWID: rowid[val] = dest for key < E
  int32_t* slot_out;         // OUT_SLOT: slot[val] = dest
  int E;
};

template <int KM>
__device__ __forceinline__ void radix_load(const RadixIO& io, int i, uint32_t& key, int32_t& val) {
  if (KM == KEY_DIRECT) {
    key = io.keys_in[i];
    val = io.vals_in ? io.vals_in[i] : i;
  } else if (KM == KEY_ROW) {
    val = i;
    key = static_cast<uint32_t>(io.rowid[io.rep[i]]);
  } else {
    val = i;
    key = static_cast<uint32_t>(load_expert(io.experts, i, io.E));
  }
}

template <int KM>
__global__ void __launch_bounds__(kRT) radix_upsweep(RadixIO io, int n, int shift, int32_t* __restrict__ hist, int nb) {
  __shared__ int cnt[kRadix];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int base = blockIdx.x * kRTile;
#pragma unroll
  for (int r = 0; r < kRItems; ++r) {
    const int i = base + r * kRT + threadIdx.x;
    if (i < n) {
      uint32_t key;
      int32_t val;
      radix_load<KM>(io, i, key, val);
      atomicAdd(&cnt[(key >> shift) & (kRadix - 1)], 1);
    }
  }
  __syncthreads();
  hist[threadIdx.x * nb + blockIdx.x] = cnt[threadIdx.x];
}

// One CTA: hist[digit][block] -> global exclusive offsets (digit-major, block-minor).
// Optionally (expert pass) writes m_e = count of digit e < E and m.
__global__ void __launch_bounds__(kRadix) radix_scan(int32_t* hist, int nb, int32_t* expert_rows, int32_t* num_rows,
                                                     int E) {
  __shared__ int tot[kRadix];
  const int dgt = threadIdx.x;
  int run = 0;
  for (int b = 0; b < nb; ++b) {
    const int v = hist[dgt * nb + b];
    hist[dgt * nb + b] = run;
    run += v;
  }
  tot[dgt] = run;
  __syncthreads();
  // exclusive scan over digits (Hillis-Steele on 256 entries)
  int x = run;
  for (int off = 1; off < kRadix; off <<= 1) {
    __syncthreads();
    const int y = dgt >= off ? tot[dgt - off] : 0;
    __syncthreads();
    x += y;
    tot[dgt] = x;
  }
  const int excl = x - run;
  for (int b = 0; b < nb; ++b) hist[dgt * nb + b] += excl;
  if (expert_rows) {
    if (dgt < E) expert_rows[dgt] = run;
    if (dgt == E) *num_rows = excl;         // firsts of all experts precede the sentinel digit
  }
}

template <int KM, int OM>
__global__ void __launch_bounds__(kRT) radix_downsweep(RadixIO io, int n, int shift, const int32_t* __restrict__ hist,
                                                      int nb) {
  __shared__ int wcnt[kRWarps][kRadix];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < kRWarps * kRadix; i += kRT) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  uint32_t key[kRItems];
  int32_t val[kRItems];
  int dg[kRItems], loc[kRItems];
  const int base = blockIdx.x * kRTile + warp * (kRItems * 32);
#pragma unroll
  for (int r = 0; r < kRItems; ++r) {
    const int i = base + r * 32 + lane;
    const bool ok = i < n;
    if (ok) radix_load<KM>(io, i, key[r], val[r]);
    dg[r] = ok ? static_cast<int>((key[r] >> shift) & (kRadix - 1)) : kRadix;   // kRadix = padding group
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, dg[r]);
    const int leader = __ffs(peers) - 1;
    int b = 0;
    if (ok) b = wcnt[warp][dg[r]];
    __syncwarp();
    if (ok && lane == leader) wcnt[warp][dg[r]] = b + __popc(peers);
    __syncwarp();
    loc[r] = b + __popc(peers & lt);
  }
  __syncthreads();
  {
    const int dgt = threadIdx.x;   // kRT == kRadix
    int run = 0;
    for (int w = 0; w < kRWarps; ++w) {
      const int v = wcnt[w][dgt];
      wcnt[w][dgt] = run;
      run += v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRItems; ++r) {
    if (dg[r] == kRadix) continue;
    const int dest = hist[dg[r] * nb + blockIdx.x] + wcnt[warp][dg[r]] + loc[r];
    if (KM == KEY_ROW) io.bucket[val[r]] = static_cast<int32_t>(key[r]);
    if (OM == OUT_ROWID) {
      if (key[r] < static_cast<uint32_t>(io.E)) io.rowid_out[val[r]] = dest;
    } else {
      io.keys_out[dest] = key[r];
      io.vals_out[dest] = val[r];
      if (OM == OUT_SLOT) io.slot_out[val[r]] = dest;
    }
  }
}

template <int KM, int OM>
void radix_pass(const RadixIO& io, int n, int shift, int32_t* hist, int32_t* expert_rows, int32_t* num_rows, int E,
                cudaStream_t st) {
  const int nb = (n + kRTile - 1) / kRTile;
  radix_upsweep<KM><<<nb, kRT, 0, st>>>(io, n, shift, hist, nb);
  radix_scan<<<1, kRadix, 0, st>>>(hist, nb, expert_rows, num_rows, E);
  radix_downsweep<KM, OM><<<nb, kRT, 0, st>>>(io, n, shift, hist, nb);
  count_launches(3);
}

// ---- centroid ---------------------------------------------------------------------------------
template <typename T>
struct CentroidArgs {
  const T* x;
  int d, k, nk;
  const int32_t* perm;
  const uint32_t* rows;     // sorted row of each perm entry
  int32_t* row_start;
  T* cent;
  float* cent32;
  float* partial;           // [n_items][2][d]
  int n_items;
};

constexpr int kMaxJ = 4;     // 16-byte chunks per lane per column block (2 KB per row block)

template <typename T>
__device__ __forceinline__ void write_centroid(const CentroidArgs<T>& a, int row, int cb0, int nch, const float (&acc)[kMaxJ][Vec<T>::N],
                                               float cnt) {
  constexpr int VN = Vec<T>::N;
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int j = 0; j < kMaxJ; ++j) {
    const int ch = cb0 + lane + 32 * j;
    if (ch >= nch) break;
    float v[VN];
#pragma unroll
    for (int e = 0; e < VN; ++e) v[e] = __fdiv_rn(acc[j][e], cnt);
    Vec<T>::store(reinterpret_cast<uint8_t*>(a.cent + static_cast<int64_t>(row) * a.d) + 16 * ch, v);
    if (a.cent32) {
      float* dst = a.cent32 + static_cast<int64_t>(row) * a.d + ch * VN;
#pragma unroll
      for (int e = 0; e < VN; e += 4) *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) centroid_kernel(CentroidArgs<T> a) {
  constexpr int VN = Vec<T>::N;
  const int warp_g = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (warp_g >= a.n_items) return;
  const int p0 = warp_g * kChunk;
  const int p1 = min(p0 + kChunk, a.nk);
  const int cntp = p1 - p0;
  const int my_p = p0 + lane;
  const bool has = lane < cntp;
  const uint32_t my_row = has ? a.rows[my_p] : 0xFFFFFFFFu;
  const int my_c = has ? a.perm[my_p] : 0;
  const uint32_t prev_row = p0 > 0 ? a.rows[p0 - 1] : 0xFFFFFFFFu;
  const uint32_t next_row = p1 < a.nk ? a.rows[p1] : 0xFFFFFFFFu;
  const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, my_row, 1);
  const bool head = has && (lane == 0 ? my_row != prev_row : my_row != up);
  if (head) a.row_start[my_row] = my_p;                       // global row boundary
  if (has && my_p == a.nk - 1) a.row_start[my_row + 1] = a.nk; // row_start[m] = n*k
  const bool item_head = has && (lane == 0 || my_row != up);
  unsigned heads = __ballot_sync(0xFFFFFFFFu, item_head);
  const int nch = a.d * static_cast<int>(sizeof(T)) / 16;      // 16-byte chunks per row
  while (heads) {
    const int s = __ffs(heads) - 1;
    heads &= heads - 1;
    const int e = heads ? __ffs(heads) - 1 : cntp;
    const uint32_t row = __shfl_sync(0xFFFFFFFFu, my_row, s);
    const bool complete = (s > 0 || prev_row != row) && (e < cntp || next_row != row);
    for (int cb0 = 0; cb0 < nch; cb0 += 32 * kMaxJ) {
      float acc[kMaxJ][VN];
#pragma unroll
      for (int j = 0; j < kMaxJ; ++j)
#pragma unroll
        for (int v = 0; v < VN; ++v) acc[j][v] = 0.0f;
      int i = s;
      for (; i + 1 < e; i += 2) {                              // 2 member rows in flight
        const int t0 = __shfl_sync(0xFFFFFFFFu, my_c, i) / a.k;
        const int t1 = __shfl_sync(0xFFFFFFFFu, my_c, i + 1) / a.k;
        const uint8_t* r0 = reinterpret_cast<const uint8_t*>(a.x + static_cast<int64_t>(t0) * a.d);
        const uint8_t* r1 = reinterpret_cast<const uint8_t*>(a.x + static_cast<int64_t>(t1) * a.d);
        float v0[kMaxJ][VN], v1[kMaxJ][VN];
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
          const int ch = cb0 + lane + 32 * j;
          if (ch < nch) {
            Vec<T>::load(r0 + 16 * ch, v0[j]);
            Vec<T>::load(r1 + 16 * ch, v1[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
          const int ch = cb0 + lane + 32 * j;
          if (ch < nch) {
#pragma unroll
            for (int v = 0; v < VN; ++v) acc[j][v] = (acc[j][v] + v0[j][v]) + v1[j][v];
          }
        }
      }
      if (i < e) {
        const int t0 = __shfl_sync(0xFFFFFFFFu, my_c, i) / a.k;
        const uint8_t* r0 = reinterpret_cast<const uint8_t*>(a.x + static_cast<int64_t>(t0) * a.d);
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
          const int ch = cb0 + lane + 32 * j;
          if (ch < nch) {
            float v0[VN];
            Vec<T>::load(r0 + 16 * ch, v0);
#pragma unroll
            for (int v = 0; v < VN; ++v) acc[j][v] += v0[v];
          }
        }
      }
      if (complete) {
        write_centroid(a, static_cast<int>(row), cb0, nch, acc, static_cast<float>(e - s));
      } else {
        float* dst = a.partial + (static_cast<int64_t>(warp_g) * 2 + (s == 0 ? 0 : 1)) * a.d;
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
          const int ch = cb0 + lane + 32 * j;
          if (ch < nch)
#pragma unroll
            for (int v = 0; v < VN; v += 4)
              *reinterpret_cast<float4*>(dst + ch * VN + v) = make_float4(acc[j][v], acc[j][v + 1], acc[j][v + 2], acc[j][v + 3]);
        }
      }
    }
  }
}

// Rows spanning several 32-entry items: the item in which the row starts adds the partials of
// the row's items in item order, divides once and rounds.
template <typename T>
__global__ void __launch_bounds__(256) centroid_fixup_kernel(CentroidArgs<T> a) {
  constexpr int VN = Vec<T>::N;
  const int item = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (item >= a.n_items) return;
  const int p0 = item * kChunk;
  const int p1 = min(p0 + kChunk, a.nk);
  if (p1 >= a.nk) return;
  const uint32_t row = a.rows[p1 - 1];
  if (a.rows[p1] != row) return;                       // last row of the item ends inside it
  const int rs = a.row_start[row];
  if (rs < p0) return;                                 // started in an earlier item: not the owner
  const int re = a.row_start[row + 1];
  const int i1 = (re - 1) / kChunk;
  const int nch = a.d * static_cast<int>(sizeof(T)) / 16;
  for (int cb0 = 0; cb0 < nch; cb0 += 32 * kMaxJ) {
    float acc[kMaxJ][VN];
#pragma unroll
    for (int j = 0; j < kMaxJ; ++j) {
      const int ch = cb0 + lane + 32 * j;
      const float* src = a.partial + (static_cast<int64_t>(item) * 2 + (rs == p0 ? 0 : 1)) * a.d + ch * VN;
#pragma unroll
      for (int v = 0; v < VN; ++v) acc[j][v] = ch < nch ? src[v] : 0.0f;
    }
    for (int it = item + 1; it <= i1; ++it) {
#pragma unroll
      for (int j = 0; j < kMaxJ; ++j) {
        const int ch = cb0 + lane + 32 * j;
        if (ch < nch) {
          const float* src = a.partial + (static_cast<int64_t>(it) * 2) * a.d + ch * VN;
#pragma unroll
          for (int v = 0; v < VN; ++v) acc[j][v] += src[v];
        }
      }
    }
    write_centroid(a, static_cast<int>(row), cb0, nch, acc, static_cast<float>(re - rs));
  }
}

__global__ void gather_rows_kernel(const uint8_t* __restrict__ x, int row_bytes, int k, const int32_t* __restrict__ vals,
                                   int nk, uint8_t* __restrict__ send) {
  const int cpr = row_bytes / 16;
  const int64_t total = static_cast<int64_t>(nk) * cpr;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(i / cpr), ch = static_cast<int>(i - int64_t(p) * cpr);
    const int t = vals[p] / k;
    reinterpret_cast<uint4*>(send + static_cast<int64_t>(p) * row_bytes)[ch] =
        reinterpret_cast<const uint4*>(x + static_cast<int64_t>(t) * row_bytes)[ch];
  }
}

int bits_for(int64_t maxval) {   // bits needed to represent values in [0, maxval]
  int b = 1;
  while ((int64_t(1) << b) <= maxval) ++b;
  return b;
}

}  // namespace

int read_and_clear_device_error(int* value, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int err = cudaStreamSynchronize(st);
  if (err) return err;
  err = cudaMemcpyFromSymbol(value, g_device_error, sizeof(int));
  if (err) return err;
  const int zero = 0;
  return cudaMemcpyToSymbol(g_device_error, &zero, sizeof(int));
}

size_t compress_workspace_layout(int64_t n, int k, int E, int d, void* base, CompressWs* ws) {
  (void)E;
  const int64_t nk = n * k;
  int64_t tsize = 1024;
  while (tsize < 2 * nk) tsize <<= 1;
  const int64_t nb = (nk + kRTile - 1) / kRTile;
  const int64_t n_items = (nk + kChunk - 1) / kChunk;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_table = take(sizeof(int32_t) * tsize);
  const size_t o_rep = take(sizeof(int32_t) * nk);
  const size_t o_k0 = take(sizeof(uint32_t) * nk);
  const size_t o_k1 = take(sizeof(uint32_t) * nk);
  const size_t o_v0 = take(sizeof(int32_t) * nk);
  const size_t o_v1 = take(sizeof(int32_t) * nk);
  const size_t o_rowid = take(sizeof(int32_t) * nk);
  const size_t o_hist = take(sizeof(int32_t) * kRadix * (nb > 0 ? nb : 1));
  const size_t o_part = take(sizeof(float) * 2 * n_items * d);
  if (ws) {
    uint8_t* b = static_cast<uint8_t*>(base);
    ws->table = reinterpret_cast<int32_t*>(b + o_table);
    ws->table_size = tsize;
    ws->rep = reinterpret_cast<int32_t*>(b + o_rep);
    ws->keys[0] = reinterpret_cast<uint32_t*>(b + o_k0);
    ws->keys[1] = reinterpret_cast<uint32_t*>(b + o_k1);
    ws->vals[0] = reinterpret_cast<int32_t*>(b + o_v0);
    ws->vals[1] = reinterpret_cast<int32_t*>(b + o_v1);
    ws->rowid = reinterpret_cast<int32_t*>(b + o_rowid);
    ws->hist = reinterpret_cast<int32_t*>(b + o_hist);
    ws->partial = reinterpret_cast<float*>(b + o_part);
    ws->n_items = n_items;
    ws->bytes = off;
  }
  return off;
}

int launch_compress(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int16_t* codes, int q,
                    const int32_t* experts, int k, int E, int32_t* bucket, int32_t* perm, int32_t* row_start,
                    int32_t* expert_rows, int32_t* num_rows, void* centroids, float* centroids_f32,
                    const CompressWs& ws, void* stream) {
  if (E > kMaxE) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nk = static_cast<int>(n * k);
  int err;
  if (nk == 0) {
    if ((err = cudaMemsetAsync(expert_rows, 0, sizeof(int32_t) * E, st))) return err;
    if ((err = cudaMemsetAsync(num_rows, 0, sizeof(int32_t), st))) return err;
    return cudaMemsetAsync(row_start, 0, sizeof(int32_t), st);
  }
  const int sms = device_sm_count();
  const int tgrid = std::min((nk + 255) / 256, 8 * sms);
  if ((err = cudaMemsetAsync(ws.table, 0xFF, sizeof(int32_t) * ws.table_size, st))) return err;
  const uint32_t mask = static_cast<uint32_t>(ws.table_size - 1);
  insert_kernel<<<tgrid, 256, 0, st>>>(codes, q, experts, k, E, nk, ws.table, mask);
  lookup_kernel<<<tgrid, 256, 0, st>>>(codes, q, experts, k, E, nk, ws.table, mask, ws.rep, ws.keys[0]);
  count_launches(2);
  // 3. firsts in (expert, position) order -> rowid, m_e, m
  RadixIO io{};
  io.E = E;
  io.keys_in = ws.keys[0];
  io.vals_in = nullptr;
  io.rowid_out = ws.rowid;
  radix_pass<KEY_DIRECT, OUT_ROWID>(io, nk, 0, ws.hist, expert_rows, num_rows, E, st);
  // 4. stable sort of all copies by row
  const int passes = (bits_for(nk - 1) + 7) / 8;
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    RadixIO r{};
    r.E = E;
    r.keys_out = ws.keys[1 - cur];
    r.vals_out = (p == passes - 1) ? perm : ws.vals[1 - cur];
    if (p == 0) {
      r.rep = ws.rep;
      r.rowid = ws.rowid;
      r.bucket = bucket;
      radix_pass<KEY_ROW, OUT_WRITE>(r, nk, 0, ws.hist, nullptr, nullptr, E, st);
    } else {
      r.keys_in = ws.keys[cur];
      r.vals_in = ws.vals[cur];
      radix_pass<KEY_DIRECT, OUT_WRITE>(r, nk, 8 * p, ws.hist, nullptr, nullptr, E, st);
    }
    cur = 1 - cur;
  }
  const uint32_t* rows_sorted = ws.keys[cur];
  // 5. centroids
  const int items = static_cast<int>(ws.n_items);
  const int cgrid = (items * 32 + 255) / 256;
  if (dtype == LSHMOE_BF16) {
    CentroidArgs<__nv_bfloat16> a{static_cast<const __nv_bfloat16*>(x), d, k, nk, perm, rows_sorted, row_start,
                                  static_cast<__nv_bfloat16*>(centroids), centroids_f32, ws.partial, items};
    centroid_kernel<<<cgrid, 256, 0, st>>>(a);
    centroid_fixup_kernel<<<cgrid, 256, 0, st>>>(a);
  } else {
    CentroidArgs<float> a{static_cast<const float*>(x), d, k, nk, perm, rows_sorted, row_start,
                          static_cast<float*>(centroids), centroids_f32, ws.partial, items};
    centroid_kernel<<<cgrid, 256, 0, st>>>(a);
    centroid_fixup_kernel<<<cgrid, 256, 0, st>>>(a);
  }
  count_launches(2);
  return cudaGetLastError();
}

int launch_permute(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int32_t* experts, int k, int E,
                   int32_t* slot, int32_t* expert_rows, void* send, const CompressWs& ws, void* stream) {
  if (E > kMaxE) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nk = static_cast<int>(n * k);
  if (nk == 0) return cudaMemsetAsync(expert_rows, 0, sizeof(int32_t) * E, st);
  // keys = expert ids (validated); one stable pass -> grouped order, slot, n_e
  RadixIO io{};
  io.E = E;
  io.experts = experts;
  io.keys_out = ws.keys[1];
  io.vals_out = ws.vals[1];
  io.slot_out = slot;
  radix_pass<KEY_EXPERT, OUT_SLOT>(io, nk, 0, ws.hist, expert_rows, ws.vals[0] /* scratch m */, E, st);
  const int row_bytes = d * (dtype == LSHMOE_F32 ? 4 : 2);
  const int64_t chunks = static_cast<int64_t>(nk) * (row_bytes / 16);
  const int grid = static_cast<int>(std::min<int64_t>((chunks + 255) / 256, 16 * device_sm_count()));
  gather_rows_kernel<<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(x), row_bytes, k, ws.vals[1], nk,
                                           static_cast<uint8_t*>(send));
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lshmoe
