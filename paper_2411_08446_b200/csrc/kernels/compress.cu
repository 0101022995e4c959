// a3-a5: group the routed copies by expert, bucket them by their composite LSH key, and reduce
// each bucket to its centroid (Alg. 1 L3, L5-L8: P:L520; §2.3).
//
// One cooperative, persistent kernel (all CTAs co-resident; grid barriers between phases), so
// the whole step is one launch + one memset and needs no host synchronisation:
//   P0 insert  : open-addressing hash table keyed by (expert, q-tuple of codes); each slot's value
//                converges (atomicMin) to the smallest copy id c = t*k+s with that key = the
//                bucket's first appearance in its expert group (reading R7).  slot_of[c] is kept,
//                so later phases read rep[c] = table[slot_of[c]] without re-probing.
//   P1 radix   : one stable counting-sort pass over key = expert (first copies) / E (others):
//                the firsts land in (expert, first position) order, and that position IS the
//                global centroid row (expert-major, first-appearance local ids); the digit totals
//                give m_e and m.
//   P2 radix   : stable LSD sort (8-bit digits, 2 passes for n*k <= 65536) of all copies by
//                row = rowid[rep[c]] -> perm (ascending copy id within a row, reading R8), bucket.
//   P3 centroid: perm split in 16-entry items; one thread per (item, 16-byte column chunk) issues
//                all 16 member loads at once (128-bit), sums in perm order in fp32, divides once
//                by the count (IEEE, reading R10) and rounds (RNE) into the send buffer.  Rows
//                crossing items leave fp32 partials;
//   P4 fix-up  : the item where such a row starts adds the partials in item order (deterministic).
// Stable ranking inside a 1024-element radix tile: per-warp __match_any_sync + per-warp digit
// counters in shared memory (a warp's rounds run in order), warp prefixes combined per digit;
// tiles' histograms are published to global memory and every CTA derives its tiles' offsets.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "../abi/lshmoe_internal.h"
#include "common.cuh"

namespace lshmoe {
namespace {

constexpr int kThreads = 256;            // == kRadix: one thread per digit in the offset step
constexpr int kRadix = 256;
constexpr int kIPT = 1;                  // radix items per thread per tile (small tiles: more CTAs busy)
constexpr int kTile = kThreads * kIPT;   // 1024 elements per radix tile
constexpr int kWarps = kThreads / 32;
constexpr int kCH = 16;                  // perm entries per centroid item
constexpr int kMaxE = 255;               // expert digit + sentinel fit one 8-bit pass
constexpr int kHdr = 64 + 2048;          // workspace header ints: barrier counter, phase + per-CTA stamps

// Device error word (read by lshmoe_check_device_error).  Bit 0: expert id outside [0, E)
// (S:L312).  Only this translation unit validates expert ids.
__device__ int g_device_error = 0;

__device__ __forceinline__ int load_expert(const int32_t* experts, int c, int E) {
  int e = experts[c];
  if (static_cast<unsigned>(e) >= static_cast<unsigned>(E)) {
    atomicOr(&g_device_error, 1);
    e = 0;                                 // keep every index in bounds; the result is flagged
  }
  return e;
}
__device__ __forceinline__ int load_expert_quiet(const int32_t* experts, int c, int E) {
  const int e = experts[c];
  return static_cast<unsigned>(e) >= static_cast<unsigned>(E) ? 0 : e;
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

// Data written by other CTAs in an earlier phase is read with ld.global.cg (L2, not L1).
template <typename T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

struct Params {
  const uint8_t* x;
  int d, row_bytes, nch;           // nch = 16-byte chunks per row
  int is_bf16;
  const int16_t* codes;
  int q;
  const int32_t* experts;
  int k, E, nk;
  int32_t* bucket;                 // compress: [nk] row of copy; permute: slot
  int32_t* perm;
  int32_t* row_start;
  int32_t* expert_rows;
  int32_t* num_rows;
  uint8_t* cent;                   // compress: centroids; permute: send buffer
  float* cent32;
  int32_t* table;
  uint32_t mask;
  unsigned* bar;                   // grid-barrier counter, memset to 0xFFFFFFFF
  int32_t* slot_of;
  int32_t* rowid;
  uint32_t* keys[2];
  int32_t* vals[2];
  int32_t* hist;                   // [ntiles][256]
  float* partial;                  // [n_items][2][d]
  int ntiles, row_passes, n_items;
  int permute;                     // 1: uncompressed baseline (group by expert only)
};

// Grid barrier over co-resident CTAs; the counter starts at 0xFFFFFFFF (memset) and barrier
// number p completes when it reaches p * gridDim.x - 1.
__device__ __forceinline__ unsigned globaltimer_lo() {
  unsigned t;
  asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
  return t;
}

// bar[2 + p] (p = 0..13): CTA 0's globaltimer (ns, low 32 bits) at kernel start (p = 0) and on
// leaving barrier p — a per-phase breakdown readable from the workspace (lshmoe_compress_phases).
__device__ __forceinline__ void stamp(unsigned* bar, unsigned p) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && p < 14) bar[2 + p] = globaltimer_lo();
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& phase) {
  ++phase;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    const unsigned target = phase * gridDim.x - 1u;
    while (static_cast<int>(*reinterpret_cast<volatile unsigned*>(bar) - target) < 0) __nanosleep(32);
    __threadfence();
    stamp(bar, phase);
  }
  __syncthreads();
}

enum PassKind { PASS_FIRSTS = 0, PASS_ROW0 = 1, PASS_ROWN = 2, PASS_PERMUTE = 3 };

__device__ __forceinline__ void pass_key(const Params& P, int kind, int pass, int i, uint32_t& key, int32_t& val) {
  if (kind == PASS_FIRSTS) {
    const int e = load_expert_quiet(P.experts, i, P.E);
    const int rep = ldcg(P.table + ldcg(P.slot_of + i));
    key = rep == i ? static_cast<uint32_t>(e) : static_cast<uint32_t>(P.E);
    val = i;
  } else if (kind == PASS_ROW0) {
    key = static_cast<uint32_t>(ldcg(P.rowid + ldcg(P.table + ldcg(P.slot_of + i))));
    val = i;
  } else if (kind == PASS_ROWN) {
    key = ldcg(P.keys[(pass - 1) & 1] + i);
    val = ldcg(P.vals[(pass - 1) & 1] + i);
  } else {
    key = static_cast<uint32_t>(load_expert(P.experts, i, P.E));
    val = i;
  }
}

struct TileRank {
  uint32_t key[kIPT];
  int32_t val[kIPT];
  int dg[kIPT];
  int loc[kIPT];
};

// Stable ranks of the elements of one tile by digit; leaves per-warp digit counts in wcnt.
__device__ __forceinline__ void rank_tile(const Params& P, int kind, int pass, int tile, int n, int shift,
                                          int (*wcnt)[kRadix], TileRank& tr) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  const int base = tile * kTile + warp * (kIPT * 32);
#pragma unroll
  for (int r = 0; r < kIPT; ++r) {   // all key loads in flight before the ordered ranking rounds
    const int i = base + r * 32 + lane;
    if (i < n) pass_key(P, kind, pass, i, tr.key[r], tr.val[r]);
  }
#pragma unroll
  for (int r = 0; r < kIPT; ++r) {
    const int i = base + r * 32 + lane;
    const bool ok = i < n;
    tr.dg[r] = ok ? static_cast<int>((tr.key[r] >> shift) & (kRadix - 1)) : kRadix;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, tr.dg[r]);
    const int leader = __ffs(peers) - 1;
    int b = 0;
    if (ok) b = wcnt[warp][tr.dg[r]];
    __syncwarp();
    if (ok && lane == leader) wcnt[warp][tr.dg[r]] = b + __popc(peers);
    __syncwarp();
    tr.loc[r] = b + __popc(peers & lt);
  }
  __syncthreads();
}

// One stable counting-sort pass over n elements (key digit at `shift`), all CTAs cooperating.
__device__ void radix_pass(const Params& P, int kind, int pass, int n, int shift, unsigned& phase,
                           int (*wcnt)[kRadix], int* s_off, int* s_tot) {
  const int ntiles = (n + kTile - 1) / kTile;
  const int tpad = (ntiles + 3) & ~3;          // hist is digit-major [256][tpad]: 128-bit row loads
  const bool one_tile = ntiles <= static_cast<int>(gridDim.x);   // keep ranks in registers
  TileRank tr;
  // (a) tile histograms
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    rank_tile(P, kind, pass, t, n, shift, wcnt, tr);
    int s = 0;
    for (int w = 0; w < kWarps; ++w) s += wcnt[w][threadIdx.x];
    P.hist[threadIdx.x * tpad + t] = s;
    if (!one_tile) __syncthreads();
  }
  grid_barrier(P.bar, phase);
  // (b) offsets + stable scatter
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int dgt = threadIdx.x;
    int tot = 0, pre = 0;
    {
      const int4* hrow = reinterpret_cast<const int4*>(P.hist + dgt * tpad);
      for (int u0 = 0; u0 < tpad; u0 += 32) {   // up to 8 x 128-bit loads in flight
        int4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = u0 + 4 * j < tpad ? __ldcg(hrow + u0 / 4 + j) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int u = u0 + 4 * j + i;
            if (u == t) pre = tot;
            if (u < ntiles) tot += e[i];
          }
        }
      }
    }
    // exclusive scan of the 256 digit totals: warp shuffles + one cross-warp step
    {
      const int lane = dgt & 31, wid = dgt >> 5;
      int x = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
      }
      if (lane == 31) s_tot[wid] = x;
      __syncthreads();
      int base = 0;
      for (int w = 0; w < wid; ++w) base += s_tot[w];
      s_tot[32 + dgt] = base + x;           // inclusive
    }
    const int excl = s_tot[32 + dgt] - tot;
    s_off[dgt] = excl + pre;
    if (t == 0 && (kind == PASS_FIRSTS || kind == PASS_PERMUTE)) {
      if (dgt < P.E) P.expert_rows[dgt] = tot;
      if (kind == PASS_FIRSTS && dgt == P.E) *P.num_rows = excl;   // firsts precede the sentinel digit
    }
    if (one_tile) __syncthreads();
    else rank_tile(P, kind, pass, t, n, shift, wcnt, tr);
    {   // warp-exclusive prefix per digit
      int run = 0;
      for (int w = 0; w < kWarps; ++w) {
        const int v = wcnt[w][dgt];
        wcnt[w][dgt] = run;
        run += v;
      }
    }
    __syncthreads();
    const int warp = threadIdx.x / 32;
#pragma unroll
    for (int r = 0; r < kIPT; ++r) {
      if (tr.dg[r] == kRadix) continue;
      const int dest = s_off[tr.dg[r]] + wcnt[warp][tr.dg[r]] + tr.loc[r];
      const uint32_t key = tr.key[r];
      const int32_t val = tr.val[r];
      if (kind == PASS_FIRSTS) {
        if (key < static_cast<uint32_t>(P.E)) P.rowid[val] = dest;
      } else if (kind == PASS_PERMUTE) {
        P.bucket[val] = dest;                 // slot of copy val
        P.vals[0][dest] = val;
      } else {
        if (kind == PASS_ROW0) P.bucket[val] = static_cast<int32_t>(key);
        if (pass == P.row_passes) {           // last pass: sorted rows + perm (+ token ids)
          P.keys[pass & 1][dest] = key;
          P.perm[dest] = val;
          P.vals[pass & 1][dest] = val / P.k;
        } else {
          P.keys[pass & 1][dest] = key;
          P.vals[pass & 1][dest] = val;
        }
      }
    }
    __syncthreads();
  }
  grid_barrier(P.bar, phase);
}

template <typename T>
__device__ __forceinline__ void acc_chunk(float* acc, const uint4& raw) {
  if (sizeof(T) == 2) {
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] += __uint_as_float(w[i] << 16);
      acc[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
    acc[0] += __uint_as_float(raw.x);
    acc[1] += __uint_as_float(raw.y);
    acc[2] += __uint_as_float(raw.z);
    acc[3] += __uint_as_float(raw.w);
  }
}

template <typename T>
__device__ __forceinline__ void store_centroid(const Params& P, int row, int ch, const float* acc, float cnt) {
  constexpr int VN = Vec<T>::N;
  float v[VN];
#pragma unroll
  for (int e = 0; e < VN; ++e) v[e] = __fdiv_rn(acc[e], cnt);
  Vec<T>::store(P.cent + static_cast<int64_t>(row) * P.row_bytes + 16 * ch, v);
  if (P.cent32) {
    float* dst = P.cent32 + static_cast<int64_t>(row) * P.d + ch * VN;
#pragma unroll
    for (int e = 0; e < VN; e += 4) *reinterpret_cast<float4*>(dst + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
  }
}

template <typename T>
__device__ void centroid_phase(const Params& P, const uint32_t* rows, const int32_t* tok) {
  constexpr int VN = Vec<T>::N;
  const int64_t work = static_cast<int64_t>(P.n_items) * P.nch;
  for (int64_t w = blockIdx.x * int64_t(kThreads) + threadIdx.x; w < work; w += int64_t(gridDim.x) * kThreads) {
    const int item = static_cast<int>(w / P.nch);
    const int ch = static_cast<int>(w - int64_t(item) * P.nch);
    const int p0 = item * kCH;
    const int cnt = min(kCH, P.nk - p0);
    uint32_t rw[kCH];
    int tk[kCH];
    // 1) the item's 16 row ids + token ids (128-bit loads), 2) the 16 member chunks: each batch
    // is issued back to back, nothing inside a batch waits on another load
    if (cnt == kCH) {
#pragma unroll
      for (int j = 0; j < kCH; j += 4) {
        const uint4 r4 = __ldcg(reinterpret_cast<const uint4*>(rows + p0 + j));
        const int4 t4 = __ldcg(reinterpret_cast<const int4*>(tok + p0 + j));
        rw[j] = r4.x; rw[j + 1] = r4.y; rw[j + 2] = r4.z; rw[j + 3] = r4.w;
        tk[j] = t4.x; tk[j + 1] = t4.y; tk[j + 2] = t4.z; tk[j + 3] = t4.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kCH; ++j) {
        rw[j] = j < cnt ? ldcg(rows + p0 + j) : 0xFFFFFFFFu;
        tk[j] = j < cnt ? ldcg(tok + p0 + j) : 0;
      }
    }
    const uint32_t prev = p0 > 0 ? ldcg(rows + p0 - 1) : 0xFFFFFFFFu;
    const uint32_t next = p0 + cnt < P.nk ? ldcg(rows + p0 + cnt) : 0xFFFFFFFFu;
    uint4 v[kCH];
#pragma unroll
    for (int j = 0; j < kCH; ++j)
      v[j] = j < cnt ? __ldg(reinterpret_cast<const uint4*>(P.x + static_cast<int64_t>(tk[j]) * P.row_bytes) + ch)
                     : make_uint4(0, 0, 0, 0);
    // segment ends (bit j: member j closes its row inside this item) and row heads
    unsigned ends = 0, heads = 0;
#pragma unroll
    for (int j = 0; j < kCH; ++j) {
      if (j < cnt) {
        ends |= static_cast<unsigned>(j == cnt - 1 || rw[j + 1 < kCH ? j + 1 : j] != rw[j]) << j;
        heads |= static_cast<unsigned>(rw[j] != (j == 0 ? prev : rw[j > 0 ? j - 1 : 0])) << j;
      }
    }
    if (ch == 0) {   // row boundaries (perm offsets)
      for (unsigned h = heads; h; h &= h - 1) {
        const int j = __ffs(h) - 1;
        P.row_start[rw[j]] = p0 + j;
      }
      if (p0 + cnt == P.nk) P.row_start[rw[cnt - 1] + 1] = P.nk;
    }
    float acc[VN];
#pragma unroll
    for (int e = 0; e < VN; ++e) acc[e] = 0.0f;
    int s = 0;
#pragma unroll
    for (int j = 0; j < kCH; ++j) {
      acc_chunk<T>(acc, v[j]);          // members past cnt are zeros after the last flush
      if ((ends >> j) & 1u) {
        const bool complete = (s > 0 || prev != rw[j]) && (j < cnt - 1 || next != rw[j]);
        if (complete) {
          store_centroid<T>(P, static_cast<int>(rw[j]), ch, acc, static_cast<float>(j + 1 - s));
        } else {
          float* dst = P.partial + (static_cast<int64_t>(item) * 2 + (s == 0 ? 0 : 1)) * P.d + ch * VN;
#pragma unroll
          for (int e = 0; e < VN; e += 4) *reinterpret_cast<float4*>(dst + e) = make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
        }
#pragma unroll
        for (int e = 0; e < VN; ++e) acc[e] = 0.0f;
        s = j + 1;
      }
    }
  }
}

template <typename T>
__device__ void fixup_phase(const Params& P, const uint32_t* rows) {
  constexpr int VN = Vec<T>::N;
  const int64_t work = static_cast<int64_t>(P.n_items) * P.nch;
  for (int64_t w = blockIdx.x * int64_t(kThreads) + threadIdx.x; w < work; w += int64_t(gridDim.x) * kThreads) {
    const int item = static_cast<int>(w / P.nch);
    const int ch = static_cast<int>(w - int64_t(item) * P.nch);
    const int p0 = item * kCH;
    const int p1 = min(p0 + kCH, P.nk);
    if (p1 >= P.nk) continue;
    const uint32_t row = ldcg(rows + p1 - 1);
    if (ldcg(rows + p1) != row) continue;             // the item's last row ends inside it
    const int rs = ldcg(P.row_start + row);
    if (rs < p0) continue;                            // started earlier: not the owner
    const int re = ldcg(P.row_start + row + 1);
    const int i1 = (re - 1) / kCH;
    float acc[VN];
    {
      const float* src = P.partial + (static_cast<int64_t>(item) * 2 + (rs == p0 ? 0 : 1)) * P.d + ch * VN;
#pragma unroll
      for (int e = 0; e < VN; e += 4) {
        const float4 f = __ldcg(reinterpret_cast<const float4*>(src + e));
        acc[e] = f.x; acc[e + 1] = f.y; acc[e + 2] = f.z; acc[e + 3] = f.w;
      }
    }
    for (int it0 = item + 1; it0 <= i1; it0 += 8) {   // 8 partials in flight, summed in item order
      float4 f[8][VN / 4];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (it0 + u <= i1) {
          const float* src = P.partial + (static_cast<int64_t>(it0 + u) * 2) * P.d + ch * VN;
#pragma unroll
          for (int e = 0; e < VN / 4; ++e) f[u][e] = __ldcg(reinterpret_cast<const float4*>(src) + e);
        }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (it0 + u <= i1) {
#pragma unroll
          for (int e = 0; e < VN / 4; ++e) {
            acc[4 * e] += f[u][e].x;
            acc[4 * e + 1] += f[u][e].y;
            acc[4 * e + 2] += f[u][e].z;
            acc[4 * e + 3] += f[u][e].w;
          }
        }
    }
    store_centroid<T>(P, static_cast<int>(row), ch, acc, static_cast<float>(re - rs));
  }
}

__device__ void insert_phase(const Params& P) {
  for (int c = blockIdx.x * kThreads + threadIdx.x; c < P.nk; c += gridDim.x * kThreads) {
    const int e = load_expert(P.experts, c, P.E);
    const int16_t* mc = P.codes + static_cast<int64_t>(c / P.k) * P.q;
    uint32_t slot = key_hash(e, mc, P.q) & P.mask;
    while (true) {
      int cur = *reinterpret_cast<volatile int32_t*>(&P.table[slot]);
      if (cur < 0) {
        const int old = atomicCAS(&P.table[slot], -1, c);
        if (old < 0) break;                  // claimed an empty slot
        cur = old;
      }
      // cur is a copy with this slot's key (a claimed slot never changes key)
      if (load_expert_quiet(P.experts, cur, P.E) == e && codes_equal(P.codes + static_cast<int64_t>(cur / P.k) * P.q, mc, P.q)) {
        if (c < cur) atomicMin(&P.table[slot], c);
        break;
      }
      slot = (slot + 1) & P.mask;
    }
    P.slot_of[c] = static_cast<int32_t>(slot);
  }
}

template <typename T>
__device__ void gather_phase(const Params& P) {   // baseline: send[p] = x[token of copy at p]
  const int64_t work = static_cast<int64_t>(P.nk) * P.nch;
  for (int64_t w = blockIdx.x * int64_t(kThreads) + threadIdx.x; w < work; w += int64_t(gridDim.x) * kThreads) {
    const int p = static_cast<int>(w / P.nch);
    const int ch = static_cast<int>(w - int64_t(p) * P.nch);
    const int t = ldcg(P.vals[0] + p) / P.k;
    reinterpret_cast<uint4*>(P.cent + static_cast<int64_t>(p) * P.row_bytes)[ch] =
        __ldg(reinterpret_cast<const uint4*>(P.x + static_cast<int64_t>(t) * P.row_bytes) + ch);
  }
}

__global__ void __launch_bounds__(kThreads) compress_kernel(Params P) {
  __shared__ int wcnt[kWarps][kRadix];
  __shared__ int s_off[kRadix];
  __shared__ int s_tot[kRadix + 32];
  unsigned phase = 0;
  stamp(P.bar, 0);
  if (P.permute) {
    radix_pass(P, PASS_PERMUTE, 0, P.nk, 0, phase, wcnt, s_off, s_tot);
    gather_phase<float>(P);
    return;
  }
  insert_phase(P);
  grid_barrier(P.bar, phase);
  radix_pass(P, PASS_FIRSTS, 0, P.nk, 0, phase, wcnt, s_off, s_tot);
  for (int p = 1; p <= P.row_passes; ++p)
    radix_pass(P, p == 1 ? PASS_ROW0 : PASS_ROWN, p, P.nk, 8 * (p - 1), phase, wcnt, s_off, s_tot);
  const uint32_t* rows = P.keys[P.row_passes & 1];
  const int32_t* tok = P.vals[P.row_passes & 1];    // token id of each perm entry
  // per-CTA centroid-phase start / end stamps (diagnostics, bar[64 + 2 * cta])
  if (threadIdx.x == 0 && blockIdx.x < 1024) P.bar[64 + 2 * blockIdx.x] = globaltimer_lo();
  if (P.is_bf16) {
    centroid_phase<__nv_bfloat16>(P, rows, tok);
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < 1024) P.bar[65 + 2 * blockIdx.x] = globaltimer_lo();
    grid_barrier(P.bar, phase);
    fixup_phase<__nv_bfloat16>(P, rows);
  } else {
    centroid_phase<float>(P, rows, tok);
    grid_barrier(P.bar, phase);
    fixup_phase<float>(P, rows);
  }
  __syncthreads();
  stamp(P.bar, phase + 1);   // CTA 0's end (other CTAs may still be finishing the fix-up)
}

int bits_for(int64_t maxval) {   // bits needed to represent values in [0, maxval]
  int b = 1;
  while ((int64_t(1) << b) <= maxval) ++b;
  return b;
}

int coop_grid() {
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compress_kernel, kThreads, 0);
    grid = std::max(1, std::min(per_sm, 4)) * device_sm_count();
  }
  return grid;
}

int launch_coop(const Params& P, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(coop_grid());
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  Params p = P;
  int err = cudaLaunchKernelEx(&cfg, compress_kernel, p);
  count_launches(1);
  return err;
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
  const int64_t ntiles = (nk + kTile - 1) / kTile;
  const int64_t n_items = (nk + kCH - 1) / kCH;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_table = take(sizeof(int32_t) * (tsize + kHdr));   // + header: barrier counter, stamps
  const size_t o_slot = take(sizeof(int32_t) * nk);
  const size_t o_k0 = take(sizeof(uint32_t) * nk);
  const size_t o_k1 = take(sizeof(uint32_t) * nk);
  const size_t o_v0 = take(sizeof(int32_t) * nk);
  const size_t o_v1 = take(sizeof(int32_t) * nk);
  const size_t o_rowid = take(sizeof(int32_t) * nk);
  const size_t o_hist = take(sizeof(int32_t) * kRadix * ((ntiles + 3) & ~int64_t(3)) + 64);
  const size_t o_part = take(sizeof(float) * 2 * n_items * d);
  if (ws) {
    uint8_t* b = static_cast<uint8_t*>(base);
    ws->table = reinterpret_cast<int32_t*>(b + o_table);
    ws->table_size = tsize;
    ws->rep = reinterpret_cast<int32_t*>(b + o_slot);
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

static Params base_params(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int32_t* experts, int k, int E,
                          const CompressWs& ws) {
  Params P{};
  P.x = static_cast<const uint8_t*>(x);
  P.d = d;
  P.row_bytes = d * (dtype == LSHMOE_F32 ? 4 : 2);
  P.nch = P.row_bytes / 16;
  P.is_bf16 = dtype == LSHMOE_BF16;
  P.experts = experts;
  P.k = k;
  P.E = E;
  P.nk = static_cast<int>(n * k);
  P.table = ws.table + kHdr;
  P.bar = reinterpret_cast<unsigned*>(ws.table);
  P.mask = static_cast<uint32_t>(ws.table_size - 1);
  P.slot_of = ws.rep;
  P.rowid = ws.rowid;
  P.keys[0] = ws.keys[0];
  P.keys[1] = ws.keys[1];
  P.vals[0] = ws.vals[0];
  P.vals[1] = ws.vals[1];
  P.hist = ws.hist;
  P.partial = ws.partial;
  P.ntiles = (P.nk + kTile - 1) / kTile;
  P.n_items = static_cast<int>(ws.n_items);
  return P;
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
  // hash table slots (-1) and the grid-barrier counter (0xFFFFFFFF) in one memset
  if ((err = cudaMemsetAsync(ws.table, 0xFF, sizeof(int32_t) * (ws.table_size + kHdr), st))) return err;
  Params P = base_params(x, dtype, n, d, experts, k, E, ws);
  P.codes = codes;
  P.q = q;
  P.bucket = bucket;
  P.perm = perm;
  P.row_start = row_start;
  P.expert_rows = expert_rows;
  P.num_rows = num_rows;
  P.cent = static_cast<uint8_t*>(centroids);
  P.cent32 = centroids_f32;
  P.row_passes = (bits_for(nk - 1) + 7) / 8;
  return launch_coop(P, st);
}

int launch_permute(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int32_t* experts, int k, int E,
                   int32_t* slot, int32_t* expert_rows, void* send, const CompressWs& ws, void* stream) {
  if (E > kMaxE + 1) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nk = static_cast<int>(n * k);
  if (nk == 0) return cudaMemsetAsync(expert_rows, 0, sizeof(int32_t) * E, st);
  int err;
  if ((err = cudaMemsetAsync(ws.table, 0xFF, sizeof(int32_t) * 64, st))) return err;   // barrier counter
  Params P = base_params(x, dtype, n, d, experts, k, E, ws);
  P.bucket = slot;
  P.expert_rows = expert_rows;
  P.cent = static_cast<uint8_t*>(send);
  P.permute = 1;
  return launch_coop(P, st);
}

}  // namespace lshmoe
