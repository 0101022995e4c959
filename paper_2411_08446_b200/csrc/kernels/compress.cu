// a3-a5: group the routed copies by expert, bucket them by their composite LSH key, and reduce
// each bucket to its centroid (Alg. 1 L3, L5-L8: P:L520; §2.3).
//
// Two or three kernels chained by programmatic dependent launch (PDL: each kernel's launch and
// prologue overlap its predecessor's tail; griddepcontrol.wait orders the data), no host
// synchronisation.  Group path (n*k <= 16K copies or <= 1024 per expert, see group_path): K12 group_kernel (one CTA per
// expert, everything in shared memory; described at its definition) -> K3.  Tiles path:
//   K1 tile_kernel   (one CTA per 256-copy tile): insert every copy into an open-addressing hash
//                    table keyed by (expert, q-tuple of codes) whose slot value converges
//                    (atomicMin) to the smallest copy id with that key = the bucket's first
//                    appearance in its expert group (reading R7).  Lanes of a warp holding the same
//                    key are merged by __match_any_sync first (one atomic per warp and key).  The
//                    tile is stably grouped by expert in shared memory (warp match + per-warp digit
//                    counters) and written out with its per-expert run offsets.
//   K2 bucket_kernel (one 1024-thread CTA per expert): gather the expert's copies in ascending copy
//                    id from the tiles' runs, flag first appearances (table[slot] == copy), number
//                    them by an ordered ballot scan (local row ids), look up every copy's row, and
//                    rank copies within rows in order (warps own contiguous sub-ranges;
//                    __match_any_sync inside a warp, per-(warp,row) counters in shared memory,
//                    prefix over warps) -> perm (grouped by row, ascending copy id within, reading
//                    R8) and row starts.
//   K3 centroid_kernel (one CTA per SM): perm split into one contiguous range per CTA; member
//                    rows are staged in shared memory by cp.async, summed in perm order in fp32,
//                    scaled once by RN(1/count) (reading R10) and rounded (RNE) into the send
//                    buffer.  Rows crossing CTA ranges leave fp32 partials; the last CTA to finish
//                    such a row (arrival counter) adds them in CTA order, so the summation order
//                    never depends on timing.
// The uncompressed baseline (permute mode) runs K1 without the hash table, K2 as a pure ordered
// gather (slot = group offset + rank), then a gather of the token rows into the send buffer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "../abi/lshmoe_internal.h"
#include "common.cuh"

namespace lshmoe {
namespace {

constexpr int kThreads = 256;            // K1 / K3 threads per CTA; K1 tile = 256 copies
constexpr int kTile = kThreads;
constexpr int kRadix = 256;              // expert digits per tile (E + sentinel <= 256)
constexpr int kWarps = kThreads / 32;
constexpr int kBThreads = 1024;          // K2 threads per CTA
constexpr int kBWarps = kBThreads / 32;
constexpr int kMaxE = 255;
constexpr int kMaxCS = 8;                // K2 CTAs per expert (portable cluster size)
constexpr int kMaxGrid = 512;            // K3 CTAs (one per SM) <= this
// Workspace header (int32 words), memset to 0xFF (= -1) before every compress:
// [2..16) stamps, [64, 64 + 2*1024) K3 per-CTA stamps, [kArrive, +kMaxGrid) arrival counters of
// rows cut by K3's CTA ranges, [kDiag, +16*kMaxGrid) per-CTA diagnostics stamps.
constexpr int kArrive = 64 + 2048;
constexpr int kDiag = kArrive + kMaxGrid;
constexpr int kHdr = kDiag + 16 * kMaxGrid;

// Device error word (read by lshmoe_check_device_error).  Bit 0: expert id outside [0, E)
// (S:L312); bit 1: an expert repeated among a token's k slots ("distinct").  Only this
// translation unit validates expert ids.
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

// Data written by other CTAs / earlier kernels of the chain is read with ld.global.cg.
template <typename T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

struct Params {
  const uint8_t* x;
  int d, row_bytes, nch;           // nch = 16-byte chunks per row
  int is_bf16;
  const int16_t* codes;
  int q;
  const int32_t* experts;
  int k, E, nk, ntiles;
  int32_t* bucket;                 // compress: [nk] row of copy; permute: slot
  int32_t* perm;
  int32_t* row_start;
  int32_t* expert_rows;
  int32_t* num_rows;
  uint8_t* cent;                   // compress: centroids; permute: send buffer
  float* cent32;
  int32_t* table;
  uint32_t mask;
  unsigned* bar;                   // workspace header (stamps, arrival counters)
  int32_t* tile_copy;
  int32_t* tile_slot;
  int32_t* tile_off;
  int32_t* rowid;
  int32_t* rowl;
  int32_t* rsl;
  int32_t* gofs;
  int32_t* big;                    // [5][CS * nk] K2 slice arrays of groups too large for shared memory
  int32_t* rtot;                   // [CS * nk] K2 per-(cluster rank, row) totals
  int32_t* fcnt;                   // [E * CS] K2 per-CTA first-appearance counts
  int cs;                          // K2 cluster size (CTAs per expert)
  float* partial;                  // [G][2][d] partial sums of rows cut by K3's CTA ranges
  int max_range;                   // K3: max perm entries per CTA range
  int dyn_smem;                    // K2: dynamic shared memory bytes
  int permute;                     // 1: uncompressed baseline (group by expert only)
  int grad;                        // 1: NEXT-1 grad_compress: weighted per-row SUMS (no 1/count)
  const float* gw;                 // grad: gate weights [nk] or nullptr (weight 1)
  int diag;                        // 1: record per-CTA globaltimer stamps (diagnostics)
  int table_clean;                 // 1: the global hash table was not used (group path): K3 skips its reset
  int early_gate;                  // 1: the gate map is complete before the preceding kernel signals its
                                   // dependents (not lshmoe_gate_hash's output): group_kernel compacts it
                                   // before griddepcontrol.wait, overlapping the hash kernel's tail
  // phase-2 dispatch fused into K3 (lshmoe_compress_p2p); p2p_peers == nullptr: off
  uint8_t* const* p2p_peers;
  int64_t p2p_mailbox, p2p_recv, p2p_data_flag, p2p_recv_cap;
  int p2p_world, p2p_me;
  unsigned long long p2p_spin_ns;   // peer-wait limit (then error bit 4 in p2p_done[1], no trap)
  unsigned* p2p_done;
  int32_t* p2p_recv_rows;
};

// K3's fused-dispatch tables (shared, set once per CTA): first global row of each expert and the
// destination row, in its owner's receive buffer, of this rank's first row of each expert.
__shared__ int g_f_roff[257];
__shared__ long long g_f_dst[256];

// Destination of centroid row `row` in its owner's receive buffer (nullptr: over capacity, flagged).
__device__ __forceinline__ uint8_t* fused_row_dst(const Params& P, int row) {
  int lo = 0, hi = P.E - 1;                 // expert of global row `row`: last e with roff[e] <= row
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g_f_roff[mid] <= row) lo = mid; else hi = mid - 1;
  }
  const int64_t drow = g_f_dst[lo] + (row - g_f_roff[lo]);
  if (drow >= P.p2p_recv_cap) {             // the owner's receive buffer is too small: drop, flag
    atomicOr(P.p2p_done + 1, 1u);
    return nullptr;
  }
  return P.p2p_peers[lo / (P.E / P.p2p_world)] + P.p2p_recv + drow * P.row_bytes;
}


__device__ __forceinline__ unsigned globaltimer_lo() {
  unsigned t;
  asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
  return t;
}
// Diagnostics stamp j of CTA blockIdx.x of kernel `kern` (0: K1, 1: K2, 2: K3).
__device__ __forceinline__ void dstamp(const Params& P, int kern, int j) {
  if (P.diag && threadIdx.x == 0 && blockIdx.x < kMaxGrid / 4)
    P.bar[kDiag + 16 * (blockIdx.x + kern * (kMaxGrid / 4)) + j] = globaltimer_lo();
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets the next PDL-launched kernel's CTAs be scheduled (onto SMs this grid leaves free) and run
// their prologue; they still block in their own pdl_wait until this grid has completed.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Exclusive scan of one int per thread over a CTA of NW warps; *total = the sum.  s = [NW + 1].
template <int NW>
__device__ __forceinline__ int block_excl_scan(int v, int* s, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) s[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int w = lane < NW ? s[lane] : 0;
    int z = w;
#pragma unroll
    for (int off = 1; off < NW; off <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, z, off);
      if (lane >= off) z += y;
    }
    if (lane < NW) s[lane] = z - w;
    if (lane == NW - 1) s[NW] = z;
  }
  __syncthreads();
  const int r = s[wid] + x - v;
  *total = s[NW];
  __syncthreads();                         // s may be reused right away
  return r;
}

// ---- K1: hash-table insert + per-tile stable grouping by expert -----------------------------
constexpr int kMaxQ = 16;                // LSHMOE_MAX_Q

// Slot of copy c.  Lanes of `act` with the same (expert, key) are merged: the lowest such lane
// (smallest copy id) inserts, the others take its slot.  key[] = the token's q codes.
__device__ __forceinline__ int insert_copy(const Params& P, unsigned act, int c, int e, const int16_t* key) {
  const int lane = threadIdx.x & 31;
  uint32_t h = fmix32(static_cast<uint32_t>(e) + 0x9E3779B9u);
#pragma unroll
  for (int i = 0; i < kMaxQ; ++i)
    if (i < P.q) h = fmix32(h ^ (static_cast<uint32_t>(static_cast<uint16_t>(key[i])) + (i << 16)));
  const unsigned peers = __match_any_sync(act, h);
  const int leader = __ffs(peers) - 1;
  // confirm the whole key against the leader's (a 32-bit hash may collide inside a warp)
  bool same = __shfl_sync(act, e, leader) == e;
#pragma unroll
  for (int i = 0; i < kMaxQ; ++i)
    if (i < P.q) same &= __shfl_sync(act, static_cast<int>(key[i]), leader) == key[i];
  const bool own = lane == leader || !same;
  int slot = 0;
  if (own) {
    slot = static_cast<int>(h & P.mask);
    while (true) {
      const int cur = atomicCAS(&P.table[slot], -1, c);
      if (cur < 0) break;                    // claimed an empty slot
      // cur is a copy with this slot's key (a claimed slot never changes key)
      bool eq = load_expert_quiet(P.experts, cur, P.E) == e;
      const int16_t* oc = P.codes + static_cast<int64_t>(cur / P.k) * P.q;
#pragma unroll
      for (int i = 0; i < kMaxQ; ++i)
        if (i < P.q) eq &= oc[i] == key[i];
      if (eq) {
        if (c < cur) atomicMin(&P.table[slot], c);
        break;
      }
      slot = (slot + 1) & static_cast<int>(P.mask);
    }
  }
  const int ls = __shfl_sync(act, slot, leader);
  return own ? slot : ls;
}

__global__ void __launch_bounds__(kThreads) tile_kernel(Params P) {
  __shared__ int wcnt[kWarps][kRadix];
  __shared__ int s_off[kRadix];
  __shared__ int s_scan[kWarps + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int E1 = P.E + 1;
  const int t = blockIdx.x;
  pdl_wait();                                // the hash kernel's codes (and every earlier write) are visible
  // (no early trigger here: bucket CTAs placed beside a small tile grid delayed K2 by ~6 us on C2)
  dstamp(P, 0, 0);
  const int c = t * kTile + tid;
  const bool ok = c < P.nk;
  const int e = ok ? load_expert(P.experts, c, P.E) : P.E;   // digit E = past the end
  if (ok && P.k > 1) {                       // the token's k experts must be distinct
    const int s = c % P.k;
    for (int s2 = 0; s2 < s; ++s2)
      if (P.experts[c - s + s2] == P.experts[c]) atomicOr(&g_device_error, 2);
  }
  int16_t key[kMaxQ];
  if (ok && !P.permute) {
    const int16_t* mc = P.codes + static_cast<int64_t>(c / P.k) * P.q;
#pragma unroll
    for (int i = 0; i < kMaxQ; ++i)
      if (i < P.q) key[i] = mc[i];
  }
  for (int i = tid; i < kWarps * kRadix; i += kThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  // stable rank of the copy among the tile's copies of its expert (one 32-copy round per warp)
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, e);
  if (lane == __ffs(peers) - 1) wcnt[warp][e] = __popc(peers);
  __syncthreads();
  int tot = 0;
  if (tid < E1) {                          // prefix over warps, per expert digit
    for (int w = 0; w < kWarps; ++w) {
      const int v = wcnt[w][tid];
      wcnt[w][tid] = tot;
      tot += v;
    }
  }
  int all;
  const int excl = block_excl_scan<kWarps>(tid < E1 ? tot : 0, s_scan, &all);
  if (tid < E1) {
    s_off[tid] = excl;
    P.tile_off[static_cast<int64_t>(t) * E1 + tid] = excl;
  }
  __syncthreads();
  const unsigned act = __ballot_sync(0xFFFFFFFFu, ok);
  int slot = 0;
  if (ok && !P.permute) slot = insert_copy(P, act, c, e, key);
  if (ok) {
    const int dest = t * kTile + s_off[e] + wcnt[warp][e] + __popc(peers & lt);
    P.tile_copy[dest] = c;
    P.tile_slot[dest] = slot;
  }
  dstamp(P, 0, 1);
}

// ---- K2: per-expert ordered bucketing, one thread-block cluster of CS CTAs per expert ----------
// CTA rank r of expert e's cluster owns the member positions [r*n_e/CS, (r+1)*n_e/CS) of the
// expert's ordered copy list.  The two ordered steps that span the whole group (numbering the
// first appearances; ranking copies within their rows) take a per-CTA partial in shared memory,
// publish the CTA's totals to the workspace, and combine them after a cluster barrier
// (barrier.cluster release/acquire orders the global writes of the cluster's CTAs).
extern __shared__ __align__(1024) uint8_t g_dsmem[];

// Cluster barrier publishing this CTA's global writes: bar.sync orders them before thread 0's
// gpu-scope fence (cumulative), whose relaxed arrive + the peers' acquiring wait form the release /
// acquire pair — one MEMBAR per CTA instead of a release arrive (MEMBAR.GPU) in every thread.
__device__ __forceinline__ void cluster_barrier() {
  __syncthreads();
  if (threadIdx.x == 0) __threadfence();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Ordered gather of positions [s0, s1) of expert e's copy list (and their slots) from the tiles'
// runs into mem[i - s0], aux[i - s0].
__device__ void gather_group(const Params& P, int e, int s0, int s1, int32_t* mem, int32_t* aux, int* s_tb, int* s_ta,
                             int* s_scan, int staged_total) {   // staged_total >= 0: single chunk pre-staged
  const int tid = threadIdx.x;
  const int E1 = P.E + 1;
  int base = 0;
  for (int t0 = 0; t0 < P.ntiles && base < s1; t0 += kBThreads) {
    int tot;
    if (staged_total >= 0) {               // the caller's sizing scan already staged this chunk
      tot = staged_total;
    } else {
      const int t = t0 + tid;
      int a = 0, cnt = 0;
      if (t < P.ntiles) {
        a = ldcg(P.tile_off + static_cast<int64_t>(t) * E1 + e);
        cnt = ldcg(P.tile_off + static_cast<int64_t>(t) * E1 + e + 1) - a;
      }
      const int excl = block_excl_scan<kBWarps>(cnt, s_scan, &tot);
      s_tb[tid] = excl;
      s_ta[tid] = a;
      __syncthreads();
    }
    const int nt = min(kBThreads, P.ntiles - t0);
    dstamp(P, 1, 7);
    // this chunk's positions [base, base + tot) intersected with [s0, s1); thread owns entries
    // i = lo_i + tid + 1024 j; tile of entry i = the last tile with s_tb <= i - base (branchless
    // search, the 8 entries interleaved)
    const int lo_i = max(s0, base) - base, hi_i = min(s1, base + tot) - base;
    int top = 1;
    while (top * 2 < nt) top *= 2;
    for (int i0 = lo_i; i0 < hi_i; i0 += 8 * kBThreads) {
      int lo[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) lo[j] = 0;
      const int nj = min(8, (hi_i - i0 - tid + kBThreads - 1) / kBThreads);   // entries of this thread
      for (int step = top; step >= 1; step >>= 1) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = i0 + j * kBThreads + tid;
          if (j < nj && lo[j] + step < nt && s_tb[lo[j] + step] <= i) lo[j] += step;
        }
      }
      int cc[8], ss[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j * kBThreads + tid;
        if (j < nj) {
          const int src = (t0 + lo[j]) * kTile + s_ta[lo[j]] + (i - s_tb[lo[j]]);
          cc[j] = ldcg(P.tile_copy + src);
          ss[j] = ldcg(P.tile_slot + src);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j * kBThreads + tid;
        if (j < nj) {
          mem[base + i - s0] = cc[j];
          aux[base + i - s0] = ss[j];
        }
      }
    }
    base += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBThreads, 1) bucket_kernel(Params P) {
  __shared__ int s_tb[kBThreads];
  __shared__ int s_ta[kBThreads];
  __shared__ int s_scan[kBWarps + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int CS = P.cs;
  const int e = blockIdx.x / CS, r = blockIdx.x - e * CS;   // cluster (CS, 1, 1): rank = blockIdx.x % CS
  const int E1 = P.E + 1;
  pdl_wait();                               // K1's tiles and table are complete and visible
  pdl_trigger();
  dstamp(P, 1, 0);
  // group size and offset: one column of the tile offsets
  int n_e, goff;
  const bool staged = P.ntiles <= kBThreads;   // one chunk of tiles: the sizing scan stages the runs
  {
    int cnt = 0, a = 0;
    for (int t = tid; t < P.ntiles; t += kBThreads) {
      const int x0 = ldcg(P.tile_off + static_cast<int64_t>(t) * E1 + e);
      cnt += ldcg(P.tile_off + static_cast<int64_t>(t) * E1 + e + 1) - x0;
      a += x0;
    }
    const int excl = block_excl_scan<kBWarps>(cnt, s_scan, &n_e);
    if (staged) {                          // tile t's run of expert e: [s_ta[t], +cnt) at member s_tb[t]
      s_tb[tid] = excl;
      s_ta[tid] = a;
    }
    block_excl_scan<kBWarps>(a, s_scan, &goff);   // copies of experts < e = the group's perm offset
  }
  dstamp(P, 1, 6);
  const int s0 = static_cast<int>(static_cast<int64_t>(r) * n_e / CS);
  const int s1 = static_cast<int>(static_cast<int64_t>(r + 1) * n_e / CS);
  const int ns = s1 - s0;
  // slice arrays: shared memory when the slice and the expert's row arrays fit, else workspace
  // (per cluster rank: [CS][nk] regions at CS * goff + r * n_e)
  int32_t *mem, *aux, *row;
  const bool in_smem = static_cast<int64_t>(12) * ns + static_cast<int64_t>(8) * n_e <= P.dyn_smem;
  const int64_t wbase = static_cast<int64_t>(CS) * goff + static_cast<int64_t>(r) * n_e;
  if (in_smem) {
    int32_t* sm = reinterpret_cast<int32_t*>(g_dsmem);
    mem = sm; aux = sm + ns; row = sm + 2 * ns;
  } else {
    mem = P.big + 0 * static_cast<int64_t>(CS) * P.nk + wbase;
    aux = P.big + 1 * static_cast<int64_t>(CS) * P.nk + wbase;
    row = P.big + 2 * static_cast<int64_t>(CS) * P.nk + wbase;
  }
  gather_group(P, e, s0, s1, mem, aux, s_tb, s_ta, s_scan, staged ? n_e : -1);
  dstamp(P, 1, 1);
  if (tid == 0 && r == 0) P.gofs[e] = goff;
  if (P.permute) {                        // baseline: slot = group offset + rank in the group
    for (int i = tid; i < ns; i += kBThreads) {
      const int c = mem[i];
      P.bucket[c] = goff + s0 + i;
      P.rowl[goff + s0 + i] = c;
    }
    if (tid == 0 && r == 0) P.expert_rows[e] = n_e;
    return;
  }
  // first copy of every member's bucket (the table is final)
  for (int i0 = 0; i0 < ns; i0 += 8 * kBThreads) {
    int v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = i0 + j * kBThreads + tid;
      if (i < ns) v[j] = ldcg(P.table + aux[i]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = i0 + j * kBThreads + tid;
      if (i < ns) aux[i] = v[j];
    }
  }
  __syncthreads();
  // local row ids of the first appearances, in member order: warps own contiguous spans of the
  // slice and count by ballots; the CTA's count is published, the cluster's prefix is its base
  const int span = ((ns + kBWarps - 1) / kBWarps + 31) & ~31;
  const int w0 = min(ns, warp * span), w1 = min(ns, w0 + span);
  int nf = 0;
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    nf += __popc(__ballot_sync(0xFFFFFFFFu, i < w1 && aux[i] == mem[i]));
  }
  int cta_f;
  int lr = block_excl_scan<kBWarps>(lane == 0 ? nf : 0, s_scan, &cta_f);
  if (tid == 0) P.fcnt[blockIdx.x] = cta_f;
  cluster_barrier();
  int m_e = 0, fbase = 0;
  for (int q = 0; q < CS; ++q) {
    const int v = ldcg(P.fcnt + e * CS + q);
    if (q < r) fbase += v;
    m_e += v;
  }
  lr = __shfl_sync(0xFFFFFFFFu, lr, 0) + fbase;
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    const bool f = i < w1 && aux[i] == mem[i];
    const unsigned fb = __ballot_sync(0xFFFFFFFFu, f);
    if (f) {
      const int rr = lr + __popc(fb & lt);
      row[i] = rr;
      P.rowid[mem[i]] = rr;
    }
    lr += __popc(fb);
  }
  cluster_barrier();                       // every CTA's first appearances have their row ids
  dstamp(P, 1, 2);
  for (int i0 = 0; i0 < ns; i0 += 8 * kBThreads) {   // the other members look their row up
    int v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = i0 + j * kBThreads + tid;
      v[j] = -1;
      if (i < ns && aux[i] != mem[i]) v[j] = ldcg(P.rowid + aux[i]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = i0 + j * kBThreads + tid;
      if (v[j] >= 0) row[i] = v[j];
    }
  }
  // rank inside rows over the slice: W warps own contiguous sub-ranges; per-(warp, row) counters;
  // rs[m_e] holds the row sizes and then the row starts (every CTA of the cluster computes them)
  int32_t *rs, *wcnt;
  int W;
  if (in_smem) {
    int32_t* sm = reinterpret_cast<int32_t*>(g_dsmem);
    rs = sm + 3 * ns;
    wcnt = rs + m_e;
    W = static_cast<int>(min(static_cast<int64_t>(kBWarps),
                             (P.dyn_smem - static_cast<int64_t>(12) * ns - static_cast<int64_t>(4) * m_e) /
                                 (4 * max(m_e, 1))));
    if (W < 1) W = 1;   // (12 ns + 8 n_e <= dyn_smem guarantees room for W = 1)
  } else {
    rs = P.big + 3 * static_cast<int64_t>(CS) * P.nk + wbase;
    wcnt = P.big + 4 * static_cast<int64_t>(CS) * P.nk + wbase;
    W = 1;
  }
  const int sub = (ns + W - 1) / W;
  for (int i = tid; i < W * m_e; i += kBThreads) wcnt[i] = 0;
  __syncthreads();
  dstamp(P, 1, 3);
  if (warp < W) {
    int32_t* wc = wcnt + warp * m_e;
    const int b0 = warp * sub, b1 = min(ns, b0 + sub);
    for (int base = b0; base < b1; base += 32) {
      const int i = base + lane;
      const bool ok = i < b1;
      const int rr = ok ? row[i] : -1;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, rr);
      const int leader = __ffs(peers) - 1;
      const int b = ok ? wc[rr] : 0;
      __syncwarp();
      if (ok && lane == leader) wc[rr] = b + __popc(peers);
      __syncwarp();
      if (ok) aux[i] = b + __popc(peers & lt);
    }
  }
  __syncthreads();
  dstamp(P, 1, 4);
  int32_t* tot = P.rtot + static_cast<int64_t>(CS) * goff;   // [CS][m_e] this cluster's per-CTA row totals
  for (int q = tid; q < m_e; q += kBThreads) {   // warp prefixes per row; this CTA's row totals
    int run = 0;
    for (int w = 0; w < W; ++w) {
      const int v = wcnt[w * m_e + q];
      wcnt[w * m_e + q] = run;
      run += v;
    }
    tot[static_cast<int64_t>(r) * m_e + q] = run;
  }
  cluster_barrier();                       // all CTAs' row totals are published
  for (int q = tid; q < m_e; q += kBThreads) {   // rows: size over the cluster; earlier CTAs' share
    int size = 0, before = 0;
    for (int c = 0; c < CS; ++c) {
      const int v = ldcg(tot + static_cast<int64_t>(c) * m_e + q);
      if (c < r) before += v;
      size += v;
    }
    rs[q] = size;
    for (int w = 0; w < W; ++w) wcnt[w * m_e + q] += before;
  }
  __syncthreads();
  {                                              // row starts: ordered scan of the row sizes
    const int rper = (m_e + kBThreads - 1) / kBThreads;
    const int r0 = min(m_e, tid * rper), r1 = min(m_e, r0 + rper);
    int sz = 0;
    for (int q = r0; q < r1; ++q) sz += rs[q];
    int total;
    int run = block_excl_scan<kBWarps>(sz, s_scan, &total);
    for (int q = r0; q < r1; ++q) {
      const int v = rs[q];
      rs[q] = run;
      if (r == 0) P.rsl[goff + q] = goff + run;
      run += v;
    }
  }
  __syncthreads();
  for (int i = tid; i < ns; i += kBThreads) {
    const int q = row[i];
    const int pos = goff + rs[q] + wcnt[(i / sub) * m_e + q] + aux[i];
    P.perm[pos] = mem[i];
    P.rowl[pos] = q;
  }
  if (tid == 0 && r == 0) P.expert_rows[e] = m_e;
  dstamp(P, 1, 5);                         // (the exchanges go through global memory: no exit barrier)
}

// ---- K12: the group path — one CTA per expert does K1 + K2 in shared memory -------------------
// CTA e scans the gate map, compacts its expert's copies in ascending copy id (ordered ballots),
// stores each member's composite key (its token's q codes) and inserts the members into a
// shared-memory hash table keyed by the codes alone (the table is private to the expert): the slot
// keeps the smallest member index with that key (= the bucket's first appearance, reading R7) and
// the bucket's size.  Local row ids = ordered prefix count of the first appearances; each member
// reads its row from its slot; row starts = exclusive scan of the sizes in row order; within-row
// ranks by W warps over contiguous member sub-ranges (match_any batches, per-(warp, row) counters,
// prefix over warps), so perm lists each row's members in ascending copy id (reading R8).  No
// global hash table, no cross-CTA round trip, no cluster barrier: the dependent global accesses
// are the gate-map reads, the code gathers and the output stores.  A group whose arrays do not fit
// in shared memory runs the same code on per-group regions of the workspace (global mode).
#ifndef LSHMOE_GTHREADS
#define LSHMOE_GTHREADS 1024   // experiment knob (compile-time): threads of the group kernel's CTA
#endif
constexpr int kGThreads = LSHMOE_GTHREADS;
constexpr int kGWarps = kGThreads / 32;
constexpr int kGRound = 16;              // gate-map entries per thread per compaction round
constexpr int kGroupSmem = 222 * 1024;   // dynamic shared memory of group_kernel (+ 2.2 KB static)

template <bool kS>
__device__ __forceinline__ int gld(const int32_t* p) {   // global mode: L2 (atomics live there)
  if constexpr (kS) return *p;
  else return __ldcg(p);
}
template <bool kS>
__device__ __forceinline__ uint32_t gldu(const uint32_t* p) {
  if constexpr (kS) return *p;
  else return __ldcg(p);
}

// Sum over the CTA (all threads receive it).  s = [kGWarps + 1].
__device__ __forceinline__ int group_sum(int v, int* s) {
  int t;
  block_excl_scan<kGWarps>(v, s, &t);
  return t;
}

// Keys of members [0, n_e): the member's token's q codes packed two per word (KW words); the hash of
// the key goes to aux.  kGB members per thread per batch, all their code loads issued before any is
// used (kGB = 4 covers a 4K-member group in one round trip).
template <bool kS, int kGB, int kKW>
__device__ __forceinline__ void group_keys(const Params& P, int n_e, int KW, const int32_t* mem, uint32_t* key,
                                           int32_t* aux) {
  const int tid = threadIdx.x;
  const int q = P.q, k = P.k;
  const bool even = (q & 1) == 0;           // rows of q int16 are 4-byte aligned: word loads
  for (int j0 = tid; j0 < n_e; j0 += kGB * kGThreads) {
    uint32_t wv[kGB][kKW];
#pragma unroll
    for (int m = 0; m < kGB; ++m) {
      const int j = j0 + m * kGThreads;
      if (j < n_e) {
        const int c = gld<kS>(mem + j);
        const int64_t t = c / k;
        if (even) {
          const uint32_t* kc = reinterpret_cast<const uint32_t*>(P.codes + t * q);
#pragma unroll
          for (int w = 0; w < kKW; ++w)
            if (w < KW) wv[m][w] = __ldg(kc + w);
        } else {
          const uint16_t* kc = reinterpret_cast<const uint16_t*>(P.codes + t * q);
#pragma unroll
          for (int w = 0; w < kKW; ++w)
            if (w < KW) wv[m][w] = static_cast<uint32_t>(__ldg(kc + 2 * w)) |
                                   (2 * w + 1 < q ? static_cast<uint32_t>(__ldg(kc + 2 * w + 1)) << 16 : 0u);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < kGB; ++m) {
      const int j = j0 + m * kGThreads;
      if (j < n_e) {
        uint32_t h = 0x9E3779B9u;
#pragma unroll
        for (int w = 0; w < kKW; ++w)
          if (w < KW) {
            key[static_cast<int64_t>(j) * KW + w] = wv[m][w];
            h = fmix32(h ^ (wv[m][w] + 0x632BE5ABu * static_cast<uint32_t>(w + 1)));
          }
        aux[j] = static_cast<int32_t>(h);
      }
    }
  }
}

// mem: the expert's members (copy ids, ascending), n_e of them, in shared memory at g_dsmem[0]
// (smem mode) or in the workspace (global mode).  Shared-memory layout (smem mode):
// [mem n_e][slot n_e][aux n_e][rs n_e][fa T][free] — 16 B per member + 4 B per table slot; the
// keys live in the workspace (read only by a warp's leader, against a claimed slot's owner), and the
// per-(warp, row) rank counters reuse the table region once the rows are assigned.
template <bool kS>
__device__ void group_body(const Params& P, int e, int n_e, int goff, int T, int KW, int32_t* mem, int* s_scan,
                           bool smem_keys) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int nk = P.nk;
  int32_t *slot, *aux, *fa, *rs, *wc;
  int64_t wc_cap;                           // ints available for the per-(warp, row) counters
  int32_t* b = P.big;
  const int64_t N = nk;
  uint32_t* key = reinterpret_cast<uint32_t*>(b + 5 * N) + static_cast<int64_t>(goff) * KW;
  if constexpr (kS) {
    int32_t* sm = reinterpret_cast<int32_t*>(g_dsmem);
    slot = sm + n_e;
    aux = slot + n_e;
    rs = aux + n_e;
    fa = rs + n_e;
    if (smem_keys) key = reinterpret_cast<uint32_t*>(fa + T);   // [key n_e x KW] after the table
    wc = fa;                                // after the rows are assigned (table and keys are free)
    wc_cap = P.dyn_smem / 4 - (wc - sm);
  } else {                                  // per-group regions of the workspace's big arrays
    slot = b + N + goff;
    aux = b + 2 * N + goff;
    rs = b + 3 * N + goff;
    fa = b + 13 * N + 4 * static_cast<int64_t>(goff);   // T <= 4 n_e in global mode
    wc = b + 21 * N + 16 * static_cast<int64_t>(goff);  // 16 warps x m_e <= 16 n_e
    wc_cap = 16ll * n_e;
  }
  if (P.permute) {                          // baseline: slot = group offset + rank in the group
    for (int j = tid; j < n_e; j += kGThreads) {
      const int c = gld<kS>(mem + j);
      P.bucket[c] = goff + j;
      P.rowl[goff + j] = c;
    }
    if (tid == 0) {
      P.expert_rows[e] = n_e;
      P.gofs[e] = goff;
    }
    return;
  }
  for (int i = tid; i < T; i += kGThreads) fa[i] = -1;
  // keys: the member's token's q codes packed two per word (workspace); the hash goes to aux.
  // kGB members per thread per batch, all their code loads issued before any is used.
  if (KW <= 4) group_keys<kS, 4, 4>(P, n_e, KW, mem, key, aux);   // q <= 8: 4 members' loads in flight
  else group_keys<kS, 2, kMaxQ / 2>(P, n_e, KW, mem, key, aux);
  dstamp(P, 1, 6);                          // diagnostics: thread 0's keys stored
  __syncthreads();                          // every key is stored before any slot is claimed
  dstamp(P, 1, 1);
  // insert: a slot's value converges (atomicMin) to the smallest member index with its key (a
  // claimed slot never changes key); a plain read first keeps claimed slots free of CAS traffic
  for (int j = tid; j < n_e; j += kGThreads) {
    uint32_t kw[kMaxQ / 2];
#pragma unroll
    for (int w = 0; w < kMaxQ / 2; ++w)
      if (w < KW) kw[w] = key[static_cast<int64_t>(j) * KW + w];
    int sl = static_cast<int>(static_cast<uint32_t>(gld<kS>(aux + j)) & static_cast<uint32_t>(T - 1));
    while (true) {
      int cur = gld<kS>(fa + sl);
      if (cur < 0) {
        cur = atomicCAS(fa + sl, -1, j);
        if (cur < 0) break;
      }
      bool eq = true;
#pragma unroll
      for (int w = 0; w < kMaxQ / 2; ++w)
        if (w < KW) eq &= key[static_cast<int64_t>(cur) * KW + w] == kw[w];
      if (eq) {
        if (j < cur) atomicMin(fa + sl, j);
        break;
      }
      sl = (sl + 1) & (T - 1);
    }
    slot[j] = sl;
  }
  __syncthreads();
  dstamp(P, 1, 2);
  for (int j0 = tid; j0 < n_e; j0 += 4 * kGThreads) {   // first?  (4 members' loads in flight)
    int sv[4], fv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) sv[m] = j0 + m * kGThreads < n_e ? gld<kS>(slot + j0 + m * kGThreads) : 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) fv[m] = j0 + m * kGThreads < n_e ? gld<kS>(fa + sv[m]) : 0;
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (j0 + m * kGThreads < n_e) aux[j0 + m * kGThreads] = fv[m] == j0 + m * kGThreads ? 1 : 0;
  }
  __syncthreads();
  // local row ids of the first appearances in member order (contiguous chunks per thread); the
  // slot's fa becomes the row id (every first-flag read is done)
  int m_e;
  {
    const int L = (n_e + kGThreads - 1) / kGThreads;
    const int j0 = min(n_e, tid * L), j1 = min(n_e, j0 + L);
    int nf = 0;
    for (int j = j0; j < j1; ++j) nf += gld<kS>(aux + j);
    int id = block_excl_scan<kGWarps>(nf, s_scan, &m_e);
    for (int j = j0; j < j1; ++j)
      if (gld<kS>(aux + j)) fa[gld<kS>(slot + j)] = id++;
  }
  __syncthreads();
  for (int j0 = tid; j0 < n_e; j0 += 4 * kGThreads) {   // slot -> row
    int sv[4], fv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) sv[m] = j0 + m * kGThreads < n_e ? gld<kS>(slot + j0 + m * kGThreads) : 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) fv[m] = j0 + m * kGThreads < n_e ? gld<kS>(fa + sv[m]) : 0;
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (j0 + m * kGThreads < n_e) slot[j0 + m * kGThreads] = fv[m];
  }
  __syncthreads();                          // the table is free: the rank counters take its place
  dstamp(P, 1, 3);
  // within-row ranks: W warps own contiguous member sub-ranges, per-(warp, row) counters
  int W = static_cast<int>(min(static_cast<int64_t>(kGWarps), wc_cap / max(m_e, 1)));
  if (W < 1) W = 1;
  const int sub = (((n_e + W - 1) / W) + 31) & ~31;
  for (int i = tid; i < W * m_e; i += kGThreads) wc[i] = 0;
  __syncthreads();
  if (warp < W) {
    int32_t* w_c = wc + static_cast<int64_t>(warp) * m_e;
    const int b0 = min(n_e, warp * sub), b1 = min(n_e, b0 + sub);
    for (int bb = b0; bb < b1; bb += 32) {
      const int i = bb + lane;
      const bool ok = i < b1;
      const int rr = ok ? gld<kS>(slot + i) : -1;
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, rr);
      const int leader = __ffs(peers) - 1;
      const int cv = ok ? gld<kS>(w_c + rr) : 0;
      __syncwarp();
      if (ok && lane == leader) w_c[rr] = cv + __popc(peers);
      __syncwarp();
      if (ok) aux[i] = cv + __popc(peers & lt);
    }
  }
  __syncthreads();
  for (int r = tid; r < m_e; r += kGThreads) {   // prefix over warps per row; the total = row size
    int run = 0;
    for (int w = 0; w < W; ++w) {
      const int v = gld<kS>(wc + static_cast<int64_t>(w) * m_e + r);
      wc[static_cast<int64_t>(w) * m_e + r] = run;
      run += v;
    }
    rs[r] = run;
  }
  __syncthreads();
  {                                         // row starts: ordered exclusive scan of the sizes
    const int L = (m_e + kGThreads - 1) / kGThreads;
    const int r0 = min(m_e, tid * L), r1 = min(m_e, r0 + L);
    int sz = 0;
    for (int r = r0; r < r1; ++r) sz += gld<kS>(rs + r);
    int tot;
    int run = block_excl_scan<kGWarps>(sz, s_scan, &tot);
    for (int r = r0; r < r1; ++r) {
      const int v = gld<kS>(rs + r);
      rs[r] = run;
      P.rsl[goff + r] = goff + run;
      run += v;
    }
  }
  __syncthreads();
  dstamp(P, 1, 4);
  for (int j0 = tid; j0 < n_e; j0 += 4 * kGThreads) {   // 4 members' loads in flight
    int rv[4], pv[4], cv[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int j = j0 + m * kGThreads;
      rv[m] = j < n_e ? gld<kS>(slot + j) : 0;
      cv[m] = j < n_e ? gld<kS>(mem + j) : 0;
      pv[m] = j < n_e ? gld<kS>(aux + j) : 0;
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int j = j0 + m * kGThreads;
      if (j < n_e) pv[m] += gld<kS>(rs + rv[m]) + gld<kS>(wc + static_cast<int64_t>(j / sub) * m_e + rv[m]);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (j0 + m * kGThreads < n_e) {
        P.perm[goff + pv[m]] = cv[m];
        P.rowl[goff + pv[m]] = rv[m];
      }
  }
  if (tid == 0) {
    P.expert_rows[e] = m_e;
    P.gofs[e] = goff;
  }
}

// Ordered compaction of expert e's copies (ascending copy id) into mem[0, cap): rounds of
// kGRound x 1024 gate-map entries, entry c = r0 + u * 1024 + tid, so (u, warp, lane) is ascending
// copy order within a round; the next round's entries are loaded before this round's scan.
// Returns n_e; *clt = copies of experts < e (invalid ids count as expert 0).  Ids outside [0, E)
// in [c0, c1) raise error bit 0.
__device__ int group_compact(const Params& P, int e, int32_t* mem, int cap, int c0, int c1, int* s_scan, int* s_cnt,
                             int* clt_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int nk = P.nk, E = P.E;
  int base = 0, clt = 0;
  int v[kGRound];
#pragma unroll
  for (int u = 0; u < kGRound; ++u) v[u] = u * kGThreads + tid < nk ? P.experts[u * kGThreads + tid] : 0x7FFFFFFF;
  for (int r0 = 0; r0 < nk; r0 += kGRound * kGThreads) {
    unsigned bl[kGRound];
#pragma unroll
    for (int u = 0; u < kGRound; ++u) {
      const int c = r0 + u * kGThreads + tid;
      int x = v[u];
      if (c < nk && static_cast<unsigned>(x) >= static_cast<unsigned>(E)) {
        if (c >= c0 && c < c1) atomicOr(&g_device_error, 1);
        x = 0;
      }
      clt += x < e;
      bl[u] = __ballot_sync(0xFFFFFFFFu, x == e);
      if (lane == 0) s_cnt[u * kGWarps + warp] = __popc(bl[u]);
    }
    if (r0 + kGRound * kGThreads < nk)      // the next round's entries, in flight during the scan
#pragma unroll
      for (int u = 0; u < kGRound; ++u) {
        const int c = r0 + kGRound * kGThreads + u * kGThreads + tid;
        v[u] = c < nk ? P.experts[c] : 0x7FFFFFFF;
      }
    __syncthreads();
    constexpr int kEnt = kGRound * kGWarps;   // 512 (u, warp) counts, scanned in (u, warp) order
    const int x = tid < kEnt ? s_cnt[tid] : 0;
    int tot;
    const int ex = block_excl_scan<kGWarps>(x, s_scan, &tot);
    if (tid < kEnt) s_cnt[tid] = ex;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kGRound; ++u)
      if ((bl[u] >> lane) & 1u) {
        const int pos = base + s_cnt[u * kGWarps + warp] + __popc(bl[u] & lt);
        if (pos < cap) mem[pos] = r0 + u * kGThreads + tid;
      }
    base += tot;
    __syncthreads();                        // s_cnt is rewritten by the next round
  }
  *clt_out = clt;
  return base;
}

__global__ void __launch_bounds__(kGThreads, 1) group_kernel(Params P) {
  __shared__ int s_scan[kGWarps + 1];
  __shared__ int s_cnt[kGRound * kGWarps];
  const int tid = threadIdx.x;
  const int e = blockIdx.x, E = P.E, nk = P.nk;
  // The gate map is an input of the step, complete before the hash kernel started (early_gate):
  // its validation and compaction (shared memory only, no global writes but the error word) run
  // while the hash kernel's last CTAs finish; the codes are read only after griddepcontrol.wait.
  if (!P.early_gate) pdl_wait();            // lshmoe_gate_hash wrote the gate map: wait first
  pdl_trigger();
  dstamp(P, 1, 0);
  // this CTA validates the copies [c0, c1): ids in [0, E) (bit 0, in the compaction pass) and,
  // for k > 1, distinct within a token (bit 1)
  const int c0 = static_cast<int>(static_cast<int64_t>(e) * nk / E);
  const int c1 = static_cast<int>(static_cast<int64_t>(e + 1) * nk / E);
  if (P.k > 1)
    for (int c = c0 + tid; c < c1; c += kGThreads) {
      const int v = P.experts[c], sl = c % P.k;
      for (int s2 = 0; s2 < sl; ++s2)
        if (P.experts[c - sl + s2] == v) atomicOr(&g_device_error, 2);
    }
  // one pass over the gate map: the members into shared memory (as many as fit), n_e, goff
  int32_t* sm = reinterpret_cast<int32_t*>(g_dsmem);
  const int cap = P.dyn_smem / 4;
  int clt;
  const int n_e = group_compact(P, e, sm, cap, c0, c1, s_scan, s_cnt, &clt);
  const int goff = group_sum(clt, s_scan);
  if (P.early_gate) pdl_wait();             // the hash kernel's codes are complete and visible
  dstamp(P, 1, 7);
  const int KW = (P.q + 1) / 2;
  int T = 64;
  while (T < n_e + n_e / 2) T <<= 1;        // load factor <= 2/3
  const int64_t need = P.permute ? 4ll * n_e : 16ll * n_e + 4ll * T;
  if (need <= P.dyn_smem) {                 // the keys too when they fit (else in the workspace)
    const bool sk = !P.permute && need + 4ll * KW * n_e <= P.dyn_smem;
    group_body<true>(P, e, n_e, goff, T, KW, sm, s_scan, sk);
  } else {                                  // global mode: the members move to the workspace
    while (T < 2 * n_e) T <<= 1;
    int32_t* gm = P.big + goff;
    if (n_e <= cap) {
      for (int j = tid; j < n_e; j += kGThreads) gm[j] = sm[j];
    } else {
      int dummy;
      group_compact(P, e, gm, n_e, 0, 0, s_scan, s_cnt, &dummy);
    }
    __syncthreads();
    group_body<false>(P, e, n_e, goff, T, KW, gm, s_scan, false);
  }
  dstamp(P, 1, 5);
}



// ---- centroid phase ------------------------------------------------------------------------
// CTA b owns the perm range [b*nk/G, (b+1)*nk/G), split again into one contiguous sub-range per
// warp, so eight segments (centroid rows) are reduced at once and the per-row boundary logic is
// warp-uniform.  Each lane prefetches its own 16-byte column chunks of the warp's next rows into
// a per-warp shared-memory ring with cp.async, kB rows per commit group and kNB groups in flight
// (a lane only ever reads what it copied, so no barrier is needed); a batch's chunks are loaded
// into registers at once and summed in perm order in fp32.  Rows cut by warp boundaries are
// combined by the first warp holding them (warp order); rows cut by the CTA range leave fp32
// partials (slot 0 = the range's first segment, slot 1 = its last) that fixup_phase adds in CTA
// order.  Columns are processed in blocks of 128 chunks (2 KB of a row) to bound registers.
constexpr int kBlkChunks = 128;          // 16-byte chunks per column block
constexpr int kCPL = kBlkChunks / 32;    // chunks per lane per block
// Centroid-phase CTA shape: kCWarps warps (LSHMOE_CWARPS, 8 or 16); the per-warp rings shrink with
// more warps so the shared memory per SM stays within budget.  16 warps (one 512-thread CTA per SM)
// hide more of the gathers' and the ring reads' latency: compress per call (scripts/compress_diag.py)
// C2 39.4 -> 37.6 us, C3 93.3 -> 85.3, C4 ~98 -> 92.0 (centroid spans C2 19.5 -> 17.3, C3 57.4 -> 45.7,
// C4 55 -> 45.8 us).
#ifndef LSHMOE_CWARPS
#define LSHMOE_CWARPS 16
#endif
static_assert(LSHMOE_CWARPS == 8 || LSHMOE_CWARPS == 16, "centroid warps: 8 or 16");
constexpr int kCWarps = LSHMOE_CWARPS;
#ifndef LSHMOE_CGRID
#define LSHMOE_CGRID 1   // experiment: centroid CTAs per SM (2 with 8 warps and 8 KB rings)
#endif
constexpr int kCPerSM = LSHMOE_CGRID;
constexpr int kCThreads = 32 * kCWarps;
constexpr int kRingSlot = 16 * kBlkChunks;
constexpr int kWpartFloats = kBlkChunks * 8;   // one warp partial slot (fp32, up to 8 per chunk)
constexpr int kQ = kCWarps == 8 ? 10 : 4;   // ring rows per warp at the largest (2 KB) slot (16 warps:
                                            // the slot-0 partials double, so the rings shrink more)
#ifndef LSHMOE_CRING
#define LSHMOE_CRING 0   // experiment: ring bytes per warp (0: kQ 2 KB slots)
#endif
constexpr int kRingWarp = LSHMOE_CRING ? LSHMOE_CRING : kQ * kRingSlot;   // ring bytes per warp; slots are packed at 16*ncb bytes,
                                            // so short rows get a deeper ring (1.5 KB rows: 13 slots)
static_assert(kWpartFloats * 4 <= kRingWarp, "a warp's slot-1 partial reuses its ring");
// ring rows per warp for CPL chunks per lane (slots packed at CPL * 512 bytes), at most 16
constexpr int ring_depth(int cpl) { return kRingWarp / (cpl * 512) < 16 ? kRingWarp / (cpl * 512) : 16; }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {   // at most N of this thread's groups pending
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename T>
__device__ __forceinline__ void add_chunk16(float* acc, uint4 raw) {
  if (sizeof(T) == 2) {
    const uint32_t u[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] += __uint_as_float(u[i] << 16);
      acc[2 * i + 1] += __uint_as_float(u[i] & 0xFFFF0000u);
    }
  } else {
    acc[0] += __uint_as_float(raw.x);
    acc[1] += __uint_as_float(raw.y);
    acc[2] += __uint_as_float(raw.z);
    acc[3] += __uint_as_float(raw.w);
  }
}

template <typename T>
__device__ __forceinline__ void add_chunk16_w(float* acc, uint4 raw, float w) {   // acc += w * x (one rounding)
  if (sizeof(T) == 2) {
    const uint32_t u[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] = fmaf(w, __uint_as_float(u[i] << 16), acc[2 * i]);
      acc[2 * i + 1] = fmaf(w, __uint_as_float(u[i] & 0xFFFF0000u), acc[2 * i + 1]);
    }
  } else {
    acc[0] = fmaf(w, __uint_as_float(raw.x), acc[0]);
    acc[1] = fmaf(w, __uint_as_float(raw.y), acc[1]);
    acc[2] = fmaf(w, __uint_as_float(raw.z), acc[2]);
    acc[3] = fmaf(w, __uint_as_float(raw.w), acc[3]);
  }
}

template <int VC>
__device__ __noinline__ void store_f32_copy(float* dst, const float* v) {   // tier-2 parity output only
#pragma unroll
  for (int e = 0; e < VC; ++e) dst[e] = v[e];
}

// centroid = acc * rc, rc = RN(1/count) (reading R10), RNE to the wire dtype; fp32 copy if requested.
template <typename T, bool kF = false>
__device__ __forceinline__ void store_chunk16(const Params& P, int row, int c16, const float* acc, float rc,
                                              uint8_t* fdst = nullptr) {
  constexpr int VC = 16 / sizeof(T);
  float v[VC];
#pragma unroll
  for (int e = 0; e < VC; ++e) v[e] = acc[e] * rc;
  uint4 out;
  if (sizeof(T) == 2) {
    uint32_t u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      u[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    out = make_uint4(u[0], u[1], u[2], u[3]);
  } else {
    out = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
  }
  *reinterpret_cast<uint4*>(P.cent + static_cast<int64_t>(row) * P.row_bytes + 16 * c16) = out;
  if constexpr (kF) {                        // fused dispatch: the row also goes to its owner
    if (fdst) *reinterpret_cast<uint4*>(fdst + 16 * c16) = out;
  }
  if (P.cent32) store_f32_copy<VC>(P.cent32 + static_cast<int64_t>(row) * P.d + c16 * VC, v);
}

template <typename T>
__device__ __forceinline__ void add_chunk8(float* acc, uint2 raw) {
  if (sizeof(T) == 2) {
    acc[0] += __uint_as_float(raw.x << 16);
    acc[1] += __uint_as_float(raw.x & 0xFFFF0000u);
    acc[2] += __uint_as_float(raw.y << 16);
    acc[3] += __uint_as_float(raw.y & 0xFFFF0000u);
  } else {
    acc[0] += __uint_as_float(raw.x);
    acc[1] += __uint_as_float(raw.y);
  }
}

// centroid = acc * RN(1/count) (reading R10), RNE to the wire dtype; fp32 copy if requested.
template <typename T, bool kF = false>
__device__ __forceinline__ void store_chunk8(const Params& P, int row, int ch, const float* acc, float cnt,
                                             uint8_t* fdst = nullptr) {
  constexpr int VC = sizeof(T) == 2 ? 4 : 2;
  const float rc = P.grad ? 1.0f : __frcp_rn(cnt);
  float v[VC];
#pragma unroll
  for (int e = 0; e < VC; ++e) v[e] = acc[e] * rc;
  uint2 out;
  if (sizeof(T) == 2) {
    __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 h1 = __floats2bfloat162_rn(v[2], v[3]);
    out = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
  } else {
    out = make_uint2(__float_as_uint(v[0]), __float_as_uint(v[1]));
  }
  *reinterpret_cast<uint2*>(P.cent + static_cast<int64_t>(row) * P.row_bytes + 8 * ch) = out;
  if constexpr (kF) {
    if (fdst) *reinterpret_cast<uint2*>(fdst + 8 * ch) = out;
  }
  if (P.cent32) {
    float* dst = P.cent32 + static_cast<int64_t>(row) * P.d + ch * VC;
#pragma unroll
    for (int e = 0; e < VC; ++e) dst[e] = v[e];
  }
}

// 32-bit divisions whenever the product fits (a 64-bit division is ~4x the instructions)
__device__ __forceinline__ int range_begin(int b, int nk, int G) {
  const uint64_t prod = static_cast<uint64_t>(b) * static_cast<uint32_t>(nk);
  return prod >> 32 ? static_cast<int>(prod / static_cast<uint32_t>(G))
                    : static_cast<int>(static_cast<uint32_t>(prod) / static_cast<uint32_t>(G));
}
__device__ __forceinline__ int range_cta(int p, int nk, int G) {   // CTA whose range holds p
  const uint64_t prod = static_cast<uint64_t>(p + 1) * static_cast<uint32_t>(G) - 1;
  return prod >> 32 ? static_cast<int>(prod / static_cast<uint32_t>(nk))
                    : static_cast<int>(static_cast<uint32_t>(prod) / static_cast<uint32_t>(nk));
}

// Dynamic shared memory of compress_kernel, named at file scope so that the centroid phase's
// addresses stay in the shared window (no generic-to-shared conversion per access).
extern __shared__ __align__(1024) uint8_t g_dsmem[];

// Centroid-phase shared memory: [warp][kQ][kRingSlot] rings | [warp][kWpartFloats] slot-0
// partials | rows[p_begin-1 .. p_end] | tok[p_begin .. p_end).
struct CentroidCtx {                     // one CTA's view of its perm range (centroid phase)
  int p_begin, p_end, range, w, lane, w_begin, w_end, tok_off;
  uint32_t prev_row;                     // row of entry w_begin - 1
  int cut_rs, cut_re;                    // threads 0 / 1: perm extent of the range's first / last row
  __device__ uint8_t* ring() const { return g_dsmem + w * kRingWarp; }
  __device__ float* slot0() const { return reinterpret_cast<float*>(g_dsmem + kCWarps * kRingWarp); }
  __device__ uint32_t* s_row() const { return reinterpret_cast<uint32_t*>(slot0() + kCWarps * kWpartFloats); }
  __device__ int32_t* s_tok() const { return reinterpret_cast<int32_t*>(s_row()) + tok_off; }
  __device__ float* s_wt(int max_range) const { return reinterpret_cast<float*>(s_tok()) + max_range; }
  __device__ uint32_t row_at(int p) const { return s_row()[p - p_begin + 1]; }
  __device__ int wbeg(int ww) const { return p_begin + range_begin(ww, range, kCWarps); }
  __device__ float* wpart(int ww, int slot) const {   // slot 0: own region; slot 1: the warp's ring
    return slot == 0 ? slot0() + ww * kWpartFloats : reinterpret_cast<float*>(g_dsmem + ww * kRingWarp);
  }
};

// One column block (chunks [c0, c0 + ncb), CPL = ceil(ncb / 32) chunks per lane) of the centroid
// phase: stream the warp's rows through its ring, reduce segments, then combine cut rows.
template <typename T, int CPL, int QD = kQ, bool kF = false>
__device__ void centroid_block(const Params& P, const CentroidCtx& X, int cb, int c0, int ncb) {
  const int slotB = 16 * CPL * 32;           // packed ring slot (this block's row bytes, rounded to a lane round)
  constexpr int VC = 16 / sizeof(T);
  const int lane = X.lane, w = X.w, w_begin = X.w_begin, w_end = X.w_end;
  const bool full = ncb == CPL * 32;
  auto issue = [&](int p, int slot) {
    if (p < w_end) {
      const uint8_t* src = P.x + static_cast<int64_t>(X.s_tok()[p - X.p_begin]) * P.row_bytes + 16 * c0;
      uint8_t* dst = X.ring() + slot * slotB;
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = lane + 32 * t;
        if (full || c < ncb) cp_async16(dst + 16 * c, src + 16 * c);
      }
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int i = 0; i < QD - 1; ++i) issue(w_begin + i, i);
  float acc[CPL][VC];
#pragma unroll
  for (int t = 0; t < CPL; ++t)
#pragma unroll
    for (int e = 0; e < VC; ++e) acc[t][e] = 0.0f;
  int seg_start = w_begin, rd = 0, wr = QD - 1;   // ring slots: next to read, next to fill
  uint32_t row = w_end > w_begin ? X.row_at(w_begin) : 0u;
#pragma unroll 1
  for (int p = w_begin; p < w_end; ++p) {
    issue(p + QD - 1, wr);
    wr = wr + 1 == QD ? 0 : wr + 1;
    cp_async_wait<QD - 1>();                  // entry p (this lane's chunks) has landed
    if (p == w_begin && cb == 0 && X.w == 0) dstamp(P, 2, 4);   // diagnostics: first row landed
    const uint8_t* st = X.ring() + rd * slotB;
    rd = rd + 1 == QD ? 0 : rd + 1;
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int c = lane + 32 * t;
      if (full || c < ncb) {
        if (P.gw) add_chunk16_w<T>(acc[t], *reinterpret_cast<const uint4*>(st + 16 * c), X.s_wt(P.max_range)[p - X.p_begin]);
        else add_chunk16<T>(acc[t], *reinterpret_cast<const uint4*>(st + 16 * c));
      }
    }
    const uint32_t next = X.row_at(p + 1);
    if (next == row && p + 1 < w_end) continue;         // the segment goes on
    const bool head = seg_start > w_begin || X.prev_row != row;   // the row starts in this warp
    if (head && next != row) {                // the whole row lies in this warp's sub-range
      const float rc = P.grad ? 1.0f : __frcp_rn(static_cast<float>(p + 1 - seg_start));
      uint8_t* fdst = nullptr;
      if constexpr (kF) fdst = fused_row_dst(P, static_cast<int>(row));   // owner row, once per row
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = lane + 32 * t;
        if (full || c < ncb) store_chunk16<T, kF>(P, static_cast<int>(row), c0 + c, acc[t], rc, fdst);
      }
    } else if (p + 1 == w_end) {
      break;                                  // the last segment stays in acc (partial, see below)
    } else {                                  // the first segment, begun in an earlier warp
      float* d0 = X.wpart(w, 0);
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = lane + 32 * t;
        if (full || c < ncb)
#pragma unroll
          for (int e = 0; e < VC; ++e) d0[c * VC + e] = acc[t][e];
      }
    }
#pragma unroll
    for (int t = 0; t < CPL; ++t)
#pragma unroll
      for (int e = 0; e < VC; ++e) acc[t][e] = 0.0f;
    seg_start = p + 1;
    row = next;
  }
  cp_async_wait<0>();                         // this lane's copies have landed ...
  __syncwarp();                               // ... and every lane's: the ring may hold the slot-1 partial
                                              // (a lane's partial overlays bytes other lanes copied;
                                              // compute-sanitizer racecheck r2)
  if (cb == 0 && X.w == 0) dstamp(P, 2, 5);   // diagnostics: warp 0's rows reduced
  const int nrows = w_end - w_begin;
  const uint32_t r_last = X.row_at(w_end - 1);
  const bool cut_end = nrows > 0 && X.row_at(w_end) == r_last;
  const bool from_before = nrows > 0 && seg_start == w_begin && X.prev_row == r_last;   // began in an earlier warp
  if (cut_end || from_before) {
    float* d1 = X.wpart(w, seg_start == w_begin ? 0 : 1);
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int c = lane + 32 * t;
      if (full || c < ncb)
#pragma unroll
        for (int e = 0; e < VC; ++e) d1[c * VC + e] = acc[t][e];
    }
  }
  __syncthreads();                            // every warp's pieces are in wpart
  // Combine the rows cut by warp boundaries; warp w owns a cut row whose first entry in this
  // CTA lies in its sub-range.  lo = that entry; hi = one past the row's last entry in the CTA.
  auto own = [&](uint32_t r, int lo) {
    int a = lo + 1, z = X.p_end;              // rows are sorted: first entry in (lo, p_end] != r
    while (a < z) {
      const int mid = (a + z) / 2;
      if (X.row_at(mid) == r) a = mid + 1; else z = mid;
    }
    const int hi = a;
    const int wl = range_cta(hi - 1 - X.p_begin, X.range, kCWarps);
    const bool before = lo == X.p_begin && X.row_at(X.p_begin - 1) == r;
    const bool after = hi == X.p_end && X.row_at(X.p_end) == r;
    const float rc = P.grad ? 1.0f : __frcp_rn(static_cast<float>(hi - lo));
    uint8_t* fdst = nullptr;
    if constexpr (kF)
      if (!(before || after)) fdst = fused_row_dst(P, static_cast<int>(r));   // owner row, once per row
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int c = lane + 32 * t;
      if (!full && c >= ncb) continue;
      float v[VC];
      const float* s0 = X.wpart(w, lo == w_begin ? 0 : 1) + c * VC;
#pragma unroll
      for (int e = 0; e < VC; ++e) v[e] = s0[e];
      for (int ww = w + 1; ww <= wl; ++ww) {
        if (X.wbeg(ww + 1) == X.wbeg(ww)) continue;          // empty sub-range
        const float* s1 = X.wpart(ww, 0) + c * VC;
#pragma unroll
        for (int e = 0; e < VC; ++e) v[e] += s1[e];
      }
      if (before || after) {
        float* dst = P.partial + (static_cast<int64_t>(blockIdx.x) * 2 + (lo == X.p_begin ? 0 : 1)) * P.d + (c0 + c) * VC;
#pragma unroll
        for (int e = 0; e < VC; ++e) dst[e] = v[e];
      } else {
        store_chunk16<T, kF>(P, static_cast<int>(r), c0 + c, v, rc, fdst);
      }
    }
  };
  if (nrows > 0) {
    const bool first_w = w == range_cta(0, X.range, kCWarps);   // first non-empty sub-range of the CTA
    if (cut_end && (first_w || !from_before)) own(r_last, seg_start);
    if (first_w) {                            // the CTA's first row, begun in an earlier CTA
      const uint32_t r0 = X.row_at(X.p_begin);
      if (X.prev_row == r0 && !(r0 == r_last && cut_end)) own(r0, X.p_begin);
    }
  }
  __syncthreads();                            // the ring is reused by the next column block
}

// Expert whose perm range holds position p (s_goff[e] <= p < s_goff[e + 1]).
__device__ __forceinline__ int expert_at(const int* s_goff, int E, int p) {
  int lo = 0, hi = E - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_goff[mid] <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Threads 0 and 1 load the perm extents [rs, re) of the range's first and last rows right after
// the index fill, so the loads are in flight during the reduction (used by merge_cut_rows).
__device__ __forceinline__ void prefetch_cut_extent(const Params& P, CentroidCtx& X, const int* s_goff,
                                                    const int* s_mrow, const int* s_cut) {
  const int which = threadIdx.x;
  if (which >= 2) return;
  if (P.grad) {                               // row extents straight from the forward's row_start
    const uint32_t r = X.row_at(which == 0 ? X.p_begin : X.p_end - 1);
    X.cut_rs = ldcg(P.row_start + r);
    X.cut_re = ldcg(P.row_start + r + 1);
  } else {
    const int e = s_cut[2 * which], lr = s_cut[2 * which + 1];
    X.cut_rs = ldcg(P.rsl + s_goff[e] + lr);
    X.cut_re = lr + 1 < s_mrow[e] ? ldcg(P.rsl + s_goff[e] + lr + 1) : s_goff[e + 1];
  }
}

// The index entries i = tid + kCThreads u (u < kPre) of a CTA's range, loaded right after the
// kernel's dependency wait so that their latency overlaps the expert-count scan.
constexpr int kPre = 4;
struct IndexPre {
  int l[kPre], c[kPre];
};
__device__ __forceinline__ void preload_index(const Params& P, IndexPre& pre) {
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int pb = range_begin(b, P.nk, G), range = range_begin(b + 1, P.nk, G) - pb;
#pragma unroll
  for (int u = 0; u < kPre; ++u) {
    const int i = tid + kCThreads * u, p = pb - 1 + i;
    pre.l[u] = 0;
    pre.c[u] = 0;
    if (i < range + 2 && p >= 0 && p < P.nk) {
      pre.l[u] = ldcg(P.rowl + p);
      if (i >= 1 && i <= range) pre.c[u] = ldcg(P.perm + p);
    }
  }
}

// Phase B of one CTA: its perm range's rows (global ids = row offset of the expert + local row),
// token ids and bucket outputs, then the centroid reduction.  s_cut[0..1] receive the (expert,
// local row) of the range's first and last entries for the cut-row merge.
template <typename T, bool kF = false>
__device__ __forceinline__ void centroid_phase(const Params& P, const int* s_goff, const int* s_roff, const int* s_mrow,
                                               int* s_cut, CentroidCtx& X, const IndexPre& pre) {
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  X.p_begin = range_begin(b, P.nk, G);
  X.p_end = range_begin(b + 1, P.nk, G);
  X.range = X.p_end - X.p_begin;
  if (X.range == 0) return;                   // CTA-uniform
  X.lane = tid % 32;
  X.w = tid / 32;
  X.tok_off = P.max_range + 2;
  uint32_t* s_row = X.s_row();
  int32_t* s_tok = X.s_tok();
#pragma unroll 1
  for (int i = tid, u = 0; i < X.range + 2; i += kCThreads, ++u) {
    const int p = X.p_begin - 1 + i;
    uint32_t row = 0xFFFFFFFFu;
    if (p >= 0 && p < P.nk) {
      const int e = expert_at(s_goff, P.E, p);
      int lr, c = 0;
      if (u < kPre) {                        // preloaded (registers, static indices)
        lr = u == 0 ? pre.l[0] : u == 1 ? pre.l[1] : u == 2 ? pre.l[2] : pre.l[3];
        c = u == 0 ? pre.c[0] : u == 1 ? pre.c[1] : u == 2 ? pre.c[2] : pre.c[3];
      } else {
        lr = ldcg(P.rowl + p);
        if (i >= 1 && i <= X.range) c = ldcg(P.perm + p);
      }
      row = static_cast<uint32_t>(s_roff[e] + lr);
      if (i >= 1 && i <= X.range) {
        s_tok[i - 1] = c / P.k;
        P.bucket[c] = static_cast<int32_t>(row);
        if (i == 1) { s_cut[0] = e; s_cut[1] = lr; }
        if (i == X.range) { s_cut[2] = e; s_cut[3] = lr; }
      }
    }
    s_row[i] = row;
  }
  __syncthreads();
  dstamp(P, 2, 1);
  prefetch_cut_extent(P, X, s_goff, s_mrow, s_cut);
  X.w_begin = X.wbeg(X.w);
  X.w_end = X.wbeg(X.w + 1);
  X.prev_row = X.row_at(X.w_begin - 1);
  for (int c0 = 0, cb = 0; c0 < P.nch; c0 += kBlkChunks, ++cb) {
    const int ncb = min(kBlkChunks, P.nch - c0);
    switch ((ncb + 31) / 32) {
      case 1: centroid_block<T, 1, ring_depth(1), kF>(P, X, cb, c0, ncb); break;
      case 2: centroid_block<T, 2, ring_depth(2), kF>(P, X, cb, c0, ncb); break;
      case 3: centroid_block<T, 3, ring_depth(3), kF>(P, X, cb, c0, ncb); break;
      default: centroid_block<T, 4, ring_depth(4), kF>(P, X, cb, c0, ncb); break;
    }
  }
}

// Rows cut by CTA ranges: each CTA holding a piece publishes its fp32 partial (centroid_block),
// then arrives on the counter of the CTA where the row starts; the last arriver adds the
// partials in CTA order (the same order whichever CTA arrives last) and stores the centroid.
#ifndef LSHMOE_MERGE_BATCH
#define LSHMOE_MERGE_BATCH 8
#endif
constexpr int kMergeBatch = LSHMOE_MERGE_BATCH;   // partials of a cut row loaded before any is added

template <typename T, bool kF = false>
__device__ void merge_cut_rows(const Params& P, const CentroidCtx& X, const int* s_goff, const int* s_mrow,
                               const int* s_cut, int* s_job) {
  constexpr int VC = sizeof(T) == 2 ? 4 : 2;
  const int G = gridDim.x, tid = threadIdx.x;
  if (X.range == 0) return;
  __syncthreads();                            // the CTA's partial writes precede the arrivals (bar.sync),
  if (tid < 2) {                              // and the arriving thread's release is cumulative
    // thread `which` handles one candidate row
    const int which = tid;
    s_job[4 * which] = -1;
    const uint32_t r0 = X.row_at(X.p_begin), rl = X.row_at(X.p_end - 1);
    const bool before = X.row_at(X.p_begin - 1) == r0;
    const bool after = X.row_at(X.p_end) == rl;
    const bool cand = which == 0 ? before : (after && !(before && rl == r0));
    if (cand) {
      const int rs = X.cut_rs, re = X.cut_re;
      const int b0 = range_cta(rs, P.nk, G), b1 = range_cta(re - 1, P.nk, G);
      int expected = b1 - b0 + 1;             // every range is non-empty when nk >= G
      if (P.nk < G) {
        expected = 0;
        for (int bb = b0; bb <= b1; ++bb) expected += range_begin(bb + 1, P.nk, G) > range_begin(bb, P.nk, G);
      }
      int old;                                // counters start at -1; acq_rel: publish ours, acquire theirs
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                   : "=r"(old) : "l"(reinterpret_cast<int*>(P.bar) + kArrive + b0) : "memory");
      if (old + 2 == expected) {
        reinterpret_cast<int*>(P.bar)[kArrive + b0] = -1;   // leave the counter at rest for the next call
        s_job[4 * which + 0] = static_cast<int>(which == 0 ? r0 : rl);
        s_job[4 * which + 1] = rs;
        s_job[4 * which + 2] = re;
        s_job[4 * which + 3] = b0 | (b1 << 16);
      }
    }
  }
  __syncthreads();
  for (int j = 0; j < 2; ++j) {
    const int row = s_job[4 * j];
    if (row < 0) continue;
    const int rs = s_job[4 * j + 1], re = s_job[4 * j + 2];
    const int b0 = s_job[4 * j + 3] & 0xFFFF, b1 = s_job[4 * j + 3] >> 16;
    const int nc8 = P.row_bytes / 8;
    const int slot0 = rs == range_begin(b0, P.nk, G) ? 0 : 1;
    const bool all_nonempty = P.nk >= G;
    uint8_t* fdst = nullptr;
    if constexpr (kF) fdst = fused_row_dst(P, row);   // owner row, once per merged row
    for (int ch = tid; ch < nc8; ch += kCThreads) {
      float acc[VC];
      const float* src = P.partial + (static_cast<int64_t>(b0) * 2 + slot0) * P.d + ch * VC;
#pragma unroll
      for (int e = 0; e < VC; ++e) acc[e] = __ldcg(src + e);
      for (int bb0 = b0 + 1; bb0 <= b1; bb0 += kMergeBatch) {   // kMergeBatch partials in flight, added in CTA order
        float tmp[kMergeBatch][VC];
        bool used[kMergeBatch];
#pragma unroll
        for (int u = 0; u < kMergeBatch; ++u) {
          const int bb = bb0 + u;
          const bool use = bb <= b1 && (all_nonempty || range_begin(bb + 1, P.nk, G) > range_begin(bb, P.nk, G));   // skip empty ranges
          const float* s2 = P.partial + (static_cast<int64_t>(bb) * 2) * P.d + ch * VC;
#pragma unroll
          used[u] = use;
#pragma unroll
          for (int e = 0; e < VC; ++e) tmp[u][e] = use ? __ldcg(s2 + e) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < kMergeBatch; ++u)
          if (used[u])
#pragma unroll
            for (int e = 0; e < VC; ++e) acc[e] += tmp[u][e];
      }
      store_chunk8<T, kF>(P, row, ch, acc, static_cast<float>(re - rs), fdst);
    }
  }
}


template <typename T>
__device__ void gather_rows(const Params& P) {   // baseline: send[p] = x[token of copy at p]
  const int64_t work = static_cast<int64_t>(P.nk) * P.nch;
  for (int64_t w = blockIdx.x * int64_t(kCThreads) + threadIdx.x; w < work; w += int64_t(gridDim.x) * kCThreads) {
    const int p = static_cast<int>(w / P.nch);
    const int ch = static_cast<int>(w - int64_t(p) * P.nch);
    const int t = ldcg(P.rowl + p) / P.k;
    reinterpret_cast<uint4*>(P.cent + static_cast<int64_t>(p) * P.row_bytes)[ch] =
        __ldg(reinterpret_cast<const uint4*>(P.x + static_cast<int64_t>(t) * P.row_bytes) + ch);
  }
}

// ---- fused phase-2 dispatch (lshmoe_compress_p2p; the protocol of p2p.cu's dispatch_p2p_kernel) ----
__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_rlx_sys64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t* f_slot(const Params& P, int rank, uint32_t ep, int src, int e) {
  return reinterpret_cast<uint64_t*>(P.p2p_peers[rank] + P.p2p_mailbox) +
         (static_cast<int64_t>(ep & 1) * P.p2p_world + src) * P.E + e;
}

// CTA 0 posts this rank's counts (epoch-tagged words) into every peer's mailbox; every CTA reads all
// sources' counts, then the destination base of each of its experts' rows in the owner's receive
// layout (local expert, source, bucket; reading R24).  CTA 0 also writes recv_rows.
__device__ void fused_prologue(const Params& P, const int* s_roff, const int* s_mrow, uint32_t* epoch_out) {
  int* s_fc = reinterpret_cast<int*>(g_dsmem);   // [w][E] counts: the ring is not in use yet
  const int tid = threadIdx.x, E = P.E, w = P.p2p_world, epr = E / w;
  const uint32_t ep = *reinterpret_cast<volatile unsigned*>(P.p2p_done + 2) + 1u;
  *epoch_out = ep;
  if (blockIdx.x == 0)
    for (int i = tid; i < w * E; i += kCThreads) {
      const int p = i / E, e = i - p * E;
      const uint64_t v = (static_cast<uint64_t>(ep) << 32) | static_cast<uint32_t>(s_mrow[e]);
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f_slot(P, p, ep, P.p2p_me, e)), "l"(v) : "memory");
    }
  const uint64_t t0 = gtimer();
  for (int i = tid; i < w * E; i += kCThreads) {
    const int src = i / E, e = i - src * E;
    uint64_t v = ld_rlx_sys64(f_slot(P, P.p2p_me, ep, src, e));
    while (static_cast<uint32_t>(v >> 32) != ep) {
      __nanosleep(32);
      if (gtimer() - t0 > P.p2p_spin_ns) {     // a peer never posted: count 0, flagged (no trap)
        atomicOr(P.p2p_done + 1, kP2PErrTimeout);
        v = static_cast<uint64_t>(ep) << 32;
        break;
      }
      v = ld_rlx_sys64(f_slot(P, P.p2p_me, ep, src, e));
    }
    s_fc[i] = static_cast<int>(v & 0xffffffffu);
  }
  __syncthreads();
  for (int e = tid; e <= E; e += kCThreads) g_f_roff[e] = s_roff[e];
  for (int e = tid; e < E; e += kCThreads) {
    const int p = e / epr, el = e - p * epr;
    long long b = 0;
    for (int e2 = 0; e2 < el; ++e2)
      for (int s2 = 0; s2 < w; ++s2) b += s_fc[s2 * E + p * epr + e2];
    for (int s2 = 0; s2 < P.p2p_me; ++s2) b += s_fc[s2 * E + p * epr + el];
    g_f_dst[e] = b;
  }
  if (blockIdx.x == 0 && P.p2p_recv_rows)
    for (int i = tid; i < epr * w; i += kCThreads) {
      const int el = i / w, s2 = i - el * w;
      P.p2p_recv_rows[i] = s_fc[s2 * E + P.p2p_me * epr + el];
    }
  __syncthreads();
}

// After every CTA's stores (the kernel's final barrier): arrive on the local counter (gpu-scope
// acq_rel); the last CTA issues one system-scope fence, records the epoch, raises data_flag[me] on
// every peer and waits until every source raised this rank's: the receive buffer is complete.
__device__ void fused_close(const Params& P, uint32_t ep) {
  if (threadIdx.x != 0) return;
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(P.p2p_done) : "memory");
  if (old != gridDim.x - 1) return;
  __threadfence_system();
  *P.p2p_done = 0;
  P.p2p_done[2] = ep;
  for (int p = 0; p < P.p2p_world; ++p)
    st_rel_sys(reinterpret_cast<uint32_t*>(P.p2p_peers[p] + P.p2p_data_flag) + P.p2p_me, ep);
  const uint32_t* fl = reinterpret_cast<const uint32_t*>(P.p2p_peers[P.p2p_me] + P.p2p_data_flag);
  const uint64_t t0 = gtimer();
  for (int s2 = 0; s2 < P.p2p_world; ++s2)
    while (static_cast<int32_t>(ld_acq_sys(fl + s2) - ep) < 0) {
      __nanosleep(64);
      if (gtimer() - t0 > P.p2p_spin_ns) {     // a peer never arrived: flagged, no trap
        atomicOr(P.p2p_done + 1, kP2PErrTimeout);
        return;
      }
    }
}

// ---- K3 ------------------------------------------------------------------------------------
// kF: the fused dispatch (lshmoe_compress_p2p) — compiled separately, so the plain kernel's
// reduction loop carries no remote-store code.
template <bool kF>
__global__ void __launch_bounds__(kCThreads, kCPerSM) centroid_kernel(Params P) {
  __shared__ int s_goff[kRadix + 1];         // perm offset of each expert group
  __shared__ int s_roff[kRadix + 1];         // first global row of each expert
  __shared__ int s_mrow[kRadix];             // m_e
  __shared__ int s_scan[kCWarps + 1];
  __shared__ int s_cut[4];
  __shared__ int s_job[8];
  const int tid = threadIdx.x;
  pdl_wait();                                // K2's perm, rows and counts are complete
  pdl_trigger();
  dstamp(P, 2, 0);
  IndexPre pre;
  if (!P.permute) preload_index(P, pre);      // in flight during the expert-count scan below
  if (!P.permute && !P.table_clean)          // K2 was the table's last reader: leave it at rest (-1)
    for (int64_t i = blockIdx.x * int64_t(kCThreads) + tid; i <= P.mask; i += int64_t(gridDim.x) * kCThreads)
      P.table[i] = -1;
  if (P.permute) {
    if (P.is_bf16) gather_rows<__nv_bfloat16>(P);
    else gather_rows<float>(P);
    return;
  }
  {
    const int m_e = tid < P.E ? ldcg(P.expert_rows + tid) : 0;
    const int go = tid < P.E ? ldcg(P.gofs + tid) : 0;   // in flight with m_e (and the index preload)
    int m;
    const int ro = block_excl_scan<kCWarps>(m_e, s_scan, &m);
    if (tid < P.E) {
      s_goff[tid] = go;
      s_roff[tid] = ro;
      s_mrow[tid] = m_e;
    }
    if (tid == 0) {
      s_goff[P.E] = P.nk;
      s_roff[P.E] = m;
      if (blockIdx.x == 0) {
        *P.num_rows = m;
        P.row_start[m] = P.nk;                // row_start[m] = n*k
      }
    }
    __syncthreads();
  }
  // row_start of every global row: rows r = blockIdx.x + G (tid + kCThreads u) of this CTA, loaded now
  // and stored after the reduction, so the load's round trip is off every CTA's critical path
  constexpr int kRS = 2;
  int rs_val[kRS];
  const int m_all = s_roff[P.E];
#pragma unroll
  for (int u = 0; u < kRS; ++u) {
    const int r = blockIdx.x + gridDim.x * (tid + kCThreads * u);
    rs_val[u] = 0;
    if (r < m_all) {
      const int e = expert_at(s_roff, P.E, r);
      rs_val[u] = ldcg(P.rsl + s_goff[e] + (r - s_roff[e]));
    }
  }
  uint32_t f_epoch = 0;
  if constexpr (kF) fused_prologue(P, s_roff, s_mrow, &f_epoch);
  // per-CTA centroid-phase start / end stamps (diagnostics, bar[64 + 2 * cta])
  if (P.diag && tid == 0 && blockIdx.x < 1024) P.bar[64 + 2 * blockIdx.x] = globaltimer_lo();
  CentroidCtx X;
  if (P.is_bf16) {
    centroid_phase<__nv_bfloat16, kF>(P, s_goff, s_roff, s_mrow, s_cut, X, pre);
    dstamp(P, 2, 2);
    merge_cut_rows<__nv_bfloat16, kF>(P, X, s_goff, s_mrow, s_cut, s_job);
  } else {
    centroid_phase<float, kF>(P, s_goff, s_roff, s_mrow, s_cut, X, pre);
    dstamp(P, 2, 2);
    merge_cut_rows<float, kF>(P, X, s_goff, s_mrow, s_cut, s_job);
  }
#pragma unroll
  for (int u = 0; u < kRS; ++u) {
    const int r = blockIdx.x + gridDim.x * (tid + kCThreads * u);
    if (r < m_all) P.row_start[r] = rs_val[u];
  }
  for (int r = blockIdx.x + gridDim.x * (tid + kCThreads * kRS); r < m_all; r += gridDim.x * kCThreads) {
    const int e = expert_at(s_roff, P.E, r);     // (m > G * 512 rows only)
    P.row_start[r] = ldcg(P.rsl + s_goff[e] + (r - s_roff[e]));
  }
  __syncthreads();
  if constexpr (kF) fused_close(P, f_epoch);   // every row was stored to its owner in the loop
  dstamp(P, 2, 3);
  if (P.diag && tid == 0 && blockIdx.x < 1024) P.bar[65 + 2 * blockIdx.x] = globaltimer_lo();
}

// ---- NEXT-1 grad_compress: G_b = sum_{(t,s) in b} g_ts dY_t over the forward's buckets --------
// The centroid kernel's machinery with the row of perm entry p = bucket[perm[p]], the gate weight
// of the copy staged beside its token id, and no 1/count; cut rows via the forward's row_start.
__global__ void __launch_bounds__(kCThreads, 1) grad_centroid_kernel(Params P) {
  __shared__ int s_cut[4];
  __shared__ int s_job[8];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  CentroidCtx X;
  X.p_begin = range_begin(b, P.nk, G);
  X.p_end = range_begin(b + 1, P.nk, G);
  X.range = X.p_end - X.p_begin;
  if (X.range == 0) return;
  X.lane = tid % 32;
  X.w = tid / 32;
  X.tok_off = P.max_range + 2;
  uint32_t* s_row = X.s_row();
  int32_t* s_tok = X.s_tok();
  float* s_w = X.s_wt(P.max_range);
  for (int i = tid; i < X.range + 2; i += kCThreads) {
    const int p = X.p_begin - 1 + i;
    uint32_t row = 0xFFFFFFFFu;
    if (p >= 0 && p < P.nk) {
      const int c = __ldg(P.perm + p);
      row = static_cast<uint32_t>(__ldg(P.bucket + c));
      if (i >= 1 && i <= X.range) {
        s_tok[i - 1] = c / P.k;
        if (P.gw) s_w[i - 1] = __ldg(P.gw + c);
      }
    }
    s_row[i] = row;
  }
  __syncthreads();
  prefetch_cut_extent(P, X, nullptr, nullptr, nullptr);
  X.w_begin = X.wbeg(X.w);
  X.w_end = X.wbeg(X.w + 1);
  X.prev_row = X.row_at(X.w_begin - 1);
  for (int c0 = 0, cb = 0; c0 < P.nch; c0 += kBlkChunks, ++cb) {
    const int ncb = min(kBlkChunks, P.nch - c0);
    const int cpl = (ncb + 31) / 32;
    if (P.is_bf16) {
      switch (cpl) {
        case 1: centroid_block<__nv_bfloat16, 1, ring_depth(1)>(P, X, cb, c0, ncb); break;
        case 2: centroid_block<__nv_bfloat16, 2, ring_depth(2)>(P, X, cb, c0, ncb); break;
        case 3: centroid_block<__nv_bfloat16, 3, ring_depth(3)>(P, X, cb, c0, ncb); break;
        default: centroid_block<__nv_bfloat16, 4, ring_depth(4)>(P, X, cb, c0, ncb); break;
      }
    } else {
      switch (cpl) {
        case 1: centroid_block<float, 1, ring_depth(1)>(P, X, cb, c0, ncb); break;
        case 2: centroid_block<float, 2, ring_depth(2)>(P, X, cb, c0, ncb); break;
        case 3: centroid_block<float, 3, ring_depth(3)>(P, X, cb, c0, ncb); break;
        default: centroid_block<float, 4, ring_depth(4)>(P, X, cb, c0, ncb); break;
      }
    }
  }
  if (P.is_bf16) merge_cut_rows<__nv_bfloat16>(P, X, nullptr, nullptr, s_cut, s_job);
  else merge_cut_rows<float>(P, X, nullptr, nullptr, s_cut, s_job);
}

constexpr int kCentroidSmemMax = 216 * 1024;   // K3 dynamic smem + static <= 227 KB
constexpr int kBucketSmem = 200 * 1024;        // K2 dynamic smem (+ 8 KB static)
int centroid_grid() { return std::min(kCPerSM * device_sm_count(), kMaxGrid); }
int centroid_max_range(int nk) {
  const int G = centroid_grid();
  return (nk + G - 1) / G + 1;
}
// K3 shared memory: per-warp rings, warp partials, the range's index arrays.
int centroid_smem(int max_range) {   // + the grad mode's per-entry weights
  return kCWarps * kRingWarp + kCWarps * kWpartFloats * 4 + 4 * (3 * max_range + 2);
}

// K2 CTAs per expert: the largest power of two CS <= kMaxCS for which all E clusters of CS CTAs
// are co-resident (cudaOccupancyMaxActiveClusters: a cluster needs CS SMs of one GPC), so the
// experts run in one wave.  LSHMOE_BUCKET_CS overrides, for experiments.
int bucket_cluster_size(int E);

int g_diag = 0;                              // lshmoe_set_diagnostics
bool diag_enabled() { return g_diag != 0; }

template <typename K>
int launch_pdl(K kernel, int grid, int block, int smem, cudaStream_t st, const Params& p, bool pdl, int cluster = 1) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  const int err = cudaLaunchKernelEx(&cfg, kernel, p);
  count_launches(1);
  return err;
}

bool carveout_max() {
  static const bool on = [] {
    const char* e = getenv("LSHMOE_CARVEOUT");
    return !(e && e[0] == '0');
  }();
  return on;
}

// The group path (group_kernel, one CTA per expert) when the gate map is one compaction round
// (n*k <= 16K copies) or the groups average at most 1024 copies; else K1 tiles + K2 clusters, whose
// per-expert CTA clusters spread big groups.  Measured (scripts/compress_diag.py, graph-timed per
// call, with the compaction overlapping the predecessor's tail): C2 32.6 us (group), C5 39.5 vs
// 48.8 (group vs tiles, 784 copies per expert), C4 83.4 vs 93.5 (1024), C3 91.9 vs 86.7 (2048:
// tiles).  LSHMOE_COMPRESS_PATH=group / tiles forces one.
bool group_path(int nk, int E) {
  static const int force = [] {
    const char* e = getenv("LSHMOE_COMPRESS_PATH");
    return !e ? 0 : (e[0] == 'g' ? 1 : (e[0] == 't' ? 2 : 0));
  }();
  if (force) return force == 1;
  return nk <= kGRound * kGThreads || static_cast<int64_t>(nk) <= 1024ll * E;
}

int launch_chain(const Params& P, cudaStream_t st) {
  static bool configured = false;
  const int max_range = centroid_max_range(P.nk);
  const int csmem = centroid_smem(max_range);
  if (!P.permute && csmem > kCentroidSmemMax) return cudaErrorInvalidValue;   // range too long
  if (!configured) {
    int err = cudaFuncSetAttribute(centroid_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCentroidSmemMax);
    if (!err) err = cudaFuncSetAttribute(centroid_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCentroidSmemMax);
    if (!err) err = cudaFuncSetAttribute(bucket_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBucketSmem);
    if (!err) err = cudaFuncSetAttribute(group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGroupSmem);
    // every kernel of the step prefers the full shared-memory carveout, so an SM never has to drain
    // and re-partition L1 / shared memory between two kernels of the chain (LSHMOE_CARVEOUT=0: off)
    if (!err && carveout_max()) err = cudaFuncSetAttribute(tile_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                           cudaSharedmemCarveoutMaxShared);
    if (err) return err;
    configured = true;
  }
  Params p = P;
  p.max_range = max_range;
  p.diag = diag_enabled() ? 1 : 0;
  int err = 0;
  if (group_path(P.nk, P.E)) {                        // one CTA per expert (group_kernel), then K3
    p.dyn_smem = kGroupSmem;
    p.table_clean = 1;
    err = launch_pdl(group_kernel, P.E, kGThreads, kGroupSmem, st, p, true);
  } else {                                   // K1 tiles + K2 clusters (LSHMOE_COMPRESS_PATH=tiles)
    p.dyn_smem = kBucketSmem;
    p.cs = bucket_cluster_size(P.E);
    err = launch_pdl(tile_kernel, P.ntiles, kThreads, 0, st, p, true);
    if (!err) err = launch_pdl(bucket_kernel, P.E * p.cs, kBThreads, kBucketSmem, st, p, true, p.cs);
  }
  if (!err) err = p.p2p_peers ? launch_pdl(centroid_kernel<true>, centroid_grid(), kCThreads, csmem, st, p, true)
                              : launch_pdl(centroid_kernel<false>, centroid_grid(), kCThreads, P.permute ? 0 : csmem, st, p, true);
  return err;
}

int bucket_cluster_size(int E) {
  static int cached_E = -1, cached_cs = 1;
  if (E == cached_E) return cached_cs;
  int cs = 1;
  for (int c = 2; c <= kMaxCS; c *= 2) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(E * c);
    cfg.blockDim = dim3(kBThreads);
    cfg.dynamicSmemBytes = kBucketSmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, bucket_kernel, &cfg) != cudaSuccess) {
      cudaGetLastError();
      break;
    }
    if (n >= E) cs = c;
    else break;
  }
  if (const char* env = getenv("LSHMOE_BUCKET_CS")) {
    const int v = atoi(env);
    if (v == 1 || v == 2 || v == 4 || v == 8) cs = v;
  }
  cached_E = E;
  cached_cs = cs;
  return cs;
}

}  // namespace

void set_compress_diag(int on) { g_diag = on ? 1 : 0; }

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
  const int64_t nk = n * k;
  int64_t tsize = 1024;
  while (tsize < 2 * nk) tsize <<= 1;
  const int64_t ntiles = (nk + kTile - 1) / kTile;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_hdr = take(sizeof(int32_t) * (kHdr + tsize));   // header + hash table: one memset
  const size_t o_tc = take(sizeof(int32_t) * ntiles * kTile);
  const size_t o_ts = take(sizeof(int32_t) * ntiles * kTile);
  const size_t o_to = take(sizeof(int32_t) * ntiles * (E + 1));
  const size_t o_rowid = take(sizeof(int32_t) * nk);
  const size_t o_rowl = take(sizeof(int32_t) * nk);
  const size_t o_rsl = take(sizeof(int32_t) * nk);
  const size_t o_gofs = take(sizeof(int32_t) * (E + 1));
  const size_t o_big = take(sizeof(int32_t) * 5 * kMaxCS * nk);
  const size_t o_rtot = take(sizeof(int32_t) * kMaxCS * nk);
  const size_t o_fcnt = take(sizeof(int32_t) * kMaxCS * (E + 1));
  const size_t o_part = take(sizeof(float) * 2 * kMaxGrid * d);
  if (ws) {
    uint8_t* b = static_cast<uint8_t*>(base);
    ws->hdr = reinterpret_cast<int32_t*>(b + o_hdr);
    ws->table = ws->hdr + kHdr;
    ws->table_size = tsize;
    ws->tile_copy = reinterpret_cast<int32_t*>(b + o_tc);
    ws->tile_slot = reinterpret_cast<int32_t*>(b + o_ts);
    ws->tile_off = reinterpret_cast<int32_t*>(b + o_to);
    ws->rowid = reinterpret_cast<int32_t*>(b + o_rowid);
    ws->rowl = reinterpret_cast<int32_t*>(b + o_rowl);
    ws->rsl = reinterpret_cast<int32_t*>(b + o_rsl);
    ws->gofs = reinterpret_cast<int32_t*>(b + o_gofs);
    ws->big = reinterpret_cast<int32_t*>(b + o_big);
    ws->rtot = reinterpret_cast<int32_t*>(b + o_rtot);
    ws->fcnt = reinterpret_cast<int32_t*>(b + o_fcnt);
    ws->partial = reinterpret_cast<float*>(b + o_part);
    ws->bytes = off;
  }
  return off;
}

// Streams whose last library launch was lshmoe_gate_hash: its kernel writes the gate map and
// signals its dependents before finishing, so the next compress on that stream must not read the
// gate map before griddepcontrol.wait.  Any other predecessor leaves the gate map complete when
// it signals (kernels without an early trigger signal at completion).  LSHMOE_EARLY_GATE=0: off.
static std::mutex g_gate_mu;
static std::vector<void*> g_gate_streams;

void note_gate_hash_stream(void* stream) {
  std::lock_guard<std::mutex> lk(g_gate_mu);
  if (std::find(g_gate_streams.begin(), g_gate_streams.end(), stream) == g_gate_streams.end())
    g_gate_streams.push_back(stream);
}

static int early_gate_for(void* stream) {
  static const bool off = [] {
    const char* e = getenv("LSHMOE_EARLY_GATE");
    return e && e[0] == '0';
  }();
  std::lock_guard<std::mutex> lk(g_gate_mu);
  auto it = std::find(g_gate_streams.begin(), g_gate_streams.end(), stream);
  if (it != g_gate_streams.end()) {
    g_gate_streams.erase(it);
    return 0;
  }
  return off ? 0 : 1;
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
  P.ntiles = (P.nk + kTile - 1) / kTile;
  P.bar = reinterpret_cast<unsigned*>(ws.hdr);
  P.table = ws.table;
  P.mask = static_cast<uint32_t>(ws.table_size - 1);
  P.tile_copy = ws.tile_copy;
  P.tile_slot = ws.tile_slot;
  P.tile_off = ws.tile_off;
  P.rowid = ws.rowid;
  P.rowl = ws.rowl;
  P.rsl = ws.rsl;
  P.gofs = ws.gofs;
  P.big = ws.big;
  P.rtot = ws.rtot;
  P.fcnt = ws.fcnt;
  P.partial = ws.partial;
  return P;
}

int launch_compress(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int16_t* codes, int q,
                    const int32_t* experts, int k, int E, int32_t* bucket, int32_t* perm, int32_t* row_start,
                    int32_t* expert_rows, int32_t* num_rows, void* centroids, float* centroids_f32,
                    const CompressWs& ws, void* stream, const P2PFuse* fuse) {
  if (E > kMaxE || q > kMaxQ) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nk = static_cast<int>(n * k);
  int err;
  if (nk == 0) {
    if ((err = cudaMemsetAsync(expert_rows, 0, sizeof(int32_t) * E, st))) return err;
    if ((err = cudaMemsetAsync(num_rows, 0, sizeof(int32_t), st))) return err;
    if ((err = cudaMemsetAsync(row_start, 0, sizeof(int32_t), st))) return err;
    if (fuse)   // no rows: the standalone dispatch kernel still posts the zero counts and handshakes
      return launch_p2p(0, fuse->peers, fuse->L, fuse->world, fuse->me, E, nullptr, expert_rows, fuse->recv_rows,
                        fuse->done, fuse->grid, fuse->spin_ns, stream);
    return 0;
  }
  // The workspace is at rest between calls (hash table slots and arrival counters -1: K3 resets
  // the table, the last arriver its counter); the diagnostics stamps are cleared only when on.
  if (diag_enabled() && (err = cudaMemsetAsync(ws.hdr, 0xFF, sizeof(int32_t) * kHdr, st))) return err;
  Params P = base_params(x, dtype, n, d, experts, k, E, ws);
  P.early_gate = early_gate_for(stream);
  P.codes = codes;
  P.q = q;
  P.bucket = bucket;
  P.perm = perm;
  P.row_start = row_start;
  P.expert_rows = expert_rows;
  P.num_rows = num_rows;
  P.cent = static_cast<uint8_t*>(centroids);
  P.cent32 = centroids_f32;
  if (fuse) {
    P.p2p_peers = fuse->peers;
    P.p2p_mailbox = fuse->L.mailbox;
    P.p2p_recv = fuse->L.recv;
    P.p2p_data_flag = fuse->L.data_flag;
    P.p2p_recv_cap = fuse->L.recv_capacity;
    P.p2p_world = fuse->world;
    P.p2p_me = fuse->me;
    P.p2p_done = fuse->done;
    P.p2p_spin_ns = fuse->spin_ns;
    P.p2p_recv_rows = fuse->recv_rows;
  }
  return launch_chain(P, st);
}

size_t grad_compress_workspace_layout(int d, void* base, int32_t** hdr, float** partial) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_hdr = take(sizeof(int32_t) * kHdr);
  const size_t o_part = take(sizeof(float) * 2 * kMaxGrid * d);
  if (base) {
    *hdr = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(base) + o_hdr);
    *partial = reinterpret_cast<float*>(static_cast<uint8_t*>(base) + o_part);
  }
  return off;
}

int launch_grad_compress(const void* dy, lshmoe_dtype dtype, int64_t n, int d, const float* gw, const int32_t* bucket,
                         const int32_t* perm, const int32_t* row_start, int k, void* grad_out, float* grad_out_f32,
                         void* ws, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nk = static_cast<int>(n * k);
  if (nk == 0) return 0;
  static bool configured = false;
  if (!configured) {
    const int err = cudaFuncSetAttribute(grad_centroid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kCentroidSmemMax);
    if (err) return err;
    configured = true;
  }
  const int max_range = centroid_max_range(nk);
  const int smem = centroid_smem(max_range);
  if (smem > kCentroidSmemMax) return cudaErrorInvalidValue;
  int32_t* hdr;
  float* partial;
  grad_compress_workspace_layout(d, ws, &hdr, &partial);
  int err = 0;                                 // arrival counters are at rest (-1) between calls
  Params P{};
  P.x = static_cast<const uint8_t*>(dy);
  P.d = d;
  P.row_bytes = d * (dtype == LSHMOE_F32 ? 4 : 2);
  P.nch = P.row_bytes / 16;
  P.is_bf16 = dtype == LSHMOE_BF16;
  P.k = k;
  P.nk = nk;
  P.bucket = const_cast<int32_t*>(bucket);
  P.perm = const_cast<int32_t*>(perm);
  P.row_start = const_cast<int32_t*>(row_start);
  P.cent = static_cast<uint8_t*>(grad_out);
  P.cent32 = grad_out_f32;
  P.bar = reinterpret_cast<unsigned*>(hdr);
  P.partial = partial;
  P.max_range = max_range;
  P.grad = 1;
  P.gw = gw;
  grad_centroid_kernel<<<centroid_grid(), kCThreads, smem, st>>>(P);
  count_launches(1);
  return cudaGetLastError();
}

int launch_permute(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int32_t* experts, int k, int E,
                   int32_t* slot, int32_t* expert_rows, void* send, const CompressWs& ws, void* stream) {
  if (E > kMaxE) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nk = static_cast<int>(n * k);
  if (nk == 0) return cudaMemsetAsync(expert_rows, 0, sizeof(int32_t) * E, st);
  Params P = base_params(x, dtype, n, d, experts, k, E, ws);
  P.early_gate = early_gate_for(stream);
  P.bucket = slot;
  P.expert_rows = expert_rows;
  P.cent = static_cast<uint8_t*>(send);
  P.permute = 1;
  return launch_chain(P, st);
}

}  // namespace lshmoe
