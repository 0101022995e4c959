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
//   P3 centroid: perm split in one contiguous range per CTA; member rows are staged in shared
//                memory by cp.async, summed in perm order in fp32, scaled once by RN(1/count)
//                (reading R10) and rounded (RNE) into the send buffer.  Rows crossing ranges
//                leave fp32 partials;
//   P4 fix-up  : the CTA where such a row starts adds the partials in CTA order (deterministic).
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
constexpr int kIPT = 4;                  // max radix items per thread per tile (runtime P.ipt <= kIPT)
constexpr int kMinTile = kThreads;       // smallest tile (ipt = 1): sizes the histogram workspace
constexpr int kHistTiles = 64;           // tile histograms staged in shared memory up to this many
constexpr int kHistPitch = kHistTiles + 1;
constexpr int kHistSmem = kRadix * kHistPitch * 4;
constexpr int kWarps = kThreads / 32;
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
  float* partial;                  // [G][2][d] partial sums of rows cut by CTA ranges
  int ntiles, row_passes;
  int max_range;                   // centroid: max perm entries per CTA range
  int ipt;                         // radix elements per thread per tile (1, 2 or 4)
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
    // release this CTA's writes (ordered before by bar.sync), then acquire everyone else's
    asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    const unsigned target = phase * gridDim.x - 1u;
    unsigned v;
    while (true) {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (static_cast<int>(v - target) >= 0) break;
      __nanosleep(20);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
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
  const int base = tile * (kThreads * P.ipt) + warp * (P.ipt * 32);
#pragma unroll
  for (int r = 0; r < kIPT; ++r) {   // all key loads in flight before the ordered ranking rounds
    const int i = base + r * 32 + lane;
    if (r < P.ipt && i < n) pass_key(P, kind, pass, i, tr.key[r], tr.val[r]);
  }
#pragma unroll
  for (int r = 0; r < kIPT; ++r) {
    const int i = base + r * 32 + lane;
    const bool ok = r < P.ipt && i < n;
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
  const int ntiles = (n + kThreads * P.ipt - 1) / (kThreads * P.ipt);
  const int tpad = (ntiles + 3) & ~3;          // hist is digit-major [256][tpad]: 128-bit row loads
  const bool one_tile = ntiles <= static_cast<int>(gridDim.x);   // keep ranks in registers
  extern __shared__ int s_hist[];              // [256][kHistPitch] when tpad <= kHistTiles
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
    if (tpad <= kHistTiles) {   // whole table -> shared memory with coalesced 128-bit loads
      const int n4 = kRadix * tpad / 4;          // <= 16 * kThreads
      int4 v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {             // all loads first: one round trip
        const int j = threadIdx.x + i * kThreads;
        v[i] = j < n4 ? __ldcg(reinterpret_cast<const int4*>(P.hist) + j) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int j = threadIdx.x + i * kThreads;
        if (j < n4) {
          const int e = 4 * j, dd = e / tpad, col = e - dd * tpad;
          int* dst = s_hist + dd * kHistPitch + col;
          dst[0] = v[i].x; dst[1] = v[i].y; dst[2] = v[i].z; dst[3] = v[i].w;
        }
      }
      __syncthreads();
      const int* row = s_hist + dgt * kHistPitch;   // pitch 65: conflict-free column walk
      for (int u = 0; u < ntiles; ++u) {
        if (u == t) pre = tot;
        tot += row[u];
      }
    } else {
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
    if (kind == PASS_ROW0 && t == 0 && threadIdx.x == 0) P.bar[20] = globaltimer_lo();   // diagnostics
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
    if (kind == PASS_ROW0 && t == 0 && threadIdx.x == 0) P.bar[21] = globaltimer_lo();   // diagnostics
  }
  grid_barrier(P.bar, phase);
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
constexpr int kRingSlot = 16 * kBlkChunks;
constexpr int kWpartFloats = kBlkChunks * 8;   // one warp partial slot (fp32, up to 8 per chunk)
constexpr int kQ = 10;                   // ring rows per warp (kQ - 1 in flight)
static_assert(kWpartFloats * 4 <= kQ * kRingSlot, "a warp's slot-1 partial reuses its ring");

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

template <int VC>
__device__ __noinline__ void store_f32_copy(float* dst, const float* v) {   // tier-2 parity output only
#pragma unroll
  for (int e = 0; e < VC; ++e) dst[e] = v[e];
}

// centroid = acc * rc, rc = RN(1/count) (reading R10), RNE to the wire dtype; fp32 copy if requested.
template <typename T>
__device__ __forceinline__ void store_chunk16(const Params& P, int row, int c16, const float* acc, float rc) {
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
template <typename T>
__device__ __forceinline__ void store_chunk8(const Params& P, int row, int ch, const float* acc, float cnt) {
  constexpr int VC = sizeof(T) == 2 ? 4 : 2;
  const float rc = __frcp_rn(cnt);
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
  if (P.cent32) {
    float* dst = P.cent32 + static_cast<int64_t>(row) * P.d + ch * VC;
#pragma unroll
    for (int e = 0; e < VC; ++e) dst[e] = v[e];
  }
}

__device__ __forceinline__ int range_begin(int b, int nk, int G) { return static_cast<int>(static_cast<int64_t>(b) * nk / G); }
__device__ __forceinline__ int range_cta(int p, int nk, int G) {   // CTA whose range holds p
  return static_cast<int>((static_cast<int64_t>(p + 1) * G - 1) / nk);
}

// Dynamic shared memory of compress_kernel, named at file scope so that the centroid phase's
// addresses stay in the shared window (no generic-to-shared conversion per access).
extern __shared__ __align__(1024) uint8_t g_dsmem[];

// Centroid-phase shared memory: [warp][kQ][kRingSlot] rings | [warp][kWpartFloats] slot-0
// partials | rows[p_begin-1 .. p_end] | tok[p_begin .. p_end).
struct CentroidCtx {                     // one CTA's view of its perm range (centroid phase)
  int p_begin, p_end, range, w, lane, w_begin, w_end, tok_off;
  uint32_t prev_row;                     // row of entry w_begin - 1
  __device__ uint8_t* ring() const { return g_dsmem + w * kQ * kRingSlot; }
  __device__ float* slot0() const { return reinterpret_cast<float*>(g_dsmem + kWarps * kQ * kRingSlot); }
  __device__ uint32_t* s_row() const { return reinterpret_cast<uint32_t*>(slot0() + kWarps * kWpartFloats); }
  __device__ int32_t* s_tok() const { return reinterpret_cast<int32_t*>(s_row()) + tok_off; }
  __device__ uint32_t row_at(int p) const { return s_row()[p - p_begin + 1]; }
  __device__ int wbeg(int ww) const { return p_begin + range_begin(ww, range, kWarps); }
  __device__ float* wpart(int ww, int slot) const {   // slot 0: own region; slot 1: the warp's ring
    return slot == 0 ? slot0() + ww * kWpartFloats : reinterpret_cast<float*>(g_dsmem + ww * kQ * kRingSlot);
  }
};

// One column block (chunks [c0, c0 + ncb), CPL = ceil(ncb / 32) chunks per lane) of the centroid
// phase: stream the warp's rows through its ring, reduce segments, then combine cut rows.
template <typename T, int CPL>
__device__ void centroid_block(const Params& P, const CentroidCtx& X, int cb, int c0, int ncb) {
  constexpr int VC = 16 / sizeof(T);
  const int lane = X.lane, w = X.w, w_begin = X.w_begin, w_end = X.w_end;
  const bool full = ncb == CPL * 32;
  auto issue = [&](int p, int slot) {
    if (p < w_end) {
      const uint8_t* src = P.x + static_cast<int64_t>(X.s_tok()[p - X.p_begin]) * P.row_bytes + 16 * c0;
      uint8_t* dst = X.ring() + slot * kRingSlot;
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = lane + 32 * t;
        if (full || c < ncb) cp_async16(dst + 16 * c, src + 16 * c);
      }
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int i = 0; i < kQ - 1; ++i) issue(w_begin + i, i);
  float acc[CPL][VC];
#pragma unroll
  for (int t = 0; t < CPL; ++t)
#pragma unroll
    for (int e = 0; e < VC; ++e) acc[t][e] = 0.0f;
  int seg_start = w_begin, rd = 0, wr = kQ - 1;   // ring slots: next to read, next to fill
  uint32_t row = w_end > w_begin ? X.row_at(w_begin) : 0u;
#pragma unroll 1
  for (int p = w_begin; p < w_end; ++p) {
    issue(p + kQ - 1, wr);
    wr = wr + 1 == kQ ? 0 : wr + 1;
    cp_async_wait<kQ - 1>();                  // entry p (this lane's chunks) has landed
    const uint8_t* st = X.ring() + rd * kRingSlot;
    rd = rd + 1 == kQ ? 0 : rd + 1;
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int c = lane + 32 * t;
      if (full || c < ncb) add_chunk16<T>(acc[t], *reinterpret_cast<const uint4*>(st + 16 * c));
    }
    const uint32_t next = X.row_at(p + 1);
    if (next == row && p + 1 < w_end) continue;         // the segment goes on
    const bool head = seg_start > w_begin || X.prev_row != row;   // the row starts in this warp
    if (cb == 0 && lane == 0) {
      if (head) P.row_start[row] = seg_start;
      if (p + 1 == P.nk) P.row_start[row + 1] = P.nk;   // row_start[m] = n*k
    }
    if (head && next != row) {                // the whole row lies in this warp's sub-range
      const float rc = __frcp_rn(static_cast<float>(p + 1 - seg_start));
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        const int c = lane + 32 * t;
        if (full || c < ncb) store_chunk16<T>(P, static_cast<int>(row), c0 + c, acc[t], rc);
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
  cp_async_wait<0>();                         // the ring is free: it may hold the slot-1 partial
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
    const int wl = range_cta(hi - 1 - X.p_begin, X.range, kWarps);
    const bool before = lo == X.p_begin && X.row_at(X.p_begin - 1) == r;
    const bool after = hi == X.p_end && X.row_at(X.p_end) == r;
    const float rc = __frcp_rn(static_cast<float>(hi - lo));
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
        store_chunk16<T>(P, static_cast<int>(r), c0 + c, v, rc);
      }
    }
  };
  if (nrows > 0) {
    const bool first_w = w == range_cta(0, X.range, kWarps);   // first non-empty sub-range of the CTA
    if (cut_end && (first_w || !from_before)) own(r_last, seg_start);
    if (first_w) {                            // the CTA's first row, begun in an earlier CTA
      const uint32_t r0 = X.row_at(X.p_begin);
      if (X.prev_row == r0 && !(r0 == r_last && cut_end)) own(r0, X.p_begin);
    }
  }
  __syncthreads();                            // the ring is reused by the next column block
}

template <typename T>
__device__ void centroid_phase(const Params& P, const uint32_t* rows, const int32_t* tok) {
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  CentroidCtx X;
  X.p_begin = range_begin(b, P.nk, G);
  X.p_end = range_begin(b + 1, P.nk, G);
  X.range = X.p_end - X.p_begin;
  if (X.range == 0) return;                   // CTA-uniform
  X.lane = tid % 32;
  X.w = tid / 32;
  X.tok_off = P.max_range + 2;
  uint32_t* s_row = X.s_row();
  int32_t* s_tok = X.s_tok();
  for (int i = tid; i < X.range + 2; i += kThreads) {
    const int p = X.p_begin - 1 + i;
    s_row[i] = (p >= 0 && p < P.nk) ? ldcg(rows + p) : 0xFFFFFFFFu;
  }
  for (int i = tid; i < X.range; i += kThreads) s_tok[i] = ldcg(tok + X.p_begin + i);
  __syncthreads();
  X.w_begin = X.wbeg(X.w);
  X.w_end = X.wbeg(X.w + 1);
  X.prev_row = X.row_at(X.w_begin - 1);
  for (int c0 = 0, cb = 0; c0 < P.nch; c0 += kBlkChunks, ++cb) {
    const int ncb = min(kBlkChunks, P.nch - c0);
    switch ((ncb + 31) / 32) {
      case 1: centroid_block<T, 1>(P, X, cb, c0, ncb); break;
      case 2: centroid_block<T, 2>(P, X, cb, c0, ncb); break;
      case 3: centroid_block<T, 3>(P, X, cb, c0, ncb); break;
      default: centroid_block<T, 4>(P, X, cb, c0, ncb); break;
    }
  }
}

// Rows cut by CTA ranges: the CTA in which such a row starts adds the partials in CTA order.
template <typename T>
__device__ void fixup_phase(const Params& P, const uint32_t* rows) {
  constexpr int VC = sizeof(T) == 2 ? 4 : 2;
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int p_begin = range_begin(b, P.nk, G), p_end = range_begin(b + 1, P.nk, G);
  if (p_end >= P.nk || p_end <= p_begin) return;
  const uint32_t row = ldcg(rows + p_end - 1);
  if (ldcg(rows + p_end) != row) return;               // the range's last row ends inside it
  const int rs = ldcg(P.row_start + row);
  if (rs < p_begin) return;                            // started in an earlier range: not the owner
  const int re = ldcg(P.row_start + row + 1);
  const int b1 = range_cta(re - 1, P.nk, G);
  const int nc8 = P.row_bytes / 8;
  for (int ch = tid; ch < nc8; ch += kThreads) {
    float acc[VC];
    const float* src = P.partial + (static_cast<int64_t>(b) * 2 + (rs == p_begin ? 0 : 1)) * P.d + ch * VC;
#pragma unroll
    for (int e = 0; e < VC; ++e) acc[e] = __ldcg(src + e);
    for (int bb = b + 1; bb <= b1; ++bb) {
      if (range_begin(bb + 1, P.nk, G) == range_begin(bb, P.nk, G)) continue;   // empty range (nk < G)
      const float* s2 = P.partial + (static_cast<int64_t>(bb) * 2) * P.d + ch * VC;
#pragma unroll
      for (int e = 0; e < VC; ++e) acc[e] += __ldcg(s2 + e);
    }
    store_chunk8<T>(P, static_cast<int>(row), ch, acc, static_cast<float>(re - rs));
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

__global__ void __launch_bounds__(kThreads, 1) compress_kernel(Params P) {
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
  if (P.is_bf16) centroid_phase<__nv_bfloat16>(P, rows, tok);
  else centroid_phase<float>(P, rows, tok);
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < 1024) P.bar[65 + 2 * blockIdx.x] = globaltimer_lo();
  grid_barrier(P.bar, phase);
  if (P.is_bf16) fixup_phase<__nv_bfloat16>(P, rows);
  else fixup_phase<float>(P, rows);
  __syncthreads();
  stamp(P.bar, phase + 1);   // CTA 0's end (other CTAs may still be finishing the fix-up)
}

int bits_for(int64_t maxval) {   // bits needed to represent values in [0, maxval]
  int b = 1;
  while ((int64_t(1) << b) <= maxval) ++b;
  return b;
}

constexpr int kMaxGrid = 512;            // CTAs of the cooperative kernel (one per SM) <= this

// Dynamic shared memory: the radix offset step's tile histograms or the centroid ring, whichever
// is larger (the phases run one after the other).
constexpr int kMaxDynSmem = 214 * 1024;   // + the kernel's static shared memory <= 227 KB
int coop_max_range(int nk) {
  const int G = std::min(device_sm_count(), kMaxGrid);
  return (nk + G - 1) / G + 1;
}
// Centroid-phase shared memory: per-warp rings, warp partials, the range's index arrays.
int centroid_smem(int max_range) {
  return kWarps * kQ * kRingSlot + kWarps * kWpartFloats * 4 + 4 * (2 * max_range + 2);
}
int coop_smem(int max_range) { return std::max(centroid_smem(max_range), kHistSmem); }

int launch_coop(const Params& P, cudaStream_t st) {
  static int configured = 0;                 // largest dynamic smem size set so far
  const int max_range = coop_max_range(P.nk);
  const int smem = coop_smem(max_range);
  if (!P.permute && centroid_smem(max_range) > kMaxDynSmem) return cudaErrorInvalidValue;   // range too long
  if (smem > configured) {
    int err = cudaFuncSetAttribute(compress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err) return err;
    configured = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(device_sm_count(), kMaxGrid));   // one CTA per SM, all co-resident
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  Params p = P;
  p.max_range = max_range;
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
  const int64_t ntiles = (nk + kMinTile - 1) / kMinTile;   // upper bound over every ipt
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
  const size_t o_part = take(sizeof(float) * 2 * kMaxGrid * d);
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
  // elements per thread per radix tile: as few as possible while keeping <= 64 tiles (the tile
  // histograms then fit in shared memory for the offset step)
  P.ipt = P.nk <= kHistTiles * kThreads ? 1 : (P.nk <= 2 * kHistTiles * kThreads ? 2 : 4);
  P.ntiles = (P.nk + kThreads * P.ipt - 1) / (kThreads * P.ipt);
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
