// tcgen05 tensor-core kernels (sm_100a): one warp-specialised, persistent TN-GEMM mainloop
// (TMA -> shared-memory ring -> single-thread tcgen05.mma -> double-buffered TMEM accumulator),
// either per CTA (cta_group::1, M = 128) or per CTA pair (cluster of 2, cta_group::2, M = 256: each
// CTA stages its 128 A rows and half of the B tile, so per-SM shared-memory traffic per MMA drops
// from 12 KB to 8 KB), with two epilogues:
//
//  * ArgmaxEpi — a2, the cross-polytope hash of Eq. 3.  Y = X R_j^T is a
//    dense contraction [n, d] x [d, d] per hash j; each 128-token x BN-coordinate accumulator tile
//    is read back from TMEM by the thread owning the token row (TMEM lane = row), which keeps a
//    running (max |y|, index, sign) over the d coordinates — ties to the smallest index (strict
//    '>' scanning columns in ascending order), a zero winner is '+' (readings R1, R2).  Y never
//    reaches HBM; only the int16 code is stored.
//  * BiasActEpi — a7, the expert FFN E(x) = W2 relu(W1 x + b1) + b2 as two grouped GEMMs
//    over the received centroid rows, segmented per local expert by a device-side tile table.
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer (leader CTA),
// warps 2-5 = epilogue (warp w reads TMEM lanes 32*(w%4) .. +31).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "../abi/lshmoe_internal.h"
#include "common.cuh"
#include "sm100.cuh"

namespace lshmoe {
namespace {

using namespace sm100;

constexpr int BM = 128;                     // rows per CTA
constexpr int BK = 64;                      // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kEpiWarps = 8;                // two warps per TMEM lane quadrant, each takes half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiScratch = 1024;           // per epilogue warp (bias slice)

constexpr int kMaxLocalExperts = 256;
constexpr int kStaticSmem = 3072;           // sched tables (2 * 257 ints) + mbarriers + TMEM slot
// kScratch: epilogue scratch bytes per epilogue warp (0 lets the ring take one more stage).
template <int BN, int kCta, int kScratch = kEpiScratch>
struct Cfg {
  static constexpr int kBRows = BN / kCta;  // B rows staged by each CTA
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = kBRows * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTxBytes = kCta * kStageBytes;   // bytes the leader's full barrier waits for
  static constexpr int kFixed = kEpiWarps * kScratch;   // dynamic smem besides the ring
  // 227 KB per CTA on sm_100, minus the 3 KB static block (scheduler tables + barriers) that keeps
  // the dynamic window 1024-byte aligned for SWIZZLE_128B
  static constexpr int kBudget = 227 * 1024 - kStaticSmem - kFixed;
  static constexpr int kStages = kBudget / kStageBytes > 8 ? 8 : kBudget / kStageBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSmem = kStages * kStageBytes + kFixed;
};
template <class Epi>
struct EpiScratch { static constexpr int value = kEpiScratch; };

struct WorkItem {
  int a_row;       // first A row of this CTA's 128-row slice
  int b_row0;      // first B row of chunk 0 (cluster tile; a CTA adds rank * BN / kCta)
  int nchunks;     // accumulator chunks of BN columns in this unit
  int valid_rows;  // rows of this CTA's slice that are real outputs (may be <= 0)
  int tag0, tag1;  // epilogue-specific (hash: (m tile, j) id, j; FFN: expert, n0)
  int part, nparts;  // hash: which BN-column slice of the d coordinates this unit covers
  int pmask;         // hash: bit s set = a piece of this (tile, j) starts at slice s (merge slots)
};

// ---- schedulers (units are per cluster; bm = 128 * kCta rows per unit) ----------------------
// Hash units are (token tile, hash j, BN-column slice): d / BN times more units than (tile, j),
// so the persistent grid's last wave is nearly full (C2: 2304 units over 148 SMs instead of 768).
// The slices of one (tile, j) are merged by the last one to finish (ArgmaxEpi::finish).
// Contiguous mode (contig = 1, no gate): cluster g takes the contiguous range [g T / G, (g+1) T / G)
// of the T = m_tiles * q * (d / BN) accumulator chunks, ordered (tile, j, slice); its k-th unit is
// the k-th (tile, j) piece inside that range, all of whose chunks it drains with one running argmax.
// Only a (tile, j) cut by a range boundary (at most two per cluster) needs the cross-CTA merge, so
// the per-unit merge protocol (a global atomic round trip and three epilogue barriers) that bounded
// the round-robin split schedule is gone from all other units.  Units past a cluster's last piece
// are empty (nchunks = 0).
__device__ __forceinline__ int crange_begin(int g, int T, int G) {
  return static_cast<int>(static_cast<int64_t>(g) * T / G);
}
__device__ __forceinline__ int crange_owner(int c, int T, int G) {   // cluster whose range holds chunk c
  return static_cast<int>((static_cast<int64_t>(c + 1) * G - 1) / T);
}

struct HashSched {
  int n, q, d, bn, bm;
  int prefetch_b;   // 0: the rotations are L2-resident
  int m_tiles;
  int gate;         // NEXT-2: 1 = one extra unit per token tile for the gate scores (B rows q*d ..)
  int contig;       // 1: contiguous chunk ranges per cluster (see above)
  int groups = 1;   // contig: MMA groups (CTAs or CTA pairs) per cluster, each on its own token tile of
                    // the cluster tile, all walking the same (j, slice) chunk sequence (same B loads)
  int G;            // clusters (contig)
  int max_pieces;   // units per cluster (contig)
  __device__ void init(void*) {}
  int split;   // 1: one unit per BN slice; 0: one unit covers all d / BN slices (no merge)
  __device__ int units() const {
    if (contig) return G * max_pieces;
    return m_tiles * (q * (split ? d / bn : 1) + gate);
  }
  __device__ WorkItem get_contig(int u, int rank, int group) const {
    WorkItem w;
    const int np = d / bn;
    const int T = ((m_tiles + groups - 1) / groups) * q * np;   // chunks of the cluster tiles
    const int g = u % G, k = u / G;
    const int c0 = crange_begin(g, T, G), c1 = crange_begin(g + 1, T, G);
    const int p = c0 / np + k;                 // (cluster tile, j) pair of this piece
    const int first = max(c0, p * np), last = min(c1, p * np + np);
    const int mt = (p / q) * groups + group, j = p - (p / q) * q;   // this group's token tile
    w.a_row = mt * bm + rank * BM;
    w.valid_rows = min(BM, n - w.a_row);
    w.nparts = np;
    w.tag1 = j;
    w.tag0 = (mt * (bm / BM) + rank) * q + j;
    // (a group whose token tile lies past n keeps the unit: its A rows read as zeros, its epilogue
    // writes nothing, and it still issues its share of the cluster's multicast B loads)
    if (first >= last || c0 >= c1) {           // past this cluster's last piece
      w.nchunks = 0;
      w.part = 0;
      w.b_row0 = 0;
      w.pmask = 0;
      return w;
    }
    w.part = first - p * np;
    w.nchunks = last - first;
    w.b_row0 = j * d + w.part * bn;
    int mask = 0;                              // where the pieces of pair p start (one per cluster)
    for (int gg = crange_owner(p * np, T, G); gg <= crange_owner(p * np + np - 1, T, G); ++gg) {
      const int b0 = max(crange_begin(gg, T, G), p * np), b1 = min(crange_begin(gg + 1, T, G), p * np + np);
      if (b0 < b1) mask |= 1 << (b0 - p * np);
    }
    w.pmask = mask;
    return w;
  }
  __device__ WorkItem get(int u, int rank, int group) const {
    if (contig) return get_contig(u, rank, group);
    WorkItem w;
    const int np = split ? d / bn : 1;
    const int upt = q * np + gate;             // units per token tile: slices fastest, then j, then the gate
    const int mt = u / upt, r = u - mt * upt;
    w.a_row = mt * bm + rank * BM;
    w.valid_rows = min(BM, n - w.a_row);
    if (r == q * np) {                         // the gate unit: scores of the E experts (<= BN columns)
      w.b_row0 = q * d;
      w.nchunks = 1;
      w.tag0 = -1;
      w.tag1 = q;
      w.part = 0;
      w.nparts = 1;
      w.pmask = 1;
      return w;
    }
    const int j = r / np, c = r - j * np;
    w.tag0 = (mt * (bm / BM) + rank) * q + j;   // this CTA's 128-token slice x hash j
    w.tag1 = j;
    if (!split) {
      w.b_row0 = j * d;
      w.nchunks = d / bn;
      w.part = 0;
      w.nparts = 1;
      w.pmask = 1;
    } else {
      w.b_row0 = j * d + c * bn;
      w.nchunks = 1;
      w.part = c;
      w.nparts = np;
      w.pmask = (1 << np) - 1;
    }
    return w;
  }
};

struct FfnSched {
  const int32_t* recv_rows;  // [E_local, world]
  int E_local, world, N, bn, bm;
  int prefetch_b;   // weight k-blocks prefetched to L2 ahead of the TMA loads
  int* seg_start;   // smem [E_local + 1]
  int* tiles_pre;   // smem [E_local + 1]
  __device__ void init(void* smem) {
    seg_start = reinterpret_cast<int*>(smem);
    tiles_pre = seg_start + (kMaxLocalExperts + 1);
    // thread e loads expert e's row counts (all loads in flight at once), warp 0 scans
    const int tid = threadIdx.x;
    if (tid < E_local) {
      int r = 0;
      for (int s = 0; s < world; ++s) r += recv_rows[tid * world + s];
      seg_start[tid] = r;
      tiles_pre[tid] = ((r + bm - 1) / bm) * (N / bn);
    }
    __syncthreads();
    if (tid < 32) {
      constexpr int kPer = (kMaxLocalExperts + 31) / 32;   // entries per lane
      int rs[kPer], ts[kPer], rsum = 0, tsum = 0;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int e = tid * kPer + i;
        rs[i] = e < E_local ? seg_start[e] : 0;
        ts[i] = e < E_local ? tiles_pre[e] : 0;
        rsum += rs[i];
        tsum += ts[i];
      }
      int rx = rsum, tx = tsum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int ry = __shfl_up_sync(0xFFFFFFFFu, rx, off), ty = __shfl_up_sync(0xFFFFFFFFu, tx, off);
        if (tid >= off) {
          rx += ry;
          tx += ty;
        }
      }
      int rrun = rx - rsum, trun = tx - tsum;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int e = tid * kPer + i;
        if (e <= E_local) {
          seg_start[e] = rrun;
          tiles_pre[e] = trun;
        }
        rrun += rs[i];
        trun += ts[i];
      }
      if (tid == 31) {                     // totals (E_local may equal kMaxLocalExperts)
        seg_start[E_local] = rx;
        tiles_pre[E_local] = tx;
      }
    }
    __syncthreads();
  }
  int order;        // 0: units expert-major (e, mt, nt); 1: N-tile-major (nt, e, mt)
  int b_evict_first = 0;   // 1: weight loads carry an L2 evict-first policy (LSHMOE_FFN_EVICT)
  int pre_kb = 0;          // weight k-blocks warmed into L2 before the dependency wait (LSHMOE_FFN_PREKB)
  __device__ int units() const { return tiles_pre[E_local]; }
  __device__ WorkItem get(int u, int rank, int /*group*/) const {
    int e = 0, mt, nt;
    const int ntn = N / bn;
    if (order == 0) {         // expert of unit u: the last e with tiles_pre[e] <= u (binary search;
      int lo = 0, hi = E_local - 1;   // empty experts share their successor's prefix, so "last" skips them)
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tiles_pre[mid] <= u) lo = mid; else hi = mid - 1;
      }
      e = lo;
      const int local = u - tiles_pre[e];
      mt = local / ntn;
      nt = local - mt * ntn;
    } else {                 // tiles_pre[e] / ntn = M-tiles of the experts before e
      const int T = tiles_pre[E_local] / ntn;
      nt = u / T;
      const int j = u - nt * T;
      while (tiles_pre[e + 1] / ntn <= j) ++e;
      mt = j - tiles_pre[e] / ntn;
    }
    WorkItem w;
    w.a_row = seg_start[e] + mt * bm + rank * BM;
    w.b_row0 = e * N + nt * bn;
    w.nchunks = 1;
    w.valid_rows = min(BM, seg_start[e + 1] - w.a_row);
    w.tag0 = e;
    w.tag1 = nt * bn;
    w.part = 0;
    w.nparts = 1;
    w.pmask = 1;
    return w;
  }
};

template <class Sched>
__device__ __forceinline__ bool sched_b_evict_first(const Sched&) { return false; }
__device__ __forceinline__ bool sched_b_evict_first(const FfnSched& s) { return s.b_evict_first != 0; }

// Before the dependency wait (the weights are inputs no predecessor writes): cluster g warms L2
// with the first pre_kb k-blocks of this CTA's half of every (expert, N-tile) weight tile
// i = g, g + G, ..., so the first TMA loads after the wait hit L2 while the predecessor's last CTAs
// finish (the centroid kernel before GEMM 1 gathers from L2 and leaves HBM idle).
template <class Sched>
__device__ __forceinline__ void sched_prefetch_static(const Sched&, const CUtensorMap*, int, int, int, int, int) {}
__device__ __forceinline__ void sched_prefetch_static(const FfnSched& s, const CUtensorMap* tmB, int cluster,
                                                      int nclusters, int rank, int brows, int kbe) {
  if (s.pre_kb <= 0) return;
  const int ntn = s.N / s.bn;
  for (int i = cluster; i < s.E_local * ntn; i += nclusters) {
    const int e = i / ntn, nt = i - e * ntn;
    const int brow = e * s.N + nt * s.bn + rank * brows;
    for (int kb = 0; kb < s.pre_kb; ++kb) tma_prefetch_l2_2d(tmB, kb * kbe, brow);
  }
}

// ---- epilogues -------------------------------------------------------------------------------
constexpr int kMaxGateK = 8;

// kGate: the NEXT-2 gate+hash variant (compiled separately so the plain hash keeps its registers).
template <bool kGate>
struct ArgmaxEpiT {
  int16_t* codes;
  int q;
  // NEXT-2 gate (reading R29), active on units with tag1 == q when zeta != nullptr: the thread
  // keeps its row's top-k (score, expert) over the columns < E of its half, ties to the smaller id.
  int32_t* zeta = nullptr;    // [n, k] ascending expert ids
  float* gw = nullptr;        // [n, k] softmax over the k selected scores
  int E = 0, k = 0;
  float gs[kMaxGateK];
  int gi[kMaxGateK];
  int exp = 0;        // experiment (LSHMOE_HASH_EXP): 1 = skip the argmax scan, 2 = skip the MMAs
  uint2* partial;     // [nparts][rows_pad][q] (|y| bits, index | sign << 31) of each slice
  int* counter;       // [slices][q] arrival counters, zero at rest (reset by the last arrival)
  int rows_pad;
  // running winner in chain 0 (chains 1-3 stay empty: the block-max scan below replaced the four
  // interleaved chains); merged by (larger |y|, then smaller index), exactly the first maximum of
  // one ascending scan.
  float cb[4];
  int ci[4];
  float best;
  int bidx;
  bool bneg;
  __device__ __forceinline__ void begin(const WorkItem&, uint8_t*) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cb[k] = -1.0f;
      ci[k] = 0;
    }
#pragma unroll
    for (int i = 0; i < kMaxGateK; ++i) {
      gs[i] = -INFINITY;
      gi[i] = 0x7FFFFFFF;
    }
  }
  // insert (s, id) into the descending top-kMaxGateK list (ids arrive ascending, so a tie never
  // displaces); the first k entries are the top-k.  Every index is a compile-time constant so the
  // lists stay in registers.
  __device__ __forceinline__ void gate_insert(float sc, int id) {
    if (!(sc > gs[kMaxGateK - 1])) return;
#pragma unroll
    for (int i = kMaxGateK - 1; i > 0; --i) {
      const bool shift = sc > gs[i - 1];
      const bool here = !shift && sc > gs[i];
      if (shift) {
        gs[i] = gs[i - 1];
        gi[i] = gi[i - 1];
      } else if (here) {
        gs[i] = sc;
        gi[i] = id;
      }
    }
    if (sc > gs[0]) {
      gs[0] = sc;
      gi[0] = id;
    }
  }
  __device__ __forceinline__ void merge_chains() {
    best = cb[0];
    bidx = ci[0];
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      const int ik = ci[k] & 0x7FFFFFFF, ib = bidx & 0x7FFFFFFF;
      if (cb[k] > best || (cb[k] == best && ik < ib)) {
        best = cb[k];
        bidx = ci[k];
      }
    }
    bneg = (bidx & 0x80000000) != 0;
    bidx &= 0x7FFFFFFF;
  }
  // Slice merge: every slice stores its per-row winner; the last slice of (tile, j) to arrive
  // merges the nparts winners in slice order (strict '>': an earlier slice keeps ties, so the
  // result equals one ascending scan over all d coordinates) and writes the code.
  __device__ __forceinline__ void finish_split(const WorkItem& w, int row, uint8_t* shared_flag, int half, int nthr) {
    const int t = w.a_row + row;
    if (half == 0 && t >= 0 && t < rows_pad)
      partial[(static_cast<int64_t>(w.part) * rows_pad + t) * q + w.tag1] =
          make_uint2(__float_as_uint(best), static_cast<uint32_t>(bidx) | (bneg ? 0x80000000u : 0u));
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");   // all epilogue warps
    int* flag = reinterpret_cast<int*>(shared_flag);
    if (threadIdx.x == 64) {                                // first epilogue thread
      // acq_rel: releases this CTA's winners (ordered before by bar.sync), acquires the others'
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(counter + w.tag0) : "memory");
      const int last = old == __popc(w.pmask) - 1;
      if (last) counter[w.tag0] = 0;                        // leave the workspace zeroed
      *flag = last;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    const int last = *reinterpret_cast<volatile int*>(flag);
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");   // flag consumed before it is reused
    if (!last || half != 0 || row >= w.valid_rows) return;
    float b = -1.0f;
    uint32_t bi = 0;
    for (int p = 0; p < w.nparts; ++p) {             // the pieces in slice order
      if (!((w.pmask >> p) & 1)) continue;
      const uint2 v = __ldcg(partial + (static_cast<int64_t>(p) * rows_pad + t) * q + w.tag1);
      const float a = __uint_as_float(v.x);
      if (a > b) {
        b = a;
        bi = v.y;
      }
    }
    const int idx = static_cast<int>(bi & 0x7FFFFFFFu);
    codes[static_cast<int64_t>(t) * q + w.tag1] = static_cast<int16_t>((bi >> 31) ? -(idx + 1) : (idx + 1));
  }
  __device__ __forceinline__ void consume(const WorkItem& w, int /*row*/, const uint32_t (&r)[32], int col0, const uint8_t*) {
    if constexpr (kGate) {
      if (w.tag1 == q) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < E) gate_insert(__uint_as_float(r[i]), col0 + i);
        return;
      }
    }
    if (exp == 1) {
      if (r[0] == 0x7FC00001u && r[31] == 0x7FC00001u) cb[0] = 1.0f;   // keep the TMEM load live
      return;
    }
    // Block maximum of |y| first (a 5-level fmax tree: |.| is a free operand modifier, max is exact
    // and order-independent), then — only when the block beats the running winner (strictly, so an
    // equal magnitude keeps the earlier column) — the first column attaining it and its sign.
    float m16[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) m16[i] = fmaxf(fabsf(__uint_as_float(r[i])), fabsf(__uint_as_float(r[i + 16])));
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
      for (int i = 0; i < w; ++i) m16[i] = fmaxf(m16[i], m16[i + w]);
    const float bm = m16[0];
    if (bm > cb[0]) {
      int idx = 0;
      bool neg = false;
#pragma unroll
      for (int i = 31; i >= 0; --i) {   // descending: the last hit is the smallest column
        const float v = __uint_as_float(r[i]);
        if (fabsf(v) == bm) {
          idx = i;
          neg = v < 0.0f;                 // -0.0f is not < 0, so a zero winner is '+'
        }
      }
      cb[0] = bm;
      ci[0] = (col0 + idx) | (neg ? static_cast<int>(0x80000000u) : 0);
    }
  }
  // half: which half of the unit's columns this thread scanned (8 epilogue warps) or 0.
  // Gate unit: the two column halves' lists meet in shared memory, the merged top-k is written in
  // ascending expert id with softmax weights.
  __device__ __forceinline__ void finish_gate(const WorkItem& w, int row, uint8_t* scratch, int half, int nthr) {
    float* ls = reinterpret_cast<float*>(scratch);                 // [128][kMaxGateK]
    int* li = reinterpret_cast<int*>(scratch + 128 * kMaxGateK * 4);
    if (half == 1)
#pragma unroll
      for (int i = 0; i < kMaxGateK; ++i) {
        ls[row * kMaxGateK + i] = gs[i];
        li[row * kMaxGateK + i] = gi[i];
      }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    if (half == 0 && row < w.valid_rows) {
      // (every loop below has a compile-time trip count: the arrays stay in registers)
#pragma unroll
      for (int i = 0; i < kMaxGateK; ++i) {  // the other half's ids are all larger: insert keeps order
        const float sc = ls[row * kMaxGateK + i];
        const int id = li[row * kMaxGateK + i];
        if (id != 0x7FFFFFFF) gate_insert(sc, id);
      }
      int ids[kMaxGateK];
      float scs[kMaxGateK];
#pragma unroll
      for (int i = 0; i < kMaxGateK; ++i) {
        ids[i] = i < k ? gi[i] : 0x7FFFFFFF;
        scs[i] = gs[i];
      }
#pragma unroll
      for (int pass = 0; pass < kMaxGateK - 1; ++pass)   // ascending expert id (odd-even network)
#pragma unroll
        for (int j = pass & 1; j + 1 < kMaxGateK; j += 2)
          if (ids[j] > ids[j + 1]) {
            const int ti = ids[j]; ids[j] = ids[j + 1]; ids[j + 1] = ti;
            const float tf = scs[j]; scs[j] = scs[j + 1]; scs[j + 1] = tf;
          }
      float mx = -INFINITY, ex[kMaxGateK], sum = 0.0f;
#pragma unroll
      for (int i = 0; i < kMaxGateK; ++i)
        if (i < k) mx = fmaxf(mx, scs[i]);
#pragma unroll
      for (int i = 0; i < kMaxGateK; ++i) {
        ex[i] = i < k ? expf(scs[i] - mx) : 0.0f;
        sum += ex[i];
      }
      const int64_t t = w.a_row + row;
#pragma unroll
      for (int i = 0; i < kMaxGateK; ++i)
        if (i < k) {
          zeta[t * k + i] = ids[i];
          gw[t * k + i] = ex[i] / sum;
        }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  }
  __device__ __forceinline__ void finish(const WorkItem& w, int row, uint8_t* scratch, int half, int nthr) {
    if constexpr (kGate) {
      if (w.tag1 == q) {
        finish_gate(w, row, scratch, half, nthr);
        return;
      }
    }
    if (w.nchunks == 0 || w.valid_rows <= 0) return;   // an empty unit / a slice past n (CTA-uniform)
    merge_chains();
    if (nthr > 128) {   // combine the two column halves of each row; the lower half wins ties
      uint2* mb = reinterpret_cast<uint2*>(scratch + 64);
      if (half == 1) mb[row] = make_uint2(__float_as_uint(best), static_cast<uint32_t>(bidx) | (bneg ? 0x80000000u : 0u));
      asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
      if (half == 0) {
        const uint2 o = mb[row];
        if (__uint_as_float(o.x) > best) {
          best = __uint_as_float(o.x);
          bidx = static_cast<int>(o.y & 0x7FFFFFFFu);
          bneg = (o.y >> 31) != 0;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    }
    if (w.nchunks < w.nparts) {                      // a piece of a cut (tile, j): merge
      finish_split(w, row, scratch, half, nthr);
      return;
    }
    if (half == 0 && row < w.valid_rows) {
      const int t = w.a_row + row;
      codes[static_cast<int64_t>(t) * q + w.tag1] = static_cast<int16_t>(bneg ? -(bidx + 1) : (bidx + 1));
    }
  }
};

using ArgmaxEpi = ArgmaxEpiT<false>;
using GateArgmaxEpi = ArgmaxEpiT<true>;

// SignBitsEpi — NEXT-3, spherical-plane hashing (§4.5; SPEC's sign-bit reading
// S:L124-132, reading R26): Y = X N^T with the q*b unit normals as B rows (one BN-wide unit holds
// all of them); a thread keeps the sign bits (y >= 0, so a zero dot and -0 give 1) of its row's
// columns as 32-bit words, the two column halves meet in shared memory, and code_j = the b bits
// of hash j.  Only the int16 codes reach HBM.
template <int BN>
struct SignBitsEpi {
  int16_t* codes;
  int q, b;
  static constexpr int kBlkPer = (BN / 32) * 4 / kEpiWarps;   // 32-column blocks per thread
  uint32_t wds[kBlkPer];
  int nw;
  __device__ void begin(const WorkItem&, uint8_t*) { nw = 0; }
  __device__ void consume(const WorkItem&, int, const uint32_t (&r)[32], int, const uint8_t*) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) m |= (__uint_as_float(r[i]) >= 0.0f ? 1u : 0u) << i;
#pragma unroll
    for (int k = 0; k < kBlkPer; ++k)      // blocks arrive in ascending column order
      if (k == nw) wds[k] = m;
    ++nw;
  }
  __device__ void finish(const WorkItem& w, int row, uint8_t* scratch, int half, int nthr) {
    uint32_t* bits = reinterpret_cast<uint32_t*>(scratch);   // [128 rows][BN / 32 words]
    constexpr int kW = BN / 32;
#pragma unroll
    for (int k = 0; k < kBlkPer; ++k) bits[row * kW + half * kBlkPer + k] = wds[k];
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    if (half == 0 && row < w.valid_rows) {
      const int64_t t = w.a_row + row;
      for (int j = 0; j < q; ++j) {
        const int c0 = j * b, wi = c0 >> 5, sh = c0 & 31;
        uint64_t v = bits[row * kW + wi];
        if (wi + 1 < kW) v |= static_cast<uint64_t>(bits[row * kW + wi + 1]) << 32;
        codes[t * q + j] = static_cast<int16_t>((v >> sh) & ((1u << b) - 1u));
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");   // scratch reused by the next unit
  }
};

template <int BN>
struct BiasActEpi {
  const __nv_bfloat16* bias;  // [E_local, N]
  __nv_bfloat16* out;         // [rows, N]
  int N;
  bool relu;
  int exp = 0;                // experiment (LSHMOE_FFN_EXP): 1 = no output stores, 2 = no MMAs
  const __nv_bfloat16* mask = nullptr;   // NEXT-1 backward: out *= [mask > 0] (the forward's hidden), no bias
  const __nv_bfloat16* bias_unit;   // this unit's BN bias values (read-only cache, warp broadcast)
  __device__ void begin(const WorkItem& w, uint8_t*) {
    bias_unit = bias ? bias + static_cast<int64_t>(w.tag0) * N + w.tag1 : nullptr;
  }
  __device__ void consume(const WorkItem& w, int row, const uint32_t (&r)[32], int col0, const uint8_t* scratch) {
    if (row >= w.valid_rows) return;
    uint32_t packed[16];
    if (mask) {                 // backward: acc * relu'(pre), relu'(pre) = [h > 0] from the saved h
      const uint4* mrow = reinterpret_cast<const uint4*>(mask + static_cast<int64_t>(w.a_row + row) * N + w.tag1 + col0);
      uint32_t mw[16];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 m4 = __ldg(mrow + i);
        mw[4 * i] = m4.x; mw[4 * i + 1] = m4.y; mw[4 * i + 2] = m4.z; mw[4 * i + 3] = m4.w;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const bool p0 = __uint_as_float(mw[i] << 16) > 0.0f, p1 = __uint_as_float(mw[i] & 0xFFFF0000u) > 0.0f;
        const float v0 = p0 ? __uint_as_float(r[2 * i]) : 0.0f;
        const float v1 = p1 ? __uint_as_float(r[2 * i + 1]) : 0.0f;
        __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
        packed[i] = *reinterpret_cast<uint32_t*>(&h);
      }
    } else {
      const uint32_t* bw = reinterpret_cast<const uint32_t*>(bias_unit) + col0 / 2;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t b2 = bias ? __ldg(bw + i) : 0u;
        float v0 = __uint_as_float(r[2 * i]) + __uint_as_float(b2 << 16);
        float v1 = __uint_as_float(r[2 * i + 1]) + __uint_as_float(b2 & 0xFFFF0000u);
        if (relu) {
          v0 = fmaxf(v0, 0.0f);
          v1 = fmaxf(v1, 0.0f);
        }
        __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
        packed[i] = *reinterpret_cast<uint32_t*>(&h);
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(w.a_row + row) * N + w.tag1 + col0);
    if (exp == 1) {
      if ((packed[0] ^ packed[7] ^ packed[15]) == 0x12345678u) dst[0] = make_uint4(0, 0, 0, 0);   // keep the math live
      return;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)   // 256-bit stores: each lane writes whole 32-byte sectors of its row
      asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 2 * i), "r"(packed[8 * i]),
                   "r"(packed[8 * i + 1]), "r"(packed[8 * i + 2]), "r"(packed[8 * i + 3]), "r"(packed[8 * i + 4]),
                   "r"(packed[8 * i + 5]), "r"(packed[8 * i + 6]), "r"(packed[8 * i + 7])
                   : "memory");
  }
  __device__ void finish(const WorkItem&, int, uint8_t*, int, int) {}
};

template <int BN>
struct EpiScratch<BiasActEpi<BN>> { static constexpr int value = 0; };   // bias read via __ldg

template <class Epi>
__device__ __forceinline__ bool epi_skip_mma(const Epi&) { return false; }
template <int BN>
__device__ __forceinline__ bool epi_skip_mma(const BiasActEpi<BN>& e) { return e.exp == 2 || e.exp == 3; }
// experiment 3 (FFN): no MMAs and no accumulator drain (TMEM loads, bias, stores): the TMA stream alone
template <class Epi>
__device__ __forceinline__ bool epi_skip_drain(const Epi&) { return false; }
template <int BN>
__device__ __forceinline__ bool epi_skip_drain(const BiasActEpi<BN>& e) { return e.exp == 3; }
template <bool G>
__device__ __forceinline__ bool epi_skip_mma(const ArgmaxEpiT<G>& e) { return e.exp == 2; }

// ---- the kernel ----------------------------------------------------------------------------------
// kEB: operand element bytes — 2 = bf16 (kind::f16, 16-element MMA K), 1 = e4m3 (kind::f8f6f4,
// 32-element MMA K).  A k-block is always 128 bytes of K per row (one SWIZZLE_128B atom row), so
// the shared-memory layout, descriptors and byte offsets are the same for both.
// kMC > 1 (CTA pairs only): the cluster holds kMC pairs walking the same B chunks on their own
// token tiles; CTA (group g, rank r) loads 1/kMC of its half-B rows and multicasts them to the CTAs of
// rank r in every group, so each B byte is read from L2 once per cluster instead of once per pair.
// Every pair's commit then frees the stage in all CTAs of the cluster (empty barriers count kMC).
template <int BN, int kCta, class Sched, class Epi, int kEB = 2, int kMC = 1>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                   Sched sched, Epi epi) {
  using C = Cfg<BN, kCta, EpiScratch<Epi>::value>;
  // Static block first (exactly kStaticSmem bytes, 1024-aligned), so the dynamic window that
  // holds the TMA ring starts 1024-byte aligned (SWIZZLE_128B atoms) without a runtime pad.
  __shared__ __align__(1024) uint8_t s_static[kStaticSmem];
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  static_assert(8 * (2 * 8 + 4) + 8 + 2 * (kMaxLocalExperts + 1) * 4 <= kStaticSmem, "static block");
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023u) != 0) __trap();   // the layout assumption above must hold
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_static);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* sched_tables = reinterpret_cast<int*>(s_static + 8 * (2 * 8 + 4) + 8);
  uint8_t* epi_scratch = smem + C::kStages * C::kStageBytes;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  constexpr int kBKe = 128 / kEB;            // K elements per k-block
  const int kblocks = K / kBKe;
  // A cluster holds `groups` MMA groups of kCta CTAs (a lone CTA or a cta_group::2 pair, whose
  // peer differs in rank bit 0); all groups of a cluster walk the same unit sequence.
  const int crank = static_cast<int>(cluster_ctarank());
  const int csize = static_cast<int>(cluster_nctarank());
  const int rank = crank % kCta;              // rank inside the MMA group
  const int group = crank / kCta;
  const int gbase = group * kCta;             // cluster rank of the group's leader
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / csize;
  const int nclusters = gridDim.x / csize;
  const uint16_t gmask = static_cast<uint16_t>(((1u << kCta) - 1u) << gbase);   // the group's CTAs
  static_assert(kMC == 1 || kCta == 2, "B multicast is built on CTA pairs");
  // stage frees go to every CTA whose stage this group's data (A, and B for kMC > 1) lands in
  const uint16_t emask = kMC > 1 ? static_cast<uint16_t>((1u << (kCta * kMC)) - 1u) : gmask;
  uint16_t bmask = 0;                         // the CTAs of this rank in every group (B multicast)
#pragma unroll
  for (int g2 = 0; g2 < kMC; ++g2) bmask |= static_cast<uint16_t>(1u << (g2 * kCta + rank));
  constexpr int kBSubRows = C::kBRows / kMC;  // B rows this CTA loads for the cluster

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kMC);            // one commit from each group's MMA issuer
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * kCta);
    }
    fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) {
    if (kCta == 2) tmem_alloc_2cta<C::kTmemCols>(tmem_slot);
    else tmem_alloc<C::kTmemCols>(tmem_slot);
  }
  if (warp == 0 && lane == 0)   // static operands only (FFN weights): an L2 warm-up before the wait
    sched_prefetch_static(sched, &tmB, blockIdx.x / static_cast<int>(cluster_nctarank()),
                          static_cast<int>(gridDim.x / cluster_nctarank()), static_cast<int>(cluster_ctarank()) % kCta,
                          C::kBRows, 128 / kEB);
  // PDL: everything above (barriers, TMEM, descriptor prefetch) overlaps the previous kernel's
  // tail; nothing a predecessor writes is read before this wait.  Then let the next kernel launch.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
  sched.init(sched_tables);   // contains __syncthreads
  tc_fence_before();
  if (kCta == 2) cluster_sync();   // peer barriers initialised before any remote arrive / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = sched.units();

  if (warp == 0) {
    // ===== TMA producer (every CTA loads its A slice and its half of B; warp converged, one
    // elected lane issues) =====
    {
      const bool b_evict_first = sched_b_evict_first(sched);
      const uint64_t b_policy = b_evict_first ? l2_evict_first_policy() : 0ull;
      int stage = 0;
      uint32_t phase = 0;
      // L2 prefetch cursor running kPrefetchB k-blocks ahead of the loads (B operand only: the
      // FFN's weights stream from HBM once; the tokens are L2-resident)
      int pu = cluster, pc = 0, pkb = 0;
      WorkItem pw{};
      if (sched.prefetch_b > 0 && pu < units) pw = sched.get(pu, rank, group);
      auto prefetch_next = [&]() {
        if (sched.prefetch_b == 0 || pu >= units) return;
        if (lane == 0) tma_prefetch_l2_2d(&tmB, pkb * kBKe, pw.b_row0 + pc * BN + rank * C::kBRows);
        if (++pkb == kblocks) {
          pkb = 0;
          if (++pc == pw.nchunks) {
            pc = 0;
            pu += nclusters;
            if (pu < units) pw = sched.get(pu, rank, group);
          }
        }
      };
      for (int i = 0; i < sched.prefetch_b; ++i) prefetch_next();
      for (int u = cluster; u < units; u += nclusters) {
        const WorkItem w = sched.get(u, rank, group);
        for (int c = 0; c < w.nchunks; ++c) {
          const int brow = w.b_row0 + c * BN + rank * C::kBRows;
          for (int kb = 0; kb < kblocks; ++kb) {
            prefetch_next();
            mbar_wait(&empty[stage], phase ^ 1);
            if (kCta == 2) {
              if (leader) mbar_arrive_expect_tx_w(&full[stage], C::kTxBytes);
              tma_load_2d_2sm_w(sA + stage * C::kABytes, &tmA, &full[stage], kb * kBKe, w.a_row);
              if constexpr (kMC > 1)
                tma_load_2d_2sm_mc_w(sB + stage * C::kBBytes + group * kBSubRows * 128, &tmB, &full[stage],
                                     kb * kBKe, brow + group * kBSubRows, bmask);
              else if (b_evict_first)   // FFN weights: read once per step, keep the token rows in L2
                tma_load_2d_2sm_ef_w(sB + stage * C::kBBytes, &tmB, &full[stage], kb * kBKe, brow, b_policy);
              else
                tma_load_2d_2sm_w(sB + stage * C::kBBytes, &tmB, &full[stage], kb * kBKe, brow);
            } else {
              mbar_arrive_expect_tx_w(&full[stage], C::kTxBytes);
              tma_load_2d_w(sA + stage * C::kABytes, &tmA, &full[stage], kb * kBKe, w.a_row);
              tma_load_2d_w(sB + stage * C::kBBytes, &tmB, &full[stage], kb * kBKe, brow);
            }
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer (the leader CTA's warp 1, converged; one elected lane issues) =====
    if (leader) {
      constexpr uint32_t idesc = kEB == 1 ? idesc_e4m3_f32(BM * kCta, BN) : idesc_bf16_f32(BM * kCta, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cluster; u < units; u += nclusters) {
        const WorkItem w = sched.get(u, rank, group);
        for (int c = 0; c < w.nchunks; ++c) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            // descriptors of the stage's k-block; +32 B of K = +2 in the 16-byte start-address field
            const uint64_t ad = smem_desc_sw128(smem_u32(sA + stage * C::kABytes));
            const uint64_t bd = smem_desc_sw128(smem_u32(sB + stage * C::kBBytes));
            static_assert(BK / 16 == 4, "mma4_commit issues four MMAs per k-block");
            if (epi_skip_mma(epi)) {      // experiment: no MMAs, the slot is freed at once
              if (kCta == 2) mma_commit_2cta_mc_w(&empty[stage], emask);
              else mma_commit_w(&empty[stage]);
            } else if (kEB == 1 && kCta == 2) {   // 32 e4m3 = 32 bytes of K per instruction
              mma4_commit_2cta_fp8(d_tmem, ad, bd, idesc, kb != 0, &empty[stage], emask);
            } else if (kEB == 1) {
              mma4_commit_1cta_fp8(d_tmem, ad, bd, idesc, kb != 0, &empty[stage]);
            } else if (kCta == 2) {             // the commit frees the slot in both CTAs of the pair
              mma4_commit_2cta_bf16(d_tmem, ad, bd, idesc, kb != 0, &empty[stage], emask);
            } else {
              mma4_commit_1cta_bf16(d_tmem, ad, bd, idesc, kb != 0, &empty[stage]);
            }
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (kCta == 2) mma_commit_2cta_mc_w(&tfull[acc], gmask);      // both epilogues may read
          else mma_commit_w(&tfull[acc]);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue warps =====
    const int quad = warp % 4;                      // TMEM lane quadrant this warp may access
    const int half = (warp - 2) / 4;                // which half of the BN columns it drains
    constexpr int kBlkPer = (BN / 32) * 4 / kEpiWarps;
    const int row = quad * 32 + lane;
    uint8_t* scratch = epi_scratch + (warp - 2) * EpiScratch<Epi>::value;
    const uint32_t tempty_leader0 = kCta == 2 ? mapa_shared(&tempty[0], gbase) : 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = cluster; u < units; u += nclusters) {
      const WorkItem w = sched.get(u, rank, group);
      epi.begin(w, scratch);
      for (int c = 0; c < w.nchunks; ++c) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN;
#pragma unroll 1
        for (int cb = half * kBlkPer; cb < (half + 1) * kBlkPer && !epi_skip_drain(epi); ++cb) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + cb * 32, r);
          tmem_ld_wait();
          epi.consume(w, row, r, (w.part + c) * BN + cb * 32, scratch);   // column within the unit's N range
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (kCta == 2) mbar_arrive_cluster(tempty_leader0 + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      epi.finish(w, row, epi_scratch, half, 32 * kEpiWarps);
    }
  }
  tc_fence_before();
  if (kCta == 2) cluster_sync();   // the pair's MMAs / remote arrivals are done before TMEM is freed
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (kCta == 2) tmem_dealloc_2cta<C::kTmemCols>(tmem_base);
    else tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// ---- host side ---------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// bf16 row-major [rows, cols] tensor, box {64 cols, box_rows rows}, SWIZZLE_128B.
// Row-major [rows, cols] tensor of bf16 (eb = 2) or bytes (eb = 1, e4m3), box {128 bytes of cols,
// box_rows rows}, SWIZZLE_128B.
int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int eb = 2) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * eb};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / eb), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, eb == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : cudaErrorInvalidValue;
}

template <int BN, int kCta, class Sched, class Epi, int kEB = 2, int kMC = 1>
int configure_tc() {
  auto kern = tc_gemm_kernel<BN, kCta, Sched, Epi, kEB, kMC>;
  static int configured = -1;     // one attribute call per instantiation
  if (configured < 0) {
    configured = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg<BN, kCta, EpiScratch<Epi>::value>::kSmem);
    if (!configured)   // clusters of up to 16 CTAs (8 are portable)
      configured = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  return configured;
}

// Clusters of csize CTAs of this instantiation that can be resident at once (0 on error): the
// persistent grid must not exceed it (GPCs whose SM count is not a multiple of csize leave SMs idle).
template <int BN, int kCta, class Sched, class Epi, int kEB = 2, int kMC = 1>
int active_clusters(int csize) {
  if (configure_tc<BN, kCta, Sched, Epi, kEB, kMC>()) return 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csize * 512);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg<BN, kCta, EpiScratch<Epi>::value>::kSmem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, tc_gemm_kernel<BN, kCta, Sched, Epi, kEB, kMC>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// groups: MMA groups per cluster (cluster = kCta * groups CTAs); grid is a multiple of the cluster.
template <int BN, int kCta, class Sched, class Epi, int kEB = 2, int kMC = 1>
int launch_tc(const CUtensorMap& a, const CUtensorMap& b, int K, const Sched& s, const Epi& e, int grid,
              cudaStream_t st, int groups = 1) {
  auto kern = tc_gemm_kernel<BN, kCta, Sched, Epi, kEB, kMC>;
  if (int err = configure_tc<BN, kCta, Sched, Epi, kEB, kMC>()) return err;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cfg<BN, kCta, EpiScratch<Epi>::value>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCta * groups;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (see the kernel's wait)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  int err = cudaLaunchKernelEx(&cfg, kern, a, b, K, s, e);
  count_launches(1);
  return err ? err : cudaGetLastError();
}

int pick_bn(int N) { return N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : 64); }

int env_bn(const char* name, int N, int dflt) {   // experiment override: 64 / 128 / 256 dividing N
  const char* env = getenv(name);
  if (!env) return dflt;
  const int v = atoi(env);
  return (v == 64 || v == 128 || v == 256) && N % v == 0 ? v : dflt;
}

// kCta = 2 needs BN / 2 rows per CTA to stay a multiple of 8 (SW128 atoms) and N >= 16 per CTA.
template <class Sched, class Epi>
int launch_bn(int bn, int cta, const void* A, int64_t a_rows, const void* B, int64_t b_rows, int K, Sched s, Epi e,
              int units_hint, cudaStream_t st, int groups = 1) {
  CUtensorMap ma, mb;
  int err = make_map(&ma, A, a_rows, K, BM);
  if (err) return err;
  err = make_map(&mb, B, b_rows, K, bn / cta);
  if (err) return err;
  s.bn = bn;
  s.bm = BM * cta;
  const int sms = device_sm_count();
  int clusters = sms / (cta * groups);
  if (units_hint > 0 && units_hint < clusters) clusters = units_hint;
  const int grid = clusters * cta * groups;
  if (cta == 2) {
    switch (bn) {
      case 256: return launch_tc<256, 2>(ma, mb, K, s, e, grid, st, groups);
      case 128: return launch_tc<128, 2>(ma, mb, K, s, e, grid, st, groups);
      default: return launch_tc<64, 2>(ma, mb, K, s, e, grid, st, groups);
    }
  }
  switch (bn) {
    case 256: return launch_tc<256, 1>(ma, mb, K, s, e, grid, st, groups);
    case 128: return launch_tc<128, 1>(ma, mb, K, s, e, grid, st, groups);
    default: return launch_tc<64, 1>(ma, mb, K, s, e, grid, st, groups);
  }
}

// Resident clusters of the hash kernel for (bn, cta, groups) (the persistent grid's size).
template <class Epi>
int hash_active_clusters(int bn, int cta, int groups) {
  const int cs = cta * groups;
  if (cta == 2) {
    switch (bn) {
      case 256: return active_clusters<256, 2, HashSched, Epi>(cs);
      case 128: return active_clusters<128, 2, HashSched, Epi>(cs);
      default: return active_clusters<64, 2, HashSched, Epi>(cs);
    }
  }
  switch (bn) {
    case 256: return active_clusters<256, 1, HashSched, Epi>(cs);
    case 128: return active_clusters<128, 1, HashSched, Epi>(cs);
    default: return active_clusters<64, 1, HashSched, Epi>(cs);
  }
}

// MMA width per GEMM: 1 = one CTA (M = 128), 2 = CTA pair (M = 256); overridable for experiments.
int cta_mode(const char* env_name, int dflt) {
  const char* env = getenv(env_name);
  if (env && (env[0] == '1' || env[0] == '2')) return env[0] - '0';
  return dflt;
}

int cta_mode_any(const char* env_name, int dflt) {   // a small positive integer from the environment
  const char* env = getenv(env_name);
  if (env && env[0] >= '1' && env[0] <= '9') return env[0] - '0';
  return dflt;
}

// Switches that make a kernel skip work (wrong results, timing experiments only) are honoured only
// when LSHMOE_EXPERIMENTS=1 is set as well, so a stray variable cannot corrupt a production run.
int experiment_mode(const char* env_name) {
  const char* on = getenv("LSHMOE_EXPERIMENTS");
  if (!on || on[0] != '1') return 0;
  const char* env = getenv(env_name);
  return env && env[0] >= '0' && env[0] <= '9' ? env[0] - '0' : 0;
}

int ffn_order() {   // experiment override LSHMOE_FFN_ORDER (0 expert-major, 1 N-tile-major)
  const char* env = getenv("LSHMOE_FFN_ORDER");
  return env ? atoi(env) : 0;
}

// The forward FFN's weight loads carry an L2 evict-first policy (LSHMOE_FFN_EVICT=0: off): the
// weights are read once per step, and without the hint their 151 MB (C2) push the step's token rows
// out of L2 before restore reads them again (C2 step 183.0 -> 179.8 us, eager restore 18.5 -> 16 us).
int ffn_evict_first() {
  const char* env = getenv("LSHMOE_FFN_EVICT");
  return env && env[0] == '0' ? 0 : 1;
}

// LSHMOE_FFN_PREKB: weight k-blocks warmed into L2 before the dependency wait (default 4), capped so
// that the warm-up stays a small fraction of L2: at most 32 MB over all E_local x N weight rows
// (C2: 4 k-blocks = 25 MB; C4's first GEMM, 134 MB per k-block: none).
int ffn_pre_kb(int E_local, int N) {
  const char* env = getenv("LSHMOE_FFN_PREKB");
  const int want = env ? atoi(env) : 4;
  const int64_t per_kb = static_cast<int64_t>(E_local) * N * 128;   // bytes of one k-block of every row
  const int64_t cap = per_kb > 0 ? (32ll << 20) / per_kb : 0;
  return static_cast<int>(std::min<int64_t>(want, cap));
}

int ffn_prefetch() {   // experiment override LSHMOE_FFN_PF (k-blocks); default 0 (measured: no gain)
  const char* env = getenv("LSHMOE_FFN_PF");
  return env ? atoi(env) : 0;
}

}  // namespace

int device_sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Hash workspace: arrival counters [ceil(n/256)*2][q] int32 (zero at rest) + slice winners
// [d/BN][rows_pad][q] uint2.  Only needed when d > BN (more than one slice per (tile, j)).
size_t hash_workspace_bytes(int64_t n, int d, int q) {
  const int bn = pick_bn(d);
  if (d <= bn) return 0;
  const int64_t rows_pad = ((n + 255) / 256) * 256;
  const size_t counters = ((sizeof(int) * (rows_pad / BM) * q) + 255) & ~size_t(255);
  return counters + sizeof(uint2) * static_cast<size_t>(d / bn) * rows_pad * q;
}

// Contiguous chunk ranges per cluster (HashSched::contig) unless LSHMOE_HASH_CONTIG=0; returns the
// cluster count G the launch must use.
int set_contig(HashSched& s, int cta, int np, int groups = 1, int max_clusters = 0) {
  const int T = ((s.m_tiles + groups - 1) / groups) * s.q * np;
  int G = max_clusters > 0 ? max_clusters : device_sm_count() / (cta * groups);
  if (T < G) G = T;
  s.groups = groups;
  const char* env = getenv("LSHMOE_HASH_CONTIG");
  if (groups == 1 && env && env[0] == '0') return T;   // round-robin split units (A/B)
  s.contig = 1;
  s.G = G;
  const int per = (T + G - 1) / G;
  s.max_pieces = (per + np - 1) / np + 1;
  return G;
}

int launch_hash_bf16(const void* x, int64_t n, int d, const void* R, int q, int16_t* codes, void* ws, void* stream) {
  // CTA pairs (M = 256, each CTA stages half of B): C2 75.7 vs 82.4 us, C4 499 vs 552 us per launch
  // (scripts/hash_groups_ab.py, graph-timed over cycled token copies)
  const int cta = cta_mode("LSHMOE_HASH_CTA", 2);
  HashSched s{};
  s.n = static_cast<int>(n);
  s.q = q;
  s.d = d;
  s.m_tiles = static_cast<int>((n + BM * cta - 1) / (BM * cta));
  const int bn = pick_bn(d);
  ArgmaxEpi e{};
  e.codes = codes;
  e.q = q;
  e.exp = experiment_mode("LSHMOE_HASH_EXP");
  e.rows_pad = static_cast<int>(((n + 255) / 256) * 256);
  // Slice split (one unit per BN slice of the d coordinates, slices merged by the last arrival)
  // evens out the persistent grid's last wave: C2 86.1 vs 90.2 us per launch, CUDA-graph timing in
  // scripts/ab_bench.py (LSHMOE_HASH_SPLIT=2 turns it off).
  s.split = (d > bn) && ws && cta_mode("LSHMOE_HASH_SPLIT", 1) == 1 ? 1 : 0;
  if (s.split) {
    const size_t counters = ((sizeof(int) * (e.rows_pad / BM) * q) + 255) & ~size_t(255);
    e.counter = static_cast<int*>(ws);
    e.partial = reinterpret_cast<uint2*>(static_cast<uint8_t*>(ws) + counters);
  }
  s.groups = 1;
  // B multicast across kMC CTA pairs of a cluster (LSHMOE_HASH_MC = 2 / 4; 1 = off)
  const int mc = cta == 2 && bn == 256 && s.split ? cta_mode_any("LSHMOE_HASH_MC", 1) : 1;
  if (mc == 2 || mc == 4) {
    const int ac = mc == 2 ? active_clusters<256, 2, HashSched, ArgmaxEpi, 2, 2>(2 * mc)
                           : active_clusters<256, 2, HashSched, ArgmaxEpi, 2, 4>(2 * mc);
    if (ac > 0) {
      const int G = set_contig(s, 2, d / bn, mc, ac);
      s.bn = bn;
      s.bm = BM * 2;
      CUtensorMap ma, mb;
      int err = make_map(&ma, x, n, d, BM);
      if (!err) err = make_map(&mb, R, static_cast<int64_t>(q) * d, d, bn / 2 / mc);
      if (err) return err;
      const int grid = G * 2 * mc;
      cudaStream_t st = static_cast<cudaStream_t>(stream);
      return mc == 2 ? launch_tc<256, 2, HashSched, ArgmaxEpi, 2, 2>(ma, mb, d, s, e, grid, st, mc)
                     : launch_tc<256, 2, HashSched, ArgmaxEpi, 2, 4>(ma, mb, d, s, e, grid, st, mc);
    }
  }
  int hint = s.m_tiles * q * (s.split ? d / bn : 1);
  int groups = 1;
  if (s.split) {
    // groups > 1: clusters of `groups` MMA groups on adjacent token tiles issue the same B loads
    // at the same time (experiment LSHMOE_HASH_GROUPS)
    if (const char* g = getenv("LSHMOE_HASH_GROUPS")) groups = std::max(1, std::min(8 / cta, atoi(g)));
    const int mc = groups > 1 ? hash_active_clusters<ArgmaxEpi>(bn, cta, groups) : 0;
    if (groups > 1 && mc <= 0) groups = 1;
    hint = set_contig(s, cta, d / bn, groups, mc);
  }
  return launch_bn(bn, cta, x, n, R, static_cast<int64_t>(q) * d, d, s, e, hint, static_cast<cudaStream_t>(stream),
                   groups);
}

// NEXT-2 gate + hash in one pass over x (reading R29): B = [R ; W_g] ([q*d + E, d]); per token
// tile one extra unit scores the E experts (one BN-wide chunk; rows past q*d + E read as zeros by
// TMA) and its epilogue writes the top-k experts and softmax weights instead of a code.
int launch_gate_hash_bf16(const void* x, int64_t n, int d, const void* RG, int q, int E, int k, int16_t* codes,
                          int32_t* zeta, float* gw, void* ws, void* stream) {
  const int bn = pick_bn(d);
  if (E > bn || k > kMaxGateK || k > E) return cudaErrorInvalidValue;
  HashSched s{};
  s.n = static_cast<int>(n);
  s.q = q;
  s.d = d;
  s.gate = 1;
  s.m_tiles = static_cast<int>((n + BM - 1) / BM);
  GateArgmaxEpi e{};
  e.codes = codes;
  e.q = q;
  e.zeta = zeta;
  e.gw = gw;
  e.E = E;
  e.k = k;
  e.rows_pad = static_cast<int>(((n + 255) / 256) * 256);
  s.split = (d > bn) && ws ? 1 : 0;
  if (s.split) {
    const size_t counters = ((sizeof(int) * (e.rows_pad / BM) * q) + 255) & ~size_t(255);
    e.counter = static_cast<int*>(ws);
    e.partial = reinterpret_cast<uint2*>(static_cast<uint8_t*>(ws) + counters);
  }
  return launch_bn(bn, 1, x, n, RG, static_cast<int64_t>(q) * d + E, d, s, e,
                   s.m_tiles * (q * (s.split ? d / bn : 1) + 1), static_cast<cudaStream_t>(stream));
}

// NEXT-2 fp8 option (reading R28): the same hash kernel on e4m3 operands (x8 [n, d] from
// lshmoe_quantize_e4m3, R8 [q*d, d] from lshmoe_rotation_e4m3), kind::f8f6f4 MMAs, 128-element
// k-blocks (half as many as bf16), the argmax epilogue unchanged.
int launch_hash_e4m3(const void* x8, int64_t n, int d, const void* R8, int q, int16_t* codes, void* ws, void* stream) {
  const int bn = pick_bn(d);
  const int cta = cta_mode("LSHMOE_HASH_CTA", 2);   // CTA pairs as the bf16 hash
  HashSched s{};
  s.n = static_cast<int>(n);
  s.q = q;
  s.d = d;
  s.bn = bn;
  s.bm = BM * cta;
  s.groups = 1;
  s.m_tiles = static_cast<int>((n + BM * cta - 1) / (BM * cta));
  ArgmaxEpi e{};
  e.codes = codes;
  e.q = q;
  e.exp = experiment_mode("LSHMOE_HASH_EXP");
  e.rows_pad = static_cast<int>(((n + 255) / 256) * 256);
  s.split = (d > bn) && ws && cta_mode("LSHMOE_HASH_SPLIT", 1) == 1 ? 1 : 0;
  if (s.split) {
    const size_t counters = ((sizeof(int) * (e.rows_pad / BM) * q) + 255) & ~size_t(255);
    e.counter = static_cast<int*>(ws);
    e.partial = reinterpret_cast<uint2*>(static_cast<uint8_t*>(ws) + counters);
  }
  CUtensorMap ma, mb;
  int err = make_map(&ma, x8, n, d, BM, 1);
  if (err) return err;
  err = make_map(&mb, R8, static_cast<int64_t>(q) * d, d, bn / cta, 1);
  if (err) return err;
  const int units = s.split ? set_contig(s, cta, d / bn) : s.m_tiles * q;
  const int grid = std::min(device_sm_count() / cta, units) * cta;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cta == 2) {
    switch (bn) {
      case 256: return launch_tc<256, 2, HashSched, ArgmaxEpi, 1>(ma, mb, d, s, e, grid, st);
      case 128: return launch_tc<128, 2, HashSched, ArgmaxEpi, 1>(ma, mb, d, s, e, grid, st);
      default: return launch_tc<64, 2, HashSched, ArgmaxEpi, 1>(ma, mb, d, s, e, grid, st);
    }
  }
  switch (bn) {
    case 256: return launch_tc<256, 1, HashSched, ArgmaxEpi, 1>(ma, mb, d, s, e, grid, st);
    case 128: return launch_tc<128, 1, HashSched, ArgmaxEpi, 1>(ma, mb, d, s, e, grid, st);
    default: return launch_tc<64, 1, HashSched, ArgmaxEpi, 1>(ma, mb, d, s, e, grid, st);
  }
}

// NEXT-3: SP hash.  B = the normals, rows q*b (the buffer holds sp_rows(q, b) >= q*b rows; rows
// past q*b are read but their bits are never used), K = d.
int sp_rows(int q, int b) {
  const int nb = q * b;
  return nb <= 64 ? 64 : (nb <= 128 ? 128 : 256);
}

template <int NP>
int launch_sp_np(const void* x, int64_t n, int d, const void* normals, int q, int b, int16_t* codes, cudaStream_t st) {
  CUtensorMap ma, mb;
  int err = make_map(&ma, x, n, d, BM);
  if (err) return err;
  err = make_map(&mb, normals, NP, d, NP);
  if (err) return err;
  HashSched s{};
  s.n = static_cast<int>(n);
  s.q = 1;
  s.d = NP;                  // one unit = one 128-token tile x all NP normal rows
  s.bn = NP;
  s.bm = BM;
  s.split = 0;
  s.m_tiles = static_cast<int>((n + BM - 1) / BM);
  SignBitsEpi<NP> e{codes, q, b};
  const int grid = std::min(device_sm_count(), s.m_tiles);
  return launch_tc<NP, 1>(ma, mb, d, s, e, grid, st);
}

int launch_sp_hash_bf16(const void* x, int64_t n, int d, const void* normals, int q, int b, int16_t* codes,
                        void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (sp_rows(q, b)) {
    case 64: return launch_sp_np<64>(x, n, d, normals, q, b, codes, st);
    case 128: return launch_sp_np<128>(x, n, d, normals, q, b, codes, st);
    default: return launch_sp_np<256>(x, n, d, normals, q, b, codes, st);
  }
}

// NEXT-1 expert backward (reading R27's H = J_E(c~)^T G, dX path only): two grouped TN GEMMs on
// the forward's machinery with the caller's transposed weights —
//   dh = (G W2) * [h > 0]   B = W2^T [E_local, d_ffn, d], K = d, mask = the forward's hidden h
//   H  = dh W1              B = W1^T [E_local, d, d_ffn], K = d_ffn, no bias
int launch_ffn_bwd_bf16(const void* G, int d, int d_ffn, const int32_t* recv_rows, int E_local, int world,
                        const void* W2T, const void* W1T, const void* hidden, void* dhidden, int64_t capacity,
                        void* H, void* stream) {
  if (E_local > kMaxLocalExperts) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cta = cta_mode("LSHMOE_FFN_CTA", 2);
  const __nv_bfloat16* hmask = static_cast<const __nv_bfloat16*>(hidden);
  FfnSched s1{recv_rows, E_local, world, d_ffn, 0, 0, 0, nullptr, nullptr, ffn_order()};
  int err;
  const int bn1 = pick_bn(d_ffn);
  if (bn1 == 256) {
    BiasActEpi<256> e1{nullptr, static_cast<__nv_bfloat16*>(dhidden), d_ffn, false};
    e1.mask = hmask;
    err = launch_bn(bn1, cta, G, capacity, W2T, static_cast<int64_t>(E_local) * d_ffn, d, s1, e1, 0, st);
  } else if (bn1 == 128) {
    BiasActEpi<128> e1{nullptr, static_cast<__nv_bfloat16*>(dhidden), d_ffn, false};
    e1.mask = hmask;
    err = launch_bn(bn1, cta, G, capacity, W2T, static_cast<int64_t>(E_local) * d_ffn, d, s1, e1, 0, st);
  } else {
    BiasActEpi<64> e1{nullptr, static_cast<__nv_bfloat16*>(dhidden), d_ffn, false};
    e1.mask = hmask;
    err = launch_bn(bn1, cta, G, capacity, W2T, static_cast<int64_t>(E_local) * d_ffn, d, s1, e1, 0, st);
  }
  if (err) return err;
  FfnSched s2{recv_rows, E_local, world, d, 0, 0, 0, nullptr, nullptr, ffn_order()};
  const int bn2 = pick_bn(d);
  if (bn2 == 256) {
    BiasActEpi<256> e2{nullptr, static_cast<__nv_bfloat16*>(H), d, false};
    return launch_bn(bn2, cta, dhidden, capacity, W1T, static_cast<int64_t>(E_local) * d, d_ffn, s2, e2, 0, st);
  } else if (bn2 == 128) {
    BiasActEpi<128> e2{nullptr, static_cast<__nv_bfloat16*>(H), d, false};
    return launch_bn(bn2, cta, dhidden, capacity, W1T, static_cast<int64_t>(E_local) * d, d_ffn, s2, e2, 0, st);
  }
  BiasActEpi<64> e2{nullptr, static_cast<__nv_bfloat16*>(H), d, false};
  return launch_bn(bn2, cta, dhidden, capacity, W1T, static_cast<int64_t>(E_local) * d, d_ffn, s2, e2, 0, st);
}

int launch_ffn_bf16(const void* in, int d, int d_ffn, const int32_t* recv_rows, int E_local, int world,
                    const void* W1, const void* b1, const void* W2, const void* b2, void* hidden, int64_t capacity,
                    void* out, void* stream) {
  if (E_local > kMaxLocalExperts) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cta = cta_mode("LSHMOE_FFN_CTA", 2);
  const int only = experiment_mode("LSHMOE_FFN_ONLY");   // experiment: 1 / 2 = launch only GEMM 1 / 2
  const int exp = experiment_mode("LSHMOE_FFN_EXP");     // experiment: 1 = no output stores, 2 = no MMAs
  FfnSched s1{recv_rows, E_local, world, d_ffn, 0, 0, ffn_prefetch(), nullptr, nullptr, ffn_order()};
  s1.b_evict_first = ffn_evict_first();
  s1.pre_kb = ffn_pre_kb(E_local, d_ffn);
  const int bn1 = env_bn("LSHMOE_FFN_BN1", d_ffn, pick_bn(d_ffn));
  int err = 0;
  if (only == 2) {
  } else if (bn1 == 256) {
    BiasActEpi<256> e1{static_cast<const __nv_bfloat16*>(b1), static_cast<__nv_bfloat16*>(hidden), d_ffn, true}; e1.exp = exp;
    err = launch_bn(bn1, cta, in, capacity, W1, static_cast<int64_t>(E_local) * d_ffn, d, s1, e1, 0, st);
  } else if (bn1 == 128) {
    BiasActEpi<128> e1{static_cast<const __nv_bfloat16*>(b1), static_cast<__nv_bfloat16*>(hidden), d_ffn, true}; e1.exp = exp;
    err = launch_bn(bn1, cta, in, capacity, W1, static_cast<int64_t>(E_local) * d_ffn, d, s1, e1, 0, st);
  } else {
    BiasActEpi<64> e1{static_cast<const __nv_bfloat16*>(b1), static_cast<__nv_bfloat16*>(hidden), d_ffn, true}; e1.exp = exp;
    err = launch_bn(bn1, cta, in, capacity, W1, static_cast<int64_t>(E_local) * d_ffn, d, s1, e1, 0, st);
  }
  if (err || only == 1) return err;
  FfnSched s2{recv_rows, E_local, world, d, 0, 0, ffn_prefetch(), nullptr, nullptr, ffn_order()};
  s2.b_evict_first = ffn_evict_first();
  s2.pre_kb = ffn_pre_kb(E_local, d);
  const int bn2 = env_bn("LSHMOE_FFN_BN2", d, pick_bn(d));
  if (bn2 == 256) {
    BiasActEpi<256> e2{static_cast<const __nv_bfloat16*>(b2), static_cast<__nv_bfloat16*>(out), d, false}; e2.exp = exp;
    return launch_bn(bn2, cta, hidden, capacity, W2, static_cast<int64_t>(E_local) * d, d_ffn, s2, e2, 0, st);
  } else if (bn2 == 128) {
    BiasActEpi<128> e2{static_cast<const __nv_bfloat16*>(b2), static_cast<__nv_bfloat16*>(out), d, false}; e2.exp = exp;
    return launch_bn(bn2, cta, hidden, capacity, W2, static_cast<int64_t>(E_local) * d, d_ffn, s2, e2, 0, st);
  }
  BiasActEpi<64> e2{static_cast<const __nv_bfloat16*>(b2), static_cast<__nv_bfloat16*>(out), d, false}; e2.exp = exp;
  return launch_bn(bn2, cta, hidden, capacity, W2, static_cast<int64_t>(E_local) * d, d_ffn, s2, e2, 0, st);
}

}  // namespace lshmoe
