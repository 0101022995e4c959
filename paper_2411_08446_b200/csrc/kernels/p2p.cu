// a6 / a8 phase 2: the centroid all-to-all (Alg. 1 L14) and its reverse
// (L16) as device-initiated copies into the peers' memory over NVLink — no host
// synchronisation and no NCCL on the data path.  Every rank owns a "window" (mapped into every
// peer with CUDA IPC) holding its receive / returned buffers, a double-buffered count mailbox and
// epoch flags.  Layouts are exactly phase 1's (comm.cpp): receive on rank p ordered (local expert,
// source, bucket) — reading R24; returned rows land in the source's centroid (send) layout.
//
// dispatch (one kernel, every CTA): CTA 0 writes this rank's per-expert counts into every peer's
// mailbox as epoch-tagged 64-bit words (no flag, no fence); every CTA polls its own mailbox until all
// w x E slots carry the epoch, derives the offsets, and copies its share of the rows (16-byte
// loads, kUnroll in flight per thread) straight into the owners' receive buffers; the last CTA to
// finish (arrival counter) raises data_flag[me] = epoch on every peer and waits until all sources
// have done the same for this rank, so the kernel ends with the receive buffer complete.
// combine: the owner copies each (local expert, source) segment back into the source's returned
// buffer at its send offset, then the same data-flag handshake (a second flag array).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../abi/lshmoe_internal.h"

namespace lshmoe {
namespace {
int p2p_experiment() {   // honoured only with LSHMOE_EXPERIMENTS=1 (see gemm_tcgen05.cu)
  const char* on = getenv("LSHMOE_EXPERIMENTS");
  const char* v = getenv("LSHMOE_P2P_EXP");
  return (on && on[0] == '1' && v) ? atoi(v) : 0;
}

constexpr int kP2PThreads = 256;

// Timing experiments only (LSHMOE_EXPERIMENTS=1 + LSHMOE_P2P_EXP bits; wrong across GPUs):
// 1 = gpu-scope flags and fences, 2 = no nanosleep in spins, 4 = skip the row copies,
// 8 = skip the closing handshake, 16 = per-CTA timestamps.
__device__ int g_p2p_exp = 0;
__device__ unsigned long long g_p2p_stamp[1024 * 4];   // exp bit 16: per-CTA globaltimer stamps
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  if (g_p2p_exp & 1) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  if (g_p2p_exp & 1) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_sys() {
  if (g_p2p_exp & 1) __threadfence();
  else __threadfence_system();
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin until every source's flag reached `epoch`.  A peer that never arrives (a rank that skipped
// the call, a straggler beyond the limit, kernels that cannot be co-resident) does not hang the
// device or trap (a trap would kill the whole context): after `spin_ns` the wait gives up, sets
// error bit 4 in done[1] (lshmoe_comm_p2p_error reports it) and the kernel finishes.
__device__ __forceinline__ void wait_flags(const uint32_t* flags, int world, uint32_t epoch, uint64_t spin_ns,
                                           unsigned* err) {
  const uint64_t t0 = global_ns();
  for (int s = 0; s < world; ++s)
    while (static_cast<int32_t>(ld_acquire_sys(flags + s) - epoch) < 0) {
      if (!(g_p2p_exp & 2)) __nanosleep(64);
      if (global_ns() - t0 > spin_ns) {
        atomicOr(err, kP2PErrTimeout);
        return;
      }
    }
}

struct P2PArgs {
  uint8_t* const* peers;   // [world] window base of every rank (peers[me] = own window)
  P2PLayout L;
  int world, me, E;
  uint32_t epoch;          // this call's epoch (> every earlier one): read from done[2] on the device
  const uint8_t* src;      // dispatch: centroids (send layout); combine: expert outputs (recv layout)
  const int32_t* expert_rows;   // dispatch: this rank's m_e [E]
  int32_t* recv_rows;      // dispatch: out [E/world][world] (may be null)
  unsigned* done;          // [0] CTA arrival counter (zero at rest); [1] error bits; [2] last epoch
  unsigned long long spin_ns;   // peer-wait limit
};

// Count mailbox slot (source `src`, expert e) of epoch `ep` in rank `rank`'s window: one 64-bit word
// (epoch << 32 | count) written with a single store, so a slot carries its own validity and needs no
// separate flag or fence; double-buffered by epoch parity (combine k still reads slot k & 1 while
// the peers post the counts of k + 1).
__device__ __forceinline__ uint64_t* mailbox_slot(const P2PArgs& a, int rank, uint32_t ep, int src, int e) {
  return reinterpret_cast<uint64_t*>(a.peers[rank] + a.L.mailbox) +
         (static_cast<int64_t>(ep & 1) * a.world + src) * a.E + e;
}
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Every CTA reads the w x E counts of epoch a.epoch from this rank's mailbox (spinning until every
// slot carries the epoch) into s_cnt[src * E + e].
__device__ void read_counts(const P2PArgs& a, int32_t* s_cnt) {
  const uint64_t t0 = global_ns();
  for (int i = threadIdx.x; i < a.world * a.E; i += kP2PThreads) {
    const int src = i / a.E, e = i - src * a.E;
    const uint64_t* slot = mailbox_slot(a, a.me, a.epoch, src, e);
    uint64_t v = ld_relaxed_sys_u64(slot);
    while (static_cast<uint32_t>(v >> 32) != a.epoch) {
      if (!(g_p2p_exp & 2)) __nanosleep(32);
      if (global_ns() - t0 > a.spin_ns) {     // a peer never posted: count 0, flagged (no trap)
        atomicOr(a.done + 1, kP2PErrTimeout);
        v = static_cast<uint64_t>(a.epoch) << 32;
        break;
      }
      v = ld_relaxed_sys_u64(slot);
    }
    s_cnt[i] = static_cast<int32_t>(v & 0xffffffffu);
  }
}

// Closing handshake: after a CTA barrier (its threads' stores ordered before thread 0), every CTA
// arrives on the local counter with a gpu-scope acq_rel atomic, so the last arriver has acquired
// every CTA's stores; it alone issues the system-scope fence (cumulative: it covers what it has
// acquired — one fence.sc.sys per call instead of one per CTA, measured 6 us less per call), resets
// the counter, raises flag[me] = epoch on every peer (st.release.sys) and waits until every source
// raised this rank's flag: the kernel ends with this rank's buffer complete.
__device__ void close_call(const P2PArgs& a, int64_t flag_off, bool dispatch, bool stamp) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned old = atom_add_acq_rel_gpu(a.done, 1u);
  if (old == gridDim.x - 1) {
    fence_sys();                                // one system-scope fence, cumulative over every CTA
    *a.done = 0;                                // at rest for the next call
    if (dispatch) a.done[2] = a.epoch;          // every CTA has read done[2] by now
    if (!(g_p2p_exp & 8)) {
      for (int p = 0; p < a.world; ++p)
        st_release_sys(reinterpret_cast<uint32_t*>(a.peers[p] + flag_off) + a.me, a.epoch);
      wait_flags(reinterpret_cast<const uint32_t*>(a.peers[a.me] + flag_off), a.world, a.epoch, a.spin_ns,
                 a.done + 1);
    }
  }
  if (stamp) g_p2p_stamp[blockIdx.x * 4 + 3] = global_ns();
}

// Grid-stride copy of `total` 16-byte chunks, kUnroll chunks in flight per thread (loads first, then
// the remote stores): chunk i -> (row r = i / nch, chunk ch); `locate` maps r to the destination
// row base pointer (nullptr: dropped).
constexpr int kUnroll = 4;
template <class Locate>
__device__ __forceinline__ void copy_rows(const P2PArgs& a, int64_t total, Locate locate) {
  const int nch = a.L.row_bytes / 16;
  const int64_t stride = int64_t(gridDim.x) * kP2PThreads;
  for (int64_t base = blockIdx.x * int64_t(kP2PThreads) + threadIdx.x; base < total; base += stride * kUnroll) {
    uint4 v[kUnroll];
    uint4* dst[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = base + u * stride;
      dst[u] = nullptr;
      if (i < total) {
        const int64_t r = i / nch;
        const int ch = static_cast<int>(i - r * nch);
        uint8_t* row = locate(r);
        if (row) {
          dst[u] = reinterpret_cast<uint4*>(row) + ch;
          v[u] = __ldg(reinterpret_cast<const uint4*>(a.src + r * a.L.row_bytes) + ch);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (dst[u]) *dst[u] = v[u];
  }
}

// Offsets from the counts (cnt[src * E + e]):
//   send_off[e]  = sum_{e' < e} cnt[me][e']                      (my rows of expert e, send layout)
//   recv_base(p, el, src) = sum_{el' < el} sum_s cnt[s][p*epr+el'] + sum_{s < src} cnt[s][p*epr+el]
__device__ int64_t recv_base(const int32_t* cnt, int world, int E, int p, int el, int src) {
  const int epr = E / world;
  int64_t b = 0;
  for (int e2 = 0; e2 < el; ++e2)
    for (int s = 0; s < world; ++s) b += cnt[s * E + p * epr + e2];
  for (int s = 0; s < src; ++s) b += cnt[s * E + p * epr + el];
  return b;
}

// The epoch lives on the device (done[2]) so that a captured CUDA graph replays correctly: dispatch
// uses done[2] + 1 and its last CTA stores it back (every CTA has read it by then); combine uses
// done[2] as left by the matching dispatch.  Every rank makes the same sequence of calls, so the
// epochs agree across ranks.
__global__ void __launch_bounds__(kP2PThreads) dispatch_p2p_kernel(P2PArgs a) {
  __shared__ int64_t s_soff[257];   // my send offsets per expert (+ total)
  __shared__ int64_t s_dst[256];    // destination row of my first row of expert e in its owner
  __shared__ int32_t s_cnt[8 * 256];
  const int tid = threadIdx.x;
  const int E = a.E, world = a.world, epr = E / world;
  a.epoch = *reinterpret_cast<volatile unsigned*>(a.done + 2) + 1u;
  const bool stamp = (g_p2p_exp & 16) && tid == 0 && blockIdx.x < 1024;
  if (stamp) g_p2p_stamp[blockIdx.x * 4] = global_ns();
  if (blockIdx.x == 0)                // my counts -> slot (me, e) of every peer's mailbox
    for (int i = tid; i < world * E; i += kP2PThreads) {
      const int p = i / E, e = i - p * E;
      st_relaxed_sys_u64(mailbox_slot(a, p, a.epoch, a.me, e),
                         (static_cast<uint64_t>(a.epoch) << 32) | static_cast<uint32_t>(a.expert_rows[e]));
    }
  read_counts(a, s_cnt);
  if (stamp) g_p2p_stamp[blockIdx.x * 4 + 1] = global_ns();
  __syncthreads();
  if (tid == 0) {
    int64_t o = 0;
    for (int e = 0; e < E; ++e) {
      s_soff[e] = o;
      o += s_cnt[a.me * E + e];
    }
    s_soff[E] = o;
  }
  for (int e = tid; e < E; e += kP2PThreads) s_dst[e] = recv_base(s_cnt, world, E, e / epr, e % epr, a.me);
  if (blockIdx.x == 0 && a.recv_rows)          // rows this rank receives per (local expert, source)
    for (int i = tid; i < epr * world; i += kP2PThreads) {
      const int el = i / world, s = i - el * world;
      a.recv_rows[i] = s_cnt[s * E + a.me * epr + el];
    }
  __syncthreads();
  const int64_t total = (g_p2p_exp & 4) ? 0 : s_soff[E] * (a.L.row_bytes / 16);
  copy_rows(a, total, [&](int64_t r) -> uint8_t* {
    int lo = 0, hi = E - 1;                   // expert of my row r: last e with s_soff[e] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_soff[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int64_t drow = s_dst[lo] + (r - s_soff[lo]);
    if (drow >= a.L.recv_capacity) {          // the owner's receive buffer is too small: drop, flag
      atomicOr(a.done + 1, 1u);
      return nullptr;
    }
    return a.peers[lo / epr] + a.L.recv + drow * a.L.row_bytes;
  });
  if (stamp) g_p2p_stamp[blockIdx.x * 4 + 2] = global_ns();
  close_call(a, a.L.data_flag, true, stamp);
}

__global__ void __launch_bounds__(kP2PThreads) combine_p2p_kernel(P2PArgs a) {
  __shared__ int64_t s_base[8 * 32 + 1];      // recv row of segment (el, src) and prefix (<= 256 segments)
  __shared__ int64_t s_soff[8 * 32];          // the source's send offset of expert me*epr + el
  __shared__ int32_t s_cnt[8 * 256];
  const int tid = threadIdx.x;
  const int E = a.E, world = a.world, epr = E / world;
  const int nseg = epr * world;
  a.epoch = *reinterpret_cast<volatile unsigned*>(a.done + 2);
  for (int i = tid; i < world * E; i += kP2PThreads) {   // the counts of the matching dispatch
    const int src = i / E, e = i - src * E;
    s_cnt[i] = static_cast<int32_t>(*mailbox_slot(a, a.me, a.epoch, src, e) & 0xffffffffu);
  }
  __syncthreads();
  if (tid == 0) {
    int64_t o = 0;
    for (int sg = 0; sg < nseg; ++sg) {
      const int el = sg / world, src = sg - el * world;
      const int e = a.me * epr + el;
      s_base[sg] = o;
      o += s_cnt[src * E + e];
      int64_t so = 0;
      for (int e2 = 0; e2 < e; ++e2) so += s_cnt[src * E + e2];
      s_soff[sg] = so;
    }
    s_base[nseg] = o;
  }
  __syncthreads();
  const int64_t total = (g_p2p_exp & 4) ? 0 : s_base[nseg] * (a.L.row_bytes / 16);
  copy_rows(a, total, [&](int64_t r) -> uint8_t* {
    int lo = 0, hi = nseg - 1;                // segment of recv row r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_base[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int64_t drow = s_soff[lo] + (r - s_base[lo]);
    if (drow >= a.L.ret_capacity) {
      atomicOr(a.done + 1, 2u);
      return nullptr;
    }
    return a.peers[lo % world] + a.L.returned + drow * a.L.row_bytes;
  });
  close_call(a, a.L.ret_flag, false, false);
}

}  // namespace

int launch_p2p(int which, uint8_t* const* peers_dev, const P2PLayout& L, int world, int me, int E, const void* src,
               const int32_t* expert_rows, int32_t* recv_rows, unsigned* done, int grid, unsigned long long spin_ns,
               void* stream) {
  P2PArgs a{peers_dev, L, world, me, E, 0u, static_cast<const uint8_t*>(src), expert_rows, recv_rows, done, spin_ns};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static int exp_set = -1;
  const int exp = p2p_experiment();
  if (exp != exp_set) {
    cudaMemcpyToSymbol(g_p2p_exp, &exp, sizeof(int));
    exp_set = exp;
  }
  if (which == 0) dispatch_p2p_kernel<<<grid, kP2PThreads, 0, st>>>(a);
  else combine_p2p_kernel<<<grid, kP2PThreads, 0, st>>>(a);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace lshmoe

extern "C" int lshmoe_debug_p2p_stamps(unsigned long long* host, int n) {   // experiments only
  return cudaMemcpyFromSymbol(host, lshmoe::g_p2p_stamp, sizeof(unsigned long long) * 4 * (n < 1024 ? n : 1024));
}
