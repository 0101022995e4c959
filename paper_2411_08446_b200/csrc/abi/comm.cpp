// a6 / a8: the centroid all-to-all-v of Alg. 1 L14 and its reverse L16, over
// NCCL on NVLink.  Expert placement: rank p owns experts [p*E/w, (p+1)*E/w).
//
// Send layout on every rank = compress's centroid layout (expert-major).  Receive layout on rank
// p = (local expert, source rank, local bucket) — DESIGN.md reading R24 — so each local expert's
// rows are contiguous for the expert FFN; rows of one (src, dst) pair are never reordered.
//
// Phase 1 (this file): ncclAllGather of the E counts, one stream synchronisation to read them on
// the host, then one grouped ncclSend/ncclRecv set (one message per (peer, expert) segment).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lshmoe_internal.h"

using namespace lshmoe;

struct lshmoe_comm {
  int world = 1;
  int rank = 0;
  ncclComm_t nccl = nullptr;
  // phase 2 (device-initiated exchange over peer memory)
  uint8_t* window = nullptr;               // this rank's window (owned)
  std::vector<uint8_t*> peers;             // every rank's window as mapped here (peers[rank] = window)
  std::vector<bool> peer_ipc;              // opened with cudaIpcOpenMemHandle (close on destroy)
  uint8_t** peers_dev = nullptr;           // device copy of `peers`
  unsigned* done = nullptr;                // [0] CTA arrival counter (zero at rest), [1] error bits, [2] epoch
  int32_t* recv_rows_dev = nullptr;        // [E/world][world] rows received per (local expert, source)
  P2PLayout L{};
  int p2p_E = 0;
  int p2p_grid = 64;                       // default CTAs per phase-2 call
  bool dispatched = false;                 // a dispatch_p2p was issued (combine needs one)
  bool local_group = false;                // virtual ranks of one process on one GPU (lshmoe_comm_local_group)
  unsigned long long spin_ns = 0;          // peer-wait limit of the phase-2 kernels (0: p2p_spin_limit_ns())
  int32_t* counts_dev = nullptr;     // [world * E_cap]
  int32_t* counts_host = nullptr;    // pinned [world * E_cap]
  int32_t* rr_host = nullptr;        // pinned [E_cap] recv_rows staging
  int E_cap = 0;
  int last_E = 0;                    // E of the last dispatch (plan valid iff > 0)
  std::vector<int32_t> counts;       // host copy of the last plan [world * E]
};

static unsigned long long comm_spin_ns(const lshmoe_comm* c) { return c->spin_ns ? c->spin_ns : p2p_spin_limit_ns(); }

static lshmoe_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return LSHMOE_OK;
  return set_error(LSHMOE_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

static lshmoe_status ensure_capacity(lshmoe_comm* c, int E) {
  if (E <= c->E_cap) return LSHMOE_OK;
  if (c->counts_dev) cudaFree(c->counts_dev);
  if (c->counts_host) cudaFreeHost(c->counts_host);
  if (c->rr_host) cudaFreeHost(c->rr_host);
  c->counts_dev = nullptr;
  c->counts_host = c->rr_host = nullptr;
  int err = cudaMalloc(&c->counts_dev, sizeof(int32_t) * c->world * E);
  if (!err) err = cudaMallocHost(&c->counts_host, sizeof(int32_t) * c->world * E);
  if (!err) err = cudaMallocHost(&c->rr_host, sizeof(int32_t) * E);
  if (err) return cuda_status(err, "lshmoe_comm: allocating count buffers");
  c->E_cap = E;
  return LSHMOE_OK;
}

extern "C" {

lshmoe_status lshmoe_exchange_plan(int world, int rank, int E, const int32_t* counts, int64_t* send_off,
                                   int64_t* recv_off, int32_t* recv_rows) {
  if (world < 1 || rank < 0 || rank >= world || E < 1 || E % world != 0)
    return set_error(LSHMOE_EINVAL, "lshmoe_exchange_plan: bad world / rank / E (E % world != 0, S:L285)");
  if (!counts || !send_off || !recv_off || !recv_rows) return set_error(LSHMOE_EINVAL, "lshmoe_exchange_plan: NULL");
  const int epr = E / world;
  // send: this rank's centroids, expert-major (rows of expert e at send_off[e])
  send_off[0] = 0;
  for (int e = 0; e < E; ++e) send_off[e + 1] = send_off[e] + counts[rank * E + e];
  // receive: segments ordered (local expert el, source src); S:L311 keeps each (src, dst) order
  recv_off[0] = 0;
  for (int el = 0; el < epr; ++el)
    for (int src = 0; src < world; ++src) {
      const size_t i = static_cast<size_t>(el) * world + src;
      const int32_t rows = counts[src * E + rank * epr + el];
      if (rows < 0) return set_error(LSHMOE_EINVAL, "lshmoe_exchange_plan: negative count");
      recv_rows[i] = rows;
      recv_off[i + 1] = recv_off[i] + rows;
    }
  return LSHMOE_OK;
}

lshmoe_status lshmoe_get_unique_id(uint8_t* id) {
  if (!id) return set_error(LSHMOE_EINVAL, "lshmoe_get_unique_id: id is NULL");
  static_assert(sizeof(ncclUniqueId) == LSHMOE_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  lshmoe_status st = nccl_status(ncclGetUniqueId(&u), "ncclGetUniqueId");
  if (st) return st;
  std::memcpy(id, &u, sizeof(u));
  return LSHMOE_OK;
}

lshmoe_status lshmoe_comm_init(const uint8_t* id, int world, int rank, lshmoe_comm** out) {
  if (!out) return set_error(LSHMOE_EINVAL, "lshmoe_comm_init: out is NULL");
  if (world < 1 || rank < 0 || rank >= world) return set_error(LSHMOE_EINVAL, "lshmoe_comm_init: bad world/rank");
  auto* c = new lshmoe_comm();
  c->world = world;
  c->rank = rank;
  // id == NULL at world > 1: a phase-2-only comm (no NCCL).  world == 1 with an id: a one-rank NCCL
  // communicator whose dispatch / combine run the phase-1 code (count all-gather, host plan, self
  // segments, grouped send/recv) instead of the aliased local exchange — phase 1 on one GPU.
  if (id) {
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    lshmoe_status st = nccl_status(ncclCommInitRank(&c->nccl, world, u, rank), "ncclCommInitRank");
    if (st) {
      delete c;
      return st;
    }
  }
  *out = c;
  return LSHMOE_OK;
}

static void p2p_release(lshmoe_comm* c) {
  for (size_t p = 0; p < c->peers.size(); ++p)
    if (c->peer_ipc.size() > p && c->peer_ipc[p] && c->peers[p]) cudaIpcCloseMemHandle(c->peers[p]);
  c->peers.clear();
  c->peer_ipc.clear();
  if (c->window) cudaFree(c->window);
  if (c->peers_dev) cudaFree(c->peers_dev);
  if (c->done) cudaFree(c->done);
  if (c->recv_rows_dev) cudaFree(c->recv_rows_dev);
  c->window = nullptr;
  c->peers_dev = nullptr;
  c->done = nullptr;
  c->recv_rows_dev = nullptr;
  c->p2p_E = 0;
}

static P2PLayout p2p_layout(int world, int E, int64_t recv_cap, int64_t ret_cap, int row_bytes) {
  P2PLayout L{};
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off += (bytes + 255) & ~int64_t(255);
    return o;
  };
  L.data_flag = take(4 * world);
  L.ret_flag = take(4 * world);
  L.mailbox = take(8 * 2 * static_cast<int64_t>(world) * E);
  L.recv = take(recv_cap * row_bytes);
  L.returned = take(ret_cap * row_bytes);
  L.recv_capacity = recv_cap;
  L.ret_capacity = ret_cap;
  L.row_bytes = row_bytes;
  L.bytes = off;
  return L;
}

// Allocates this rank's window (zeroed: flags and mailboxes at rest) and its device-side state.
static lshmoe_status p2p_alloc(lshmoe_comm* c, int E, int64_t recv_cap, int64_t ret_cap, int row_bytes) {
  p2p_release(c);
  c->L = p2p_layout(c->world, E, recv_cap, ret_cap, row_bytes);
  int err = cudaMalloc(&c->window, c->L.bytes);
  if (!err) err = cudaMemset(c->window, 0, c->L.bytes);
  if (!err) err = cudaMalloc(&c->peers_dev, sizeof(uint8_t*) * c->world);
  if (!err) err = cudaMalloc(&c->done, 4 * sizeof(unsigned));
  if (!err) err = cudaMemset(c->done, 0, 4 * sizeof(unsigned));
  if (!err) err = cudaMalloc(&c->recv_rows_dev, sizeof(int32_t) * E);
  if (err) return cuda_status(err, "lshmoe_comm_p2p_init: allocation");
  c->peers.assign(c->world, nullptr);
  c->peer_ipc.assign(c->world, false);
  c->peers[c->rank] = c->window;
  c->p2p_E = E;
  c->dispatched = false;
  int dev = 0, sms = 148;
  if (!cudaGetDevice(&dev)) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  c->p2p_grid = 2 * sms;                   // two 256-thread CTAs per SM
  return LSHMOE_OK;
}

static lshmoe_status p2p_publish_peers(lshmoe_comm* c) {
  const int err = cudaMemcpy(c->peers_dev, c->peers.data(), sizeof(uint8_t*) * c->world, cudaMemcpyHostToDevice);
  return cuda_status(err, "lshmoe_comm_p2p_init: peer table");
}

static lshmoe_status p2p_check(const lshmoe_comm* c, int64_t recv_capacity, int64_t ret_capacity, int row_bytes,
                               int E, const char* fn) {
  if (!c) return set_error(LSHMOE_EINVAL, std::string(fn) + ": comm is NULL");
  if (recv_capacity < 0 || ret_capacity < 0 || row_bytes < 16 || row_bytes % 16 || E < 1 || E % c->world)
    return set_error(LSHMOE_EINVAL, std::string(fn) + ": bad capacity / row_bytes (multiple of 16) / E");
  if (c->world > 8 || E > 256) return set_error(LSHMOE_EUNSUPPORTED, std::string(fn) + ": world <= 8, E <= 256");
  return LSHMOE_OK;
}

lshmoe_status lshmoe_comm_p2p_alloc(lshmoe_comm* c, int64_t recv_capacity, int64_t ret_capacity, int row_bytes,
                                    int E) {
  lshmoe_status st = p2p_check(c, recv_capacity, ret_capacity, row_bytes, E, "lshmoe_comm_p2p_alloc");
  if (st) return st;
  st = p2p_alloc(c, E, recv_capacity, ret_capacity, row_bytes);
  if (st) return st;
  return p2p_publish_peers(c);   // world 1 is complete; world > 1 needs lshmoe_comm_p2p_open
}

lshmoe_status lshmoe_comm_p2p_handle(const lshmoe_comm* c, uint8_t* handle) {
  if (!c || !c->window || !handle) return set_error(LSHMOE_EINVAL, "lshmoe_comm_p2p_handle: no window / NULL");
  cudaIpcMemHandle_t h;
  const int err = cudaIpcGetMemHandle(&h, c->window);
  if (err) return cuda_status(err, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == LSHMOE_P2P_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  std::memcpy(handle, &h, sizeof(h));
  return LSHMOE_OK;
}

lshmoe_status lshmoe_comm_p2p_open(lshmoe_comm* c, const uint8_t* handles) {
  if (!c || !c->window || !handles) return set_error(LSHMOE_EINVAL, "lshmoe_comm_p2p_open: no window / NULL");
  for (int p = 0; p < c->world; ++p) {
    if (p == c->rank || c->peer_ipc[p]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + static_cast<size_t>(p) * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    const int err = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (err) return cuda_status(err, "cudaIpcOpenMemHandle (peer window)");
    c->peers[p] = static_cast<uint8_t*>(ptr);
    c->peer_ipc[p] = true;
  }
  return p2p_publish_peers(c);
}

lshmoe_status lshmoe_comm_p2p_init(lshmoe_comm* c, int64_t recv_capacity, int64_t ret_capacity, int row_bytes,
                                   int E) {
  lshmoe_status st = lshmoe_comm_p2p_alloc(c, recv_capacity, ret_capacity, row_bytes, E);
  if (st || c->world == 1) return st;
  if (!c->nccl) return set_error(LSHMOE_EINVAL, "lshmoe_comm_p2p_init: no NCCL to exchange handles (use _open)");
  constexpr size_t kH = LSHMOE_P2P_HANDLE_BYTES;
  uint8_t* dev = nullptr;
  int err = cudaMalloc(&dev, kH * c->world);
  if (err) return cuda_status(err, "lshmoe_comm_p2p_init: handle buffer");
  std::vector<uint8_t> all(kH * c->world);
  st = lshmoe_comm_p2p_handle(c, all.data() + kH * c->rank);
  if (!st) err = cudaMemcpy(dev + kH * c->rank, all.data() + kH * c->rank, kH, cudaMemcpyHostToDevice);
  if (!st && !err) {
    st = nccl_status(ncclAllGather(dev + kH * c->rank, dev, kH, ncclUint8, c->nccl, nullptr),
                     "ncclAllGather(ipc handles)");
    if (!st) err = cudaMemcpy(all.data(), dev, kH * c->world, cudaMemcpyDeviceToHost);
  }
  cudaFree(dev);
  if (st) return st;
  if (err) return cuda_status(err, "lshmoe_comm_p2p_init: handle exchange");
  return lshmoe_comm_p2p_open(c, all.data());
}

lshmoe_status lshmoe_comm_local_group(int world, int64_t recv_capacity, int64_t ret_capacity, int row_bytes, int E,
                                      lshmoe_comm** out) {
  if (!out || world < 1 || world > 8) return set_error(LSHMOE_EINVAL, "lshmoe_comm_local_group: bad world / out");
  if (recv_capacity < 0 || ret_capacity < 0 || row_bytes < 16 || row_bytes % 16 || E < 1 || E % world || E > 256)
    return set_error(LSHMOE_EINVAL, "lshmoe_comm_local_group: bad sizes");
  std::vector<lshmoe_comm*> cs(world);
  for (int r = 0; r < world; ++r) {
    cs[r] = new lshmoe_comm();
    cs[r]->world = world;
    cs[r]->rank = r;
    cs[r]->local_group = true;
    lshmoe_status st = p2p_alloc(cs[r], E, recv_capacity, ret_capacity, row_bytes);
    if (st) {
      for (int q = 0; q <= r; ++q) lshmoe_comm_destroy(cs[q]);
      return st;
    }
  }
  for (int r = 0; r < world; ++r) {
    for (int p = 0; p < world; ++p) cs[r]->peers[p] = cs[p]->window;   // same process: plain pointers
    cs[r]->p2p_grid = cs[r]->p2p_grid / world > 0 ? cs[r]->p2p_grid / world : 1;   // all ranks co-resident
    lshmoe_status st = p2p_publish_peers(cs[r]);
    if (st) {
      for (int q = 0; q < world; ++q) lshmoe_comm_destroy(cs[q]);
      return st;
    }
  }
  for (int r = 0; r < world; ++r) out[r] = cs[r];
  return LSHMOE_OK;
}


lshmoe_status lshmoe_comm_p2p_set_timeout(lshmoe_comm* c, double seconds) {
  if (!c || !(seconds > 0) || seconds > 1e6) return set_error(LSHMOE_EINVAL, "lshmoe_comm_p2p_set_timeout: bad comm / seconds");
  c->spin_ns = static_cast<unsigned long long>(seconds * 1e9);
  return LSHMOE_OK;
}

lshmoe_status lshmoe_comm_p2p_buffers(lshmoe_comm* c, void** recv, void** returned, int32_t** recv_rows) {
  if (!c || !c->window) return set_error(LSHMOE_EINVAL, "lshmoe_comm_p2p_buffers: no phase-2 window");
  if (recv) *recv = c->window + c->L.recv;
  if (returned) *returned = c->window + c->L.returned;
  if (recv_rows) *recv_rows = c->recv_rows_dev;
  return LSHMOE_OK;
}

lshmoe_status lshmoe_comm_p2p_error(lshmoe_comm* c, int32_t* value, lshmoe_stream stream) {
  if (!c || !c->window || !value) return set_error(LSHMOE_EINVAL, "lshmoe_comm_p2p_error: no window / NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned v = 0;
  int err = cudaMemcpyAsync(&v, c->done + 1, sizeof(v), cudaMemcpyDeviceToHost, s);
  if (!err) err = cudaStreamSynchronize(s);
  if (!err && v) err = cudaMemsetAsync(c->done + 1, 0, sizeof(unsigned), s);
  if (err) return cuda_status(err, "lshmoe_comm_p2p_error");
  *value = static_cast<int32_t>(v);
  if (v & kP2PErrTimeout)
    return set_error(LSHMOE_EDEVICE, "phase-2 exchange: a peer did not arrive within the spin limit "
                                     "(LSHMOE_P2P_TIMEOUT_S); the call's results are invalid");
  if (v) return set_error(LSHMOE_EDEVICE, v & 1 ? "phase-2 dispatch: a receive buffer was too small (rows dropped)"
                                                 : "phase-2 combine: a returned buffer was too small (rows dropped)");
  return LSHMOE_OK;
}

lshmoe_status lshmoe_dispatch_p2p(lshmoe_comm* c, const void* centroids, const int32_t* expert_rows, int grid,
                                  lshmoe_stream stream) {
  if (!c || !c->window) return set_error(LSHMOE_EINVAL, "lshmoe_dispatch_p2p: no phase-2 window");
  if (!expert_rows) return set_error(LSHMOE_EINVAL, "lshmoe_dispatch_p2p: expert_rows is NULL");
  const int g = grid > 0 ? grid : c->p2p_grid;
  const lshmoe_status st = cuda_status(launch_p2p(0, c->peers_dev, c->L, c->world, c->rank, c->p2p_E, centroids,
                                                  expert_rows, c->recv_rows_dev, c->done, g, comm_spin_ns(c),
                                                  stream),
                                       "lshmoe_dispatch_p2p");
  if (!st) c->dispatched = true;
  return st;
}

lshmoe_status lshmoe_combine_p2p(lshmoe_comm* c, const void* expert_out, int grid, lshmoe_stream stream) {
  if (!c || !c->window || !c->dispatched) return set_error(LSHMOE_EINVAL, "lshmoe_combine_p2p: no matching dispatch");
  const int g = grid > 0 ? grid : c->p2p_grid;
  return cuda_status(launch_p2p(1, c->peers_dev, c->L, c->world, c->rank, c->p2p_E, expert_out, nullptr, nullptr,
                                c->done, g, comm_spin_ns(c), stream),
                     "lshmoe_combine_p2p");
}

lshmoe_status lshmoe_comm_destroy(lshmoe_comm* c) {
  if (!c) return LSHMOE_OK;
  p2p_release(c);
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->counts_dev) cudaFree(c->counts_dev);
  if (c->counts_host) cudaFreeHost(c->counts_host);
  if (c->rr_host) cudaFreeHost(c->rr_host);
  delete c;
  return LSHMOE_OK;
}

lshmoe_status lshmoe_comm_last_counts(const lshmoe_comm* c, int32_t* counts, int E) {
  if (!c || !counts) return set_error(LSHMOE_EINVAL, "lshmoe_comm_last_counts: NULL");
  if (c->last_E != E || !c->nccl) return set_error(LSHMOE_EINVAL, "lshmoe_comm_last_counts: no plan for this E");
  std::memcpy(counts, c->counts.data(), sizeof(int32_t) * c->world * E);
  return LSHMOE_OK;
}

lshmoe_status lshmoe_dispatch(lshmoe_comm* c, const void* centroids, lshmoe_dtype dtype, int d,
                              const int32_t* expert_rows, int E, void* recv, int64_t recv_capacity,
                              int32_t* recv_rows, int64_t* recv_total, lshmoe_stream stream) {
  const int world = c ? c->world : 1;
  if (dtype != LSHMOE_F32 && dtype != LSHMOE_BF16) return set_error(LSHMOE_EINVAL, "lshmoe_dispatch: bad dtype");
  if (d < 1 || E < 1 || E % world != 0) return set_error(LSHMOE_EINVAL, "lshmoe_dispatch: bad d / E (E % world != 0, S:L285)");
  if (!centroids || !expert_rows || !recv || !recv_rows) return set_error(LSHMOE_EINVAL, "lshmoe_dispatch: NULL pointer");
  const size_t row_bytes = static_cast<size_t>(d) * (dtype == LSHMOE_F32 ? 4 : 2);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (world == 1 && !(c && c->nccl)) {   // recv_rows [E, 1] == expert_rows: alias it to skip the copy
    int err = launch_local_exchange(centroids, recv == centroids ? nullptr : recv, recv_capacity,
                                    static_cast<int>(row_bytes), expert_rows, E,
                                    recv_rows == expert_rows ? nullptr : recv_rows, stream);
    return cuda_status(err, "lshmoe_dispatch (local)");
  }
  if (!c->nccl) return set_error(LSHMOE_EINVAL, "lshmoe_dispatch: comm has no NCCL (created without an id)");
  lshmoe_status st = ensure_capacity(c, E);
  if (st) return st;
  const int epr = E / world;
  st = nccl_status(ncclAllGather(expert_rows, c->counts_dev, E, ncclInt32, c->nccl, s), "ncclAllGather(counts)");
  if (st) return st;
  int err = cudaMemcpyAsync(c->counts_host, c->counts_dev, sizeof(int32_t) * world * E, cudaMemcpyDeviceToHost, s);
  if (!err) err = cudaStreamSynchronize(s);
  if (err) return cuda_status(err, "lshmoe_dispatch: reading counts");
  st = lshmoe_check_device_error(stream);
  if (st) return st;
  c->counts.assign(c->counts_host, c->counts_host + world * E);
  c->last_E = E;
  const int32_t* cnt = c->counts.data();
  const int me = c->rank;
  std::vector<int64_t> off(E + 1, 0), rpos(static_cast<size_t>(epr) * world + 1, 0);
  st = lshmoe_exchange_plan(world, me, E, cnt, off.data(), rpos.data(), c->rr_host);
  if (st) return st;
  const int64_t total = rpos[static_cast<size_t>(epr) * world];
  if (total > recv_capacity) return set_error(LSHMOE_EINVAL, "lshmoe_dispatch: recv_capacity too small");
  if (recv_total) *recv_total = total;
  err = cudaMemcpyAsync(recv_rows, c->rr_host, sizeof(int32_t) * epr * world, cudaMemcpyHostToDevice, s);
  if (err) return cuda_status(err, "lshmoe_dispatch: recv_rows");
  const char* cbase = static_cast<const char*>(centroids);
  char* rbase = static_cast<char*>(recv);
  // self segments
  for (int el = 0; el < epr; ++el) {
    const int e = me * epr + el;
    const int64_t rows = cnt[me * E + e];
    if (!rows) continue;
    err = cudaMemcpyAsync(rbase + rpos[static_cast<size_t>(el) * world + me] * row_bytes, cbase + off[e] * row_bytes,
                          rows * row_bytes, cudaMemcpyDeviceToDevice, s);
    if (err) return cuda_status(err, "lshmoe_dispatch: self copy");
  }
  st = nccl_status(ncclGroupStart(), "ncclGroupStart");
  if (st) return st;
  for (int p = 0; p < world; ++p) {
    if (p == me) continue;
    for (int el = 0; el < epr; ++el) {
      const int e = p * epr + el;
      const int64_t rows = cnt[me * E + e];
      if (rows) ncclSend(cbase + off[e] * row_bytes, rows * row_bytes, ncclUint8, p, c->nccl, s);
    }
  }
  for (int src = 0; src < world; ++src) {
    if (src == me) continue;
    for (int el = 0; el < epr; ++el) {
      const int64_t rows = cnt[src * E + me * epr + el];
      if (rows) ncclRecv(rbase + rpos[static_cast<size_t>(el) * world + src] * row_bytes, rows * row_bytes, ncclUint8,
                         src, c->nccl, s);
    }
  }
  st = nccl_status(ncclGroupEnd(), "ncclGroupEnd (dispatch)");
  if (st) return st;
  ncclResult_t async_err = ncclSuccess;
  ncclCommGetAsyncError(c->nccl, &async_err);
  return nccl_status(async_err, "dispatch async");
}

lshmoe_status lshmoe_combine(lshmoe_comm* c, const void* expert_out, lshmoe_dtype dtype, int d,
                             const int32_t* expert_rows, int E, void* returned, int64_t returned_capacity,
                             lshmoe_stream stream) {
  const int world = c ? c->world : 1;
  if (dtype != LSHMOE_F32 && dtype != LSHMOE_BF16) return set_error(LSHMOE_EINVAL, "lshmoe_combine: bad dtype");
  if (d < 1 || E < 1 || E % world != 0) return set_error(LSHMOE_EINVAL, "lshmoe_combine: bad d / E");
  if (!expert_out || !expert_rows || !returned) return set_error(LSHMOE_EINVAL, "lshmoe_combine: NULL pointer");
  const size_t row_bytes = static_cast<size_t>(d) * (dtype == LSHMOE_F32 ? 4 : 2);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (world == 1 && !(c && c->nccl)) {
    int err = launch_local_exchange(expert_out, returned == expert_out ? nullptr : returned, returned_capacity,
                                    static_cast<int>(row_bytes), expert_rows, E, nullptr, stream);
    return cuda_status(err, "lshmoe_combine (local)");
  }
  if (!c->nccl) return set_error(LSHMOE_EINVAL, "lshmoe_combine: comm has no NCCL (created without an id)");
  if (c->last_E != E) return set_error(LSHMOE_EINVAL, "lshmoe_combine: no matching dispatch plan on this comm");
  const int epr = E / world;
  const int me = c->rank;
  const int32_t* cnt = c->counts.data();
  std::vector<int64_t> off(E + 1, 0), rpos(static_cast<size_t>(epr) * world + 1, 0);
  std::vector<int32_t> rr(static_cast<size_t>(epr) * world);
  lshmoe_status pst = lshmoe_exchange_plan(world, me, E, cnt, off.data(), rpos.data(), rr.data());
  if (pst) return pst;
  if (off[E] > returned_capacity) return set_error(LSHMOE_EINVAL, "lshmoe_combine: returned_capacity too small");
  const char* obase = static_cast<const char*>(expert_out);
  char* tbase = static_cast<char*>(returned);
  int err;
  for (int el = 0; el < epr; ++el) {
    const int e = me * epr + el;
    const int64_t rows = cnt[me * E + e];
    if (!rows) continue;
    err = cudaMemcpyAsync(tbase + off[e] * row_bytes, obase + rpos[static_cast<size_t>(el) * world + me] * row_bytes,
                          rows * row_bytes, cudaMemcpyDeviceToDevice, s);
    if (err) return cuda_status(err, "lshmoe_combine: self copy");
  }
  lshmoe_status st = nccl_status(ncclGroupStart(), "ncclGroupStart");
  if (st) return st;
  for (int src = 0; src < world; ++src) {          // results go back to their source rank
    if (src == me) continue;
    for (int el = 0; el < epr; ++el) {
      const int64_t rows = cnt[src * E + me * epr + el];
      if (rows) ncclSend(obase + rpos[static_cast<size_t>(el) * world + src] * row_bytes, rows * row_bytes, ncclUint8,
                         src, c->nccl, s);
    }
  }
  for (int p = 0; p < world; ++p) {                // my centroids' results come back from owner p
    if (p == me) continue;
    for (int el = 0; el < epr; ++el) {
      const int e = p * epr + el;
      const int64_t rows = cnt[me * E + e];
      if (rows) ncclRecv(tbase + off[e] * row_bytes, rows * row_bytes, ncclUint8, p, c->nccl, s);
    }
  }
  st = nccl_status(ncclGroupEnd(), "ncclGroupEnd (combine)");
  if (st) return st;
  ncclResult_t async_err = ncclSuccess;
  ncclCommGetAsyncError(c->nccl, &async_err);
  return nccl_status(async_err, "combine async");
}

}  // extern "C"

namespace lshmoe {
// Phase-2 window of `c` for the fused compress + dispatch (lshmoe_compress_p2p in lshmoe.cpp).
int comm_p2p_fuse(lshmoe_comm* c, int E, P2PFuse* out) {
  if (!c || !c->window || !c->peers_dev) return LSHMOE_EINVAL;
  if (E != c->p2p_E) return LSHMOE_EINVAL;
  if (c->local_group && c->world > 1) return LSHMOE_EUNSUPPORTED;
  out->peers = c->peers_dev;
  out->L = c->L;
  out->world = c->world;
  out->me = c->rank;
  out->done = c->done;
  out->recv_rows = c->recv_rows_dev;
  out->grid = c->p2p_grid;
  out->spin_ns = comm_spin_ns(c);
  return LSHMOE_OK;
}
void comm_p2p_mark_dispatched(lshmoe_comm* c) { c->dispatched = true; }

unsigned long long p2p_spin_limit_ns() {
  static unsigned long long v = [] {
    double s = 300.0;
    if (const char* e = getenv("LSHMOE_P2P_TIMEOUT_S")) {
      const double x = atof(e);
      if (x > 0) s = x;
    }
    return static_cast<unsigned long long>(s * 1e9);
  }();
  return v;
}
}  // namespace lshmoe
