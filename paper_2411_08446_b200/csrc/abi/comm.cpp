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

#include <cstring>
#include <string>
#include <vector>

#include "lshmoe_internal.h"

using namespace lshmoe;

struct lshmoe_comm {
  int world = 1;
  int rank = 0;
  ncclComm_t nccl = nullptr;
  int32_t* counts_dev = nullptr;     // [world * E_cap]
  int32_t* counts_host = nullptr;    // pinned [world * E_cap]
  int32_t* rr_host = nullptr;        // pinned [E_cap] recv_rows staging
  int E_cap = 0;
  int last_E = 0;                    // E of the last dispatch (plan valid iff > 0)
  std::vector<int32_t> counts;       // host copy of the last plan [world * E]
};

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
  if (world > 1 && !id) return set_error(LSHMOE_EINVAL, "lshmoe_comm_init: id is NULL at world > 1");
  auto* c = new lshmoe_comm();
  c->world = world;
  c->rank = rank;
  if (world > 1) {
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

lshmoe_status lshmoe_comm_destroy(lshmoe_comm* c) {
  if (!c) return LSHMOE_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->counts_dev) cudaFree(c->counts_dev);
  if (c->counts_host) cudaFreeHost(c->counts_host);
  if (c->rr_host) cudaFreeHost(c->rr_host);
  delete c;
  return LSHMOE_OK;
}

lshmoe_status lshmoe_comm_last_counts(const lshmoe_comm* c, int32_t* counts, int E) {
  if (!c || !counts) return set_error(LSHMOE_EINVAL, "lshmoe_comm_last_counts: NULL");
  if (c->last_E != E || c->world == 1) return set_error(LSHMOE_EINVAL, "lshmoe_comm_last_counts: no plan for this E");
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
  if (world == 1) {   // recv_rows [E, 1] == expert_rows: alias it to skip the copy
    int err = launch_local_exchange(centroids, recv == centroids ? nullptr : recv, recv_capacity,
                                    static_cast<int>(row_bytes), expert_rows, E,
                                    recv_rows == expert_rows ? nullptr : recv_rows, stream);
    return cuda_status(err, "lshmoe_dispatch (local)");
  }
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
  if (world == 1) {
    int err = launch_local_exchange(expert_out, returned == expert_out ? nullptr : returned, returned_capacity,
                                    static_cast<int>(row_bytes), expert_rows, E, nullptr, stream);
    return cuda_status(err, "lshmoe_combine (local)");
  }
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
