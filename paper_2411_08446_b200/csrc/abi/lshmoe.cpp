// C-ABI surface of liblshmoe.so: argument validation, error reporting and dispatch to the
// sm_100a kernel launchers.  See include/lshmoe.h for the contract of every entry point.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>

#include "lshmoe_internal.h"

namespace lshmoe {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

lshmoe_status set_error(lshmoe_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

lshmoe_status cuda_status(int err, const char* what) {
  if (err == 0) return LSHMOE_OK;
  return set_error(LSHMOE_ECUDA, std::string(what) + ": " + cudaGetErrorString(static_cast<cudaError_t>(err)));
}

}  // namespace lshmoe

using namespace lshmoe;

#define REQUIRE(cond, st, msg)                                  \
  do {                                                          \
    if (!(cond)) return set_error((st), std::string(__func__) + ": " + (msg)); \
  } while (0)

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static size_t dsize(lshmoe_dtype t) { return t == LSHMOE_F32 ? 4 : 2; }

static lshmoe_status check_token_shape(const char* fn, lshmoe_dtype dtype, int64_t n, int d) {
  if (dtype != LSHMOE_F32 && dtype != LSHMOE_BF16) return set_error(LSHMOE_EINVAL, std::string(fn) + ": bad dtype");
  if (n < 0) return set_error(LSHMOE_EINVAL, std::string(fn) + ": n < 0 (S:L146)");
  if (d < 1) return set_error(LSHMOE_EINVAL, std::string(fn) + ": d < 1 (S:L51)");
  if (d > 32767) return set_error(LSHMOE_EUNSUPPORTED, std::string(fn) + ": d > 32767 does not fit int16 codes");
  if (dtype == LSHMOE_BF16 && d % 64 != 0)
    return set_error(LSHMOE_EUNSUPPORTED, std::string(fn) + ": bf16 path needs d % 64 == 0");
  if (dtype == LSHMOE_F32 && d % 4 != 0)
    return set_error(LSHMOE_EUNSUPPORTED, std::string(fn) + ": f32 path needs d % 4 == 0");
  return LSHMOE_OK;
}

extern "C" {

int lshmoe_abi_version(void) { return LSHMOE_ABI_VERSION; }

int64_t lshmoe_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }
void lshmoe_set_diagnostics(int on) { set_compress_diag(on); }

const char* lshmoe_last_error(void) { return g_last_error.c_str(); }

lshmoe_status lshmoe_check_device_error(lshmoe_stream stream) {
  int v = 0;
  int err = read_and_clear_device_error(&v, stream);
  if (err) return cuda_status(err, "lshmoe_check_device_error");
  if (v & 1) return set_error(LSHMOE_EDEVICE, "device error word set: expert id outside [0, E) (S:L312)");
  if (v) return set_error(LSHMOE_EDEVICE, "device error word set: an expert appears twice among a token's k slots "
                                          "(the k experts must be distinct, S:L227)");
  return LSHMOE_OK;
}

lshmoe_status lshmoe_rotation(int d, int q, uint64_t seed, lshmoe_dtype dtype, void* out) {
  REQUIRE(d >= 1, LSHMOE_EINVAL, "d < 1 (S:L51)");
  REQUIRE(q >= 1, LSHMOE_EINVAL, "q < 1");
  REQUIRE(out != nullptr, LSHMOE_EINVAL, "out is NULL");
  REQUIRE(dtype == LSHMOE_F32 || dtype == LSHMOE_BF16, LSHMOE_EINVAL, "bad dtype");
  REQUIRE(d <= 32767, LSHMOE_EUNSUPPORTED, "d > 32767");
  return rotation_host(d, q, seed, dtype, out);
}

lshmoe_status lshmoe_hash_workspace(int64_t n, int d, int q, lshmoe_dtype dtype, size_t* bytes) {
  REQUIRE(bytes != nullptr, LSHMOE_EINVAL, "bytes is NULL");
  REQUIRE(n >= 0 && d >= 1 && q >= 1, LSHMOE_EINVAL, "bad sizes");
  *bytes = dtype == LSHMOE_BF16 ? hash_workspace_bytes(n, d, q) : 0;
  return LSHMOE_OK;
}

lshmoe_status lshmoe_hash(const void* x, lshmoe_dtype dtype, int64_t n, int d, const void* rotation, int q,
                          int16_t* codes, void* workspace, size_t workspace_bytes, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(q >= 1, LSHMOE_EINVAL, "q < 1");
  REQUIRE(q <= LSHMOE_MAX_Q, LSHMOE_EUNSUPPORTED, "q > LSHMOE_MAX_Q");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(x && rotation && codes, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(x) && aligned16(rotation), LSHMOE_EINVAL, "x / rotation must be 16-byte aligned");
  int err;
  if (dtype == LSHMOE_F32) {
    REQUIRE(d <= 352, LSHMOE_EUNSUPPORTED, "f32 (SIMT) hash supports d <= 352 (the x tile is staged in shared memory)");
    err = launch_hash_f32(static_cast<const float*>(x), n, d, static_cast<const float*>(rotation), q, codes, stream);
  } else {
    const size_t need = hash_workspace_bytes(n, d, q);
    REQUIRE(workspace_bytes >= need, LSHMOE_EINVAL, "workspace too small (see lshmoe_hash_workspace)");
    REQUIRE(need == 0 || (workspace && aligned16(workspace)), LSHMOE_EINVAL, "workspace NULL or misaligned");
    err = launch_hash_bf16(x, n, d, rotation, q, codes, workspace, stream);
  }
  return cuda_status(err, "lshmoe_hash");
}

lshmoe_status lshmoe_gate_hash(const void* x, int64_t n, int d, const void* RG, int q, int E, int k, int16_t* codes,
                               int32_t* zeta, float* gw, void* workspace, size_t workspace_bytes, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, LSHMOE_BF16, n, d);
  if (st) return st;
  REQUIRE(q >= 1 && E >= 1 && k >= 1 && k <= E, LSHMOE_EINVAL, "bad q / E / k (k <= E, S:L228)");
  REQUIRE(q <= LSHMOE_MAX_Q && k <= 8 && E <= (d < 256 ? d : 256), LSHMOE_EUNSUPPORTED,
          "gate_hash needs q <= LSHMOE_MAX_Q, k <= 8, E <= min(d, 256)");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(x && RG && codes && zeta && gw && aligned16(x) && aligned16(RG), LSHMOE_EINVAL, "NULL or misaligned pointer");
  const size_t need = hash_workspace_bytes(n, d, q);
  REQUIRE(workspace_bytes >= need, LSHMOE_EINVAL, "workspace too small (see lshmoe_hash_workspace)");
  REQUIRE(need == 0 || (workspace && aligned16(workspace)), LSHMOE_EINVAL, "workspace NULL or misaligned");
  note_gate_hash_stream(stream);   // before the launch: a failed launch only costs the overlap
  return cuda_status(launch_gate_hash_bf16(x, n, d, RG, q, E, k, codes, zeta, gw, workspace, stream),
                     "lshmoe_gate_hash");
}

lshmoe_status lshmoe_rotation_e4m3(int d, int q, uint64_t seed, uint8_t* out) {
  REQUIRE(d >= 1 && q >= 1, LSHMOE_EINVAL, "d < 1 or q < 1");
  REQUIRE(q <= LSHMOE_MAX_Q, LSHMOE_EUNSUPPORTED, "q > LSHMOE_MAX_Q");
  REQUIRE(out != nullptr, LSHMOE_EINVAL, "out is NULL");
  return rotation_e4m3_host(d, q, seed, out);
}

lshmoe_status lshmoe_quantize_e4m3(const void* x, int64_t n, int d, uint8_t* x8, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, LSHMOE_BF16, n, d);
  if (st) return st;
  if (n == 0) return LSHMOE_OK;
  REQUIRE(x && x8 && aligned16(x) && aligned16(x8), LSHMOE_EINVAL, "x / x8 NULL or misaligned");
  return cuda_status(launch_quantize_e4m3(x, n, d, x8, stream), "lshmoe_quantize_e4m3");
}

lshmoe_status lshmoe_hash_e4m3(const uint8_t* x8, int64_t n, int d, const uint8_t* R8, int q, int16_t* codes,
                               void* workspace, size_t workspace_bytes, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, LSHMOE_BF16, n, d);
  if (st) return st;
  REQUIRE(q >= 1, LSHMOE_EINVAL, "q < 1");
  REQUIRE(q <= LSHMOE_MAX_Q, LSHMOE_EUNSUPPORTED, "q > LSHMOE_MAX_Q");
  REQUIRE(d % 128 == 0, LSHMOE_EUNSUPPORTED, "e4m3 hash needs d % 128 == 0");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(x8 && R8 && codes && aligned16(x8) && aligned16(R8), LSHMOE_EINVAL, "NULL or misaligned pointer");
  const size_t need = hash_workspace_bytes(n, d, q);
  REQUIRE(workspace_bytes >= need, LSHMOE_EINVAL, "workspace too small (see lshmoe_hash_workspace)");
  REQUIRE(need == 0 || (workspace && aligned16(workspace)), LSHMOE_EINVAL, "workspace NULL or misaligned");
  return cuda_status(launch_hash_e4m3(x8, n, d, R8, q, codes, workspace, stream), "lshmoe_hash_e4m3");
}

lshmoe_status lshmoe_hd3_signs(int q, uint64_t rotation_seed, uint32_t* out) {
  REQUIRE(q >= 1, LSHMOE_EINVAL, "q < 1");
  REQUIRE(q <= LSHMOE_MAX_Q, LSHMOE_EUNSUPPORTED, "q > LSHMOE_MAX_Q");
  REQUIRE(out != nullptr, LSHMOE_EINVAL, "out is NULL");
  hd3_signs_host(q, rotation_seed, out);
  return LSHMOE_OK;
}

lshmoe_status lshmoe_hash_hd3(const void* x, lshmoe_dtype dtype, int64_t n, int d, const uint32_t* signs, int q,
                              int16_t* codes, lshmoe_stream stream) {
  REQUIRE(dtype == LSHMOE_F32 || dtype == LSHMOE_BF16, LSHMOE_EINVAL, "bad dtype");
  REQUIRE(n >= 0 && d >= 1, LSHMOE_EINVAL, "n < 0 or d < 1");
  REQUIRE(q >= 1, LSHMOE_EINVAL, "q < 1");
  REQUIRE(q <= LSHMOE_MAX_Q, LSHMOE_EUNSUPPORTED, "q > LSHMOE_MAX_Q");
  REQUIRE(d <= 1024, LSHMOE_EUNSUPPORTED, "the structured rotation pads x to 1024: d <= 1024");
  REQUIRE(d % (dtype == LSHMOE_BF16 ? 8 : 4) == 0, LSHMOE_EUNSUPPORTED, "needs d % 8 == 0 (bf16) / d % 4 == 0 (f32)");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(x && signs && codes, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(x), LSHMOE_EINVAL, "x must be 16-byte aligned");
  return cuda_status(launch_hd3_hash(x, dtype == LSHMOE_BF16, n, d, signs, q, codes, stream), "lshmoe_hash_hd3");
}

int lshmoe_sp_rows(int q, int b) { return (q >= 1 && b >= 1 && q * b <= 256) ? sp_rows(q, b) : 0; }

lshmoe_status lshmoe_sp_hash(const void* x, lshmoe_dtype dtype, int64_t n, int d, const void* normals, int q, int b,
                             int16_t* codes, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(q >= 1 && b >= 1, LSHMOE_EINVAL, "q < 1 or b < 1");
  REQUIRE(q <= LSHMOE_MAX_Q && b <= 15 && q * b <= 256, LSHMOE_EUNSUPPORTED, "need q <= LSHMOE_MAX_Q, b <= 15, q*b <= 256");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(x && normals && codes, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(x) && aligned16(normals), LSHMOE_EINVAL, "x / normals must be 16-byte aligned");
  int err;
  if (dtype == LSHMOE_F32) {
    REQUIRE(d <= 352, LSHMOE_EUNSUPPORTED, "f32 (SIMT) SP hash supports d <= 352 (the x tile is staged in shared memory)");
    err = launch_sp_hash_f32(static_cast<const float*>(x), n, d, static_cast<const float*>(normals), q, b, codes, stream);
  } else {
    err = launch_sp_hash_bf16(x, n, d, normals, q, b, codes, stream);
  }
  return cuda_status(err, "lshmoe_sp_hash");
}

lshmoe_status lshmoe_compress_workspace(int64_t n, int k, int E, int q, int d, lshmoe_dtype dtype, size_t* bytes) {
  (void)q;
  (void)dtype;
  REQUIRE(bytes != nullptr, LSHMOE_EINVAL, "bytes is NULL");
  REQUIRE(n >= 0 && k >= 1 && E >= 1 && d >= 1, LSHMOE_EINVAL, "bad sizes");
  REQUIRE(n * k < (int64_t(1) << 31), LSHMOE_EUNSUPPORTED, "n * k >= 2^31");
  *bytes = compress_workspace_layout(n, k, E, d, nullptr, nullptr);
  return LSHMOE_OK;
}

lshmoe_status lshmoe_compress(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int16_t* codes, int q,
                              const int32_t* experts, int k, int E, int32_t* bucket, int32_t* perm,
                              int32_t* row_start, int32_t* expert_rows, int32_t* num_rows, void* centroids,
                              float* centroids_f32, void* workspace, size_t workspace_bytes, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(q >= 1, LSHMOE_EINVAL, "q < 1");
  REQUIRE(q <= LSHMOE_MAX_Q, LSHMOE_EUNSUPPORTED, "q > LSHMOE_MAX_Q");
  REQUIRE(k >= 1 && E >= 1, LSHMOE_EINVAL, "k < 1 or E < 1");
  REQUIRE(k <= E, LSHMOE_EINVAL, "k > E (S:L228)");
  REQUIRE(n * k < (int64_t(1) << 31), LSHMOE_EUNSUPPORTED, "n * k >= 2^31");
  REQUIRE(row_start && expert_rows && num_rows, LSHMOE_EINVAL, "NULL output pointer");
  if (n > 0) {
    REQUIRE(x && codes && experts && bucket && perm && centroids, LSHMOE_EINVAL, "NULL pointer");
    REQUIRE(aligned16(x) && aligned16(centroids) && (!centroids_f32 || aligned16(centroids_f32)),
            LSHMOE_EINVAL, "x / centroids must be 16-byte aligned");
  }
  size_t need = compress_workspace_layout(n, k, E, d, nullptr, nullptr);
  REQUIRE(workspace_bytes >= need, LSHMOE_EINVAL, "workspace too small (see lshmoe_compress_workspace)");
  REQUIRE(need == 0 || (workspace && aligned16(workspace)), LSHMOE_EINVAL, "workspace NULL or misaligned");
  CompressWs ws;
  compress_workspace_layout(n, k, E, d, workspace, &ws);
  int err = launch_compress(x, dtype, n, d, codes, q, experts, k, E, bucket, perm, row_start, expert_rows, num_rows,
                            centroids, centroids_f32, ws, stream);
  return cuda_status(err, "lshmoe_compress");
}

lshmoe_status lshmoe_compress_p2p(lshmoe_comm* comm, const void* x, lshmoe_dtype dtype, int64_t n, int d,
                                  const int16_t* codes, int q, const int32_t* experts, int k, int E, int32_t* bucket,
                                  int32_t* perm, int32_t* row_start, int32_t* expert_rows, int32_t* num_rows,
                                  void* centroids, void* workspace, size_t workspace_bytes, lshmoe_stream stream) {
  P2PFuse fuse;
  const int fst = comm_p2p_fuse(comm, E, &fuse);
  REQUIRE(fst != LSHMOE_EUNSUPPORTED, LSHMOE_EUNSUPPORTED,
          "a local group at world > 1 cannot run the fused kernel (its CTAs occupy every SM, so the virtual "
          "ranks' kernels could not be co-resident): use lshmoe_compress + lshmoe_dispatch_p2p");
  REQUIRE(fst == LSHMOE_OK, LSHMOE_EINVAL,
          "comm has no phase-2 window for this number of experts (lshmoe_comm_p2p_init)");
  REQUIRE(d * (dtype == LSHMOE_F32 ? 4 : 2) == fuse.L.row_bytes, LSHMOE_EINVAL, "row bytes differ from the window's");
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(q >= 1, LSHMOE_EINVAL, "q < 1");
  REQUIRE(q <= LSHMOE_MAX_Q, LSHMOE_EUNSUPPORTED, "q > LSHMOE_MAX_Q");
  REQUIRE(k >= 1 && E >= 1, LSHMOE_EINVAL, "k < 1 or E < 1");
  REQUIRE(k <= E, LSHMOE_EINVAL, "k > E (S:L228)");
  REQUIRE(n * k < (int64_t(1) << 31), LSHMOE_EUNSUPPORTED, "n * k >= 2^31");
  REQUIRE(row_start && expert_rows && num_rows, LSHMOE_EINVAL, "NULL output pointer");
  if (n > 0) {
    REQUIRE(x && codes && experts && bucket && perm && centroids, LSHMOE_EINVAL, "NULL pointer");
    REQUIRE(aligned16(x) && aligned16(centroids), LSHMOE_EINVAL, "x / centroids must be 16-byte aligned");
  }
  size_t need = compress_workspace_layout(n, k, E, d, nullptr, nullptr);
  REQUIRE(workspace_bytes >= need, LSHMOE_EINVAL, "workspace too small (see lshmoe_compress_workspace)");
  REQUIRE(need == 0 || (workspace && aligned16(workspace)), LSHMOE_EINVAL, "workspace NULL or misaligned");
  CompressWs ws;
  compress_workspace_layout(n, k, E, d, workspace, &ws);
  int err = launch_compress(x, dtype, n, d, codes, q, experts, k, E, bucket, perm, row_start, expert_rows, num_rows,
                            centroids, nullptr, ws, stream, &fuse);
  st = cuda_status(err, "lshmoe_compress_p2p");
  if (!st) comm_p2p_mark_dispatched(comm);   // only a launched dispatch licenses a combine
  return st;
}

lshmoe_status lshmoe_expert_ffn_backward(const void* grad_out, lshmoe_dtype dtype, int d, int d_ffn,
                                         const int32_t* recv_rows, int experts_local, int world, const void* W2T,
                                         const void* W1T, const void* hidden, void* dhidden, int64_t capacity,
                                         void* grad_in, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, capacity, d);
  if (st) return st;
  REQUIRE(d_ffn >= 1 && experts_local >= 1 && world >= 1, LSHMOE_EINVAL, "bad sizes");
  if (dtype == LSHMOE_BF16) REQUIRE(d_ffn % 64 == 0, LSHMOE_EUNSUPPORTED, "bf16 FFN needs d_ffn % 64 == 0");
  if (dtype == LSHMOE_F32) REQUIRE(d_ffn % 4 == 0, LSHMOE_EUNSUPPORTED, "f32 FFN needs d_ffn % 4 == 0");
  if (capacity == 0) return LSHMOE_OK;
  REQUIRE(grad_out && recv_rows && W2T && W1T && hidden && dhidden && grad_in, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(grad_out) && aligned16(hidden) && aligned16(dhidden) && aligned16(grad_in) && aligned16(W1T) &&
              aligned16(W2T),
          LSHMOE_EINVAL, "operands must be 16-byte aligned");
  return cuda_status(launch_expert_ffn_backward(grad_out, dtype, d, d_ffn, recv_rows, experts_local, world, W2T, W1T,
                                                hidden, dhidden, capacity, grad_in, stream),
                     "lshmoe_expert_ffn_backward");
}

lshmoe_status lshmoe_grad_compress_workspace(int d, size_t* bytes) {
  REQUIRE(bytes != nullptr && d >= 1, LSHMOE_EINVAL, "bad arguments");
  *bytes = grad_compress_workspace_layout(d, nullptr, nullptr, nullptr);
  return LSHMOE_OK;
}

lshmoe_status lshmoe_grad_compress(const void* dy, lshmoe_dtype dtype, int64_t n, int d, const float* gate_weight,
                                   const int32_t* bucket, const int32_t* perm, const int32_t* row_start, int k,
                                   void* grad_out, float* grad_out_f32, void* workspace, size_t workspace_bytes,
                                   lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(k >= 1, LSHMOE_EINVAL, "k < 1");
  REQUIRE(n * k < (int64_t(1) << 31), LSHMOE_EUNSUPPORTED, "n * k >= 2^31");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(dy && bucket && perm && row_start && grad_out, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(dy) && aligned16(grad_out) && (!grad_out_f32 || aligned16(grad_out_f32)), LSHMOE_EINVAL,
          "dy / grad_out must be 16-byte aligned");
  REQUIRE(workspace && workspace_bytes >= grad_compress_workspace_layout(d, nullptr, nullptr, nullptr), LSHMOE_EINVAL,
          "workspace too small (see lshmoe_grad_compress_workspace)");
  return cuda_status(launch_grad_compress(dy, dtype, n, d, gate_weight, bucket, perm, row_start, k, grad_out,
                                          grad_out_f32, workspace, stream),
                     "lshmoe_grad_compress");
}

lshmoe_status lshmoe_grad_restore(const void* dy, const void* x, const void* ct, const void* ret, const void* G,
                                  const void* H, lshmoe_dtype dtype, int64_t n, int d, const int32_t* bucket,
                                  const int32_t* row_start, int k, const float* g, void* dx, float* dg,
                                  lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(k >= 1, LSHMOE_EINVAL, "k < 1");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(dy && x && ct && ret && G && H && bucket && row_start && dx, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(dy) && aligned16(x) && aligned16(ct) && aligned16(ret) && aligned16(G) && aligned16(H) &&
              aligned16(dx),
          LSHMOE_EINVAL, "rows must be 16-byte aligned");
  return cuda_status(launch_grad_restore(dy, x, ct, ret, G, H, dtype, n, d, bucket, row_start, k, g, dx, dg, stream),
                     "lshmoe_grad_restore");
}

lshmoe_status lshmoe_restore(const void* x, const void* ct, const void* ret, lshmoe_dtype dtype, int64_t n, int d,
                             const int32_t* bucket, int k, const float* g, void* y, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(k >= 1, LSHMOE_EINVAL, "k < 1");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(x && ct && ret && bucket && y, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(x) && aligned16(ct) && aligned16(ret) && aligned16(y), LSHMOE_EINVAL, "rows must be 16-byte aligned");
  return cuda_status(launch_restore(x, ct, ret, dtype, n, d, bucket, k, g, y, stream), "lshmoe_restore");
}

lshmoe_status lshmoe_expert_ffn(const void* in, lshmoe_dtype dtype, int d, int d_ffn, const int32_t* recv_rows,
                                int experts_local, int world, const void* W1, const void* b1, const void* W2,
                                const void* b2, void* hidden, int64_t capacity, void* out, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, capacity, d);
  if (st) return st;
  REQUIRE(d_ffn >= 1 && experts_local >= 1 && world >= 1, LSHMOE_EINVAL, "bad sizes");
  if (dtype == LSHMOE_BF16) REQUIRE(d_ffn % 64 == 0, LSHMOE_EUNSUPPORTED, "bf16 FFN needs d_ffn % 64 == 0");
  if (dtype == LSHMOE_F32) REQUIRE(d_ffn % 4 == 0, LSHMOE_EUNSUPPORTED, "f32 FFN needs d_ffn % 4 == 0");
  if (capacity == 0) return LSHMOE_OK;
  REQUIRE(in && recv_rows && W1 && b1 && W2 && b2 && hidden && out, LSHMOE_EINVAL, "NULL pointer");
  REQUIRE(aligned16(in) && aligned16(hidden) && aligned16(out) && aligned16(W1) && aligned16(W2),
          LSHMOE_EINVAL, "operands must be 16-byte aligned");
  return cuda_status(launch_expert_ffn(in, dtype, d, d_ffn, recv_rows, experts_local, world, W1, b1, W2, b2, hidden,
                                       capacity, out, stream),
                     "lshmoe_expert_ffn");
}

lshmoe_status lshmoe_permute(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int32_t* experts, int k, int E,
                             int32_t* slot, int32_t* expert_rows, void* send, void* workspace, size_t workspace_bytes,
                             lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(k >= 1 && E >= 1 && k <= E, LSHMOE_EINVAL, "bad k / E");
  REQUIRE(n * k < (int64_t(1) << 31), LSHMOE_EUNSUPPORTED, "n * k >= 2^31");
  REQUIRE(expert_rows, LSHMOE_EINVAL, "NULL expert_rows");
  if (n > 0) REQUIRE(x && experts && slot && send && aligned16(x) && aligned16(send), LSHMOE_EINVAL, "bad pointer");
  size_t need = compress_workspace_layout(n, k, E, d, nullptr, nullptr);
  REQUIRE(workspace_bytes >= need, LSHMOE_EINVAL, "workspace too small");
  CompressWs ws;
  compress_workspace_layout(n, k, E, d, workspace, &ws);
  return cuda_status(launch_permute(x, dtype, n, d, experts, k, E, slot, expert_rows, send, ws, stream), "lshmoe_permute");
}

lshmoe_status lshmoe_unpermute(const void* returned, lshmoe_dtype dtype, int64_t n, int d, const int32_t* slot, int k,
                               const float* g, void* y, lshmoe_stream stream) {
  lshmoe_status st = check_token_shape(__func__, dtype, n, d);
  if (st) return st;
  REQUIRE(k >= 1, LSHMOE_EINVAL, "k < 1");
  if (n == 0) return LSHMOE_OK;
  REQUIRE(returned && slot && y && aligned16(returned) && aligned16(y), LSHMOE_EINVAL, "bad pointer");
  return cuda_status(launch_unpermute(returned, dtype, n, d, slot, k, g, y, stream), "lshmoe_unpermute");
}

}  // extern "C"
