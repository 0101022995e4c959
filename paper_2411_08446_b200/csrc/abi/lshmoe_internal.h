// Internal declarations shared by the C-ABI layer (csrc/abi) and the kernel launchers
// (csrc/kernels).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include "../../../include/lshmoe.h"

namespace lshmoe {

// ---- errors -------------------------------------------------------------------------------
lshmoe_status set_error(lshmoe_status st, const std::string& msg);
lshmoe_status cuda_status(int cuda_err, const char* what);   // ECUDA with cudaGetErrorString

// ---- host ---------------------------------------------------------------------------------
lshmoe_status rotation_host(int d, int q, uint64_t seed, lshmoe_dtype dtype, void* out);
lshmoe_status rotation_e4m3_host(int d, int q, uint64_t seed, uint8_t* out);
void hd3_signs_host(int q, uint64_t seed, uint32_t* out);   // NEXT-4 sign bits [q][3][32]
int launch_hd3_hash(const void* x, int is_bf16, int64_t n, int d, const uint32_t* signs, int q, int16_t* codes,
                    void* stream);
int launch_quantize_e4m3(const void* x, int64_t n, int d, uint8_t* out, void* stream);
int launch_gate_hash_bf16(const void* x, int64_t n, int d, const void* RG, int q, int E, int k, int16_t* codes,
                          int32_t* zeta, float* gw, void* ws, void* stream);
int launch_hash_e4m3(const void* x8, int64_t n, int d, const void* R8, int q, int16_t* codes, void* ws, void* stream);

// ---- launchers (csrc/kernels/*.cu); all return cudaError_t as int -------------------------
int launch_hash_f32(const float* x, int64_t n, int d, const float* R, int q, int16_t* codes, void* stream);
int launch_hash_bf16(const void* x, int64_t n, int d, const void* R, int q, int16_t* codes, void* ws, void* stream);
size_t hash_workspace_bytes(int64_t n, int d, int q);
int sp_rows(int q, int b);
int launch_sp_hash_f32(const float* x, int64_t n, int d, const float* N, int q, int b, int16_t* codes, void* stream);
int launch_sp_hash_bf16(const void* x, int64_t n, int d, const void* N, int q, int b, int16_t* codes, void* stream);

struct CompressWs {            // carved from the caller's workspace by compress_workspace_layout
  int32_t* hdr;                // [kHdr] barrier counter, diagnostics stamps, cut-row arrival counters
  int32_t* table;              // [table_size] hash table: slot -> first copy id (follows hdr)
  int64_t table_size;          // power of two >= 2 n k
  int32_t* tile_copy;          // [ntiles * 256] copy ids, each 256-copy tile stably grouped by expert
  int32_t* tile_slot;          // [ntiles * 256] their hash-table slots
  int32_t* tile_off;           // [ntiles][E + 1] start of each expert's run inside a tile
  int32_t* rowid;              // [nk] local centroid row of each first copy (by copy id)
  int32_t* rowl;               // [nk] local row of each perm position (permute mode: perm)
  int32_t* rsl;                // [nk] perm position of each row's first member, at grp_off[e] + row
  int32_t* gofs;               // [E] perm offset of each expert group
  int32_t* big;                // [5][8 nk] K2 slice arrays of groups too large for shared memory
  int32_t* rtot;               // [8 nk] K2 per-(cluster rank, row) totals
  int32_t* fcnt;               // [8 (E + 1)] K2 per-CTA first-appearance counts
  float* partial;              // [kMaxGrid][2][d] centroid partial sums of rows cut by CTA ranges
  size_t bytes;
};
size_t compress_workspace_layout(int64_t n, int k, int E, int d, void* base, CompressWs* ws);

// lshmoe_gate_hash launched on `stream`: the next compress there reads the gate map only after
// griddepcontrol.wait (compress.cu)
void note_gate_hash_stream(void* stream);
int launch_compress(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int16_t* codes, int q,
                    const int32_t* experts, int k, int E, int32_t* bucket, int32_t* perm,
                    int32_t* row_start, int32_t* expert_rows, int32_t* num_rows, void* centroids,
                    float* centroids_f32, const CompressWs& ws, void* stream,
                    const struct P2PFuse* fuse = nullptr);

int launch_permute(const void* x, lshmoe_dtype dtype, int64_t n, int d, const int32_t* experts, int k,
                   int E, int32_t* slot, int32_t* expert_rows, void* send, const CompressWs& ws, void* stream);
int launch_unpermute(const void* returned, lshmoe_dtype dtype, int64_t n, int d, const int32_t* slot, int k,
                     const float* g, void* y, void* stream);

size_t grad_compress_workspace_layout(int d, void* base, int32_t** hdr, float** partial);
int launch_grad_compress(const void* dy, lshmoe_dtype dtype, int64_t n, int d, const float* gw, const int32_t* bucket,
                         const int32_t* perm, const int32_t* row_start, int k, void* grad_out, float* grad_out_f32,
                         void* ws, void* stream);
int launch_grad_restore(const void* dy, const void* x, const void* ct, const void* ret, const void* G, const void* H,
                        lshmoe_dtype dtype, int64_t n, int d, const int32_t* bucket, const int32_t* row_start, int k,
                        const float* g, void* dx, float* dg, void* stream);

int launch_restore(const void* x, const void* ct, const void* ret, lshmoe_dtype dtype, int64_t n, int d,
                   const int32_t* bucket, int k, const float* g, void* y, void* stream);

// Copies rows [0, sum(counts[0..E))) of src to dst (d columns) and counts -> counts_out.
int launch_local_exchange(const void* src, void* dst, int64_t capacity_rows, int row_bytes,
                          const int32_t* counts, int E, int32_t* counts_out, void* stream);

int launch_expert_ffn(const void* in, lshmoe_dtype dtype, int d, int d_ffn, const int32_t* recv_rows,
                      int experts_local, int world, const void* W1, const void* b1, const void* W2,
                      const void* b2, void* hidden, int64_t capacity, void* out, void* stream);

int launch_ffn_bf16(const void* in, int d, int d_ffn, const int32_t* recv_rows, int E_local, int world,
                    const void* W1, const void* b1, const void* W2, const void* b2, void* hidden, int64_t capacity,
                    void* out, void* stream);
int launch_ffn_bwd_bf16(const void* G, int d, int d_ffn, const int32_t* recv_rows, int E_local, int world,
                        const void* W2T, const void* W1T, const void* hidden, void* dhidden, int64_t capacity,
                        void* H, void* stream);
int launch_expert_ffn_backward(const void* grad_out, lshmoe_dtype dtype, int d, int d_ffn, const int32_t* recv_rows,
                               int E_local, int world, const void* W2T, const void* W1T, const void* hidden,
                               void* dhidden, int64_t capacity, void* grad_in, void* stream);

// Phase-2 exchange window (p2p.cu / comm.cpp): byte offsets inside every rank's window.
struct P2PLayout {
  int64_t data_flag, ret_flag;             // uint32 [world] epoch flags
  int64_t mailbox;                         // uint64 [2][world][E] (epoch << 32 | count), by epoch parity
  int64_t recv, returned;                  // row buffers (row_bytes each)
  int64_t recv_capacity, ret_capacity;     // rows
  int row_bytes;
  int64_t bytes;                           // window size
};
// Phase-2 dispatch fused into the centroid kernel (lshmoe_compress_p2p): the kernel posts the counts,
// reads every source's, and stores each centroid row straight into its owner's receive buffer too.
struct P2PFuse {
  uint8_t* const* peers;     // device [world] window bases
  P2PLayout L;
  int world, me;
  unsigned* done;            // [0] arrivals, [1] errors, [2] epoch
  int32_t* recv_rows;        // device [E/world][world] out
  int grid;                  // the comm's phase-2 grid (the nk == 0 fallback launch)
  unsigned long long spin_ns;   // peer-wait limit (then error bit 4, no trap)
};
// comm.cpp: LSHMOE_OK, EINVAL (no window for E) or EUNSUPPORTED (a local group at world > 1: the
// fused kernel needs one CTA per SM, so the virtual ranks could not be co-resident).  Does not mark
// the comm as dispatched: call comm_p2p_mark_dispatched after the launch succeeded.
int comm_p2p_fuse(::lshmoe_comm* c, int E, P2PFuse* out);
void comm_p2p_mark_dispatched(::lshmoe_comm* c);
// Error bits of done[1]: 1 = a receive buffer too small (dispatch), 2 = a returned buffer too small
// (combine), 4 = a peer did not arrive within the spin limit (the call's results are invalid).
constexpr unsigned kP2PErrTimeout = 4u;

int launch_p2p(int which, uint8_t* const* peers_dev, const P2PLayout& L, int world, int me, int E, const void* src,
               const int32_t* expert_rows, int32_t* recv_rows, unsigned* done, int grid, unsigned long long spin_ns,
               void* stream);
// Peer-wait limit of the phase-2 kernels in ns: LSHMOE_P2P_TIMEOUT_S (seconds), default 300 s.
unsigned long long p2p_spin_limit_ns();

int read_and_clear_device_error(int* value, void* stream);
// Programmatic dependent launch for the GEMM and restore kernels (LSHMOE_PDL=0 turns it off, A/B).
bool pdl_enabled();
void set_compress_diag(int on);   // per-CTA globaltimer stamps in the compress workspace header
void count_launches(int n);   // kernels launched by this library (lshmoe_kernel_launches)
int device_sm_count();

}  // namespace lshmoe
