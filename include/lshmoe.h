/*
 * lshmoe.h — C ABI of the B200-native LSH-MoE compressed expert-parallel dispatch/combine path.
 *
 * The operations follow Algorithm 1 of "LSH-MoE" (arXiv 2411.08446, App. A,
 * L513-543, cited P:Lnnn).  One MoE layer on one rank is, in order:
 *
 *   lshmoe_hash      Alg. 1 L5   IDX_i <- LSH(X_i), cross-polytope hash Eq. 3
 *   lshmoe_compress  Alg. 1 L3, L5-L12  dispatch X into X_i by zeta, divide each X_i
 *                    into clusters by bucket, centroid = Mean (§2.3)
 *   lshmoe_dispatch  Alg. 1 L14  Input <- all-to-all(C)
 *   lshmoe_expert_ffn Alg. 1 L15 Output <- Expert(Input)   [harness utility]
 *   lshmoe_combine   Alg. 1 L16  E(C) <- all-to-all(Output)
 *   lshmoe_restore   Alg. 1 L17-19 residual compensation Eq. 4-5,
 *                    summed over the k gated experts as in Eq. 2
 *
 * Conventions (all functions):
 *  - Every function returns an lshmoe_status; nothing throws.  On a non-OK status
 *    lshmoe_last_error() returns a thread-local message.
 *  - Pointers are DEVICE pointers unless marked [host].  The caller owns and allocates every
 *    buffer (e.g. torch tensors); the library never allocates device memory on the hot path.
 *    Only lshmoe_comm_init allocates (NCCL communicator + a small pinned host plan buffer).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are stream-ordered and
 *    asynchronous, except lshmoe_rotation (pure host), lshmoe_dispatch at world > 1 (one host
 *    synchronisation to learn the all-to-all-v counts), lshmoe_comm_* and
 *    lshmoe_check_device_error.
 *  - Matrices are row-major.  Token rows (x, centroids, recv, y) must be 16-byte aligned with
 *    pitch d * sizeof(dtype); f32 needs d % 4 == 0, bf16 needs d % 64 == 0 (the tcgen05 hash
 *    tiles K and N in multiples of 64) — else LSHMOE_EUNSUPPORTED.
 *  - Routed copies: copy id c = t*k + s is slot s of token t; zeta (`experts`) is int32 [n, k]
 *    with ids in [0, num_experts) distinct within a row.  Ids out of range raise the
 *    device error word (see LSHMOE_EDEVICE).
 *  - Determinism: every output is a deterministic function of the inputs, independent of the
 *    stream, the world size w and repeated runs.
 *  - Aliasing: y may alias x in lshmoe_restore; at world == 1 recv may equal centroids and
 *    returned may equal expert_out (the exchange is then skipped).  Nothing else may alias.
 */
#ifndef LSHMOE_H_
#define LSHMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSHMOE_ABI_VERSION 1
#define LSHMOE_UNIQUE_ID_BYTES 128
#define LSHMOE_P2P_HANDLE_BYTES 64   /* cudaIpcMemHandle_t */
#define LSHMOE_MAX_Q 16

typedef enum {
  LSHMOE_OK = 0,
  LSHMOE_EINVAL = 1,       /* host-detected bad argument: n < 0, d < 1, q < 1, k < 1, k > E,
                              E % world != 0, NULL required pointer, misaligned pointer,
                              capacity / workspace smaller than required */
  LSHMOE_EUNSUPPORTED = 2, /* valid but outside the kernels' envelope: bf16 with d % 64 != 0,
                              f32 with d % 4 != 0, d > 32767 (int16 codes), q > LSHMOE_MAX_Q,
                              n * k >= 2^31 */
  LSHMOE_ECUDA = 3,        /* CUDA runtime / launch error */
  LSHMOE_ENCCL = 4,        /* NCCL error, including ncclCommGetAsyncError */
  LSHMOE_EDEVICE = 5       /* device-side validation failed (expert id outside [0, E), S:L312;
                              an expert repeated among a token's k slots, "distinct");
                              latched in a device error word, reported by the next call that
                              synchronises (lshmoe_dispatch at world > 1, lshmoe_check_device_error) */
} lshmoe_status;

typedef enum { LSHMOE_F32 = 0, LSHMOE_BF16 = 1 } lshmoe_dtype;   /* token = wire = output dtype */

typedef void* lshmoe_stream;                                     /* cudaStream_t */
typedef struct lshmoe_comm lshmoe_comm;

int lshmoe_abi_version(void);
const char* lshmoe_last_error(void);
/* Cumulative number of CUDA kernels this library has launched in this process (all threads);
   the bench reports the per-step difference as "gpu_launches". */
int64_t lshmoe_kernel_launches(void);
/* Diagnostics switch (default off): when on, lshmoe_compress's kernels record per-CTA globaltimer
   stamps in the header of its workspace (layout: csrc/kernels/compress.cu, kDiag), read by the
   Python binding's compress_diag().  Process-wide; affects launches issued after the call. */
void lshmoe_set_diagnostics(int on);

/* Synchronises `stream`, reads and clears the device error word.  LSHMOE_EDEVICE if a kernel
   latched an error since the last check. */
lshmoe_status lshmoe_check_device_error(lshmoe_stream stream);

/* ---- a1: random rotations (Eq. 3, "R is a random rotation matrix"; reading R3) ------
   Writes q row-major d x d matrices R_j (y = R_j x) to out [host] (q*d*d elements of dtype).
   Recipe (DESIGN.md §3 R3): SplitMix64 counter stream seeded with
   rotation_seed ^ (0x9E3779B97F4A7C15 * (j+1)), Irwin-Hall(12) approximately-Gaussian G_j,
   modified Gram-Schmidt over the columns of G_j in fp64 with left-to-right sums and no FMA,
   R_j = Q_j^T, rounded fp64 -> fp32 (RNE) -> bf16 (RNE) for bf16.  Pure host function,
   deterministic, bit-identical to the independent oracle (tests/test_abi.py, T0). */
lshmoe_status lshmoe_rotation(int d, int q, uint64_t rotation_seed, lshmoe_dtype dtype, void* out);

/* ---- a2: cross-polytope hash, Eq. 3 --------------------------------------------
   x [n, d] dtype, rotation [q, d, d] dtype (from lshmoe_rotation) -> codes int16 [n, q]:
   code_tj = sign(y_i*) * (i*+1), i* = argmax_i |y_i|, y = R_j x_t (reading R1); ties to the
   smallest i, a zero winner is '+' (reading R2).  bf16: tcgen05 tensor cores, bf16 x bf16
   products, fp32 accumulation; f32: SIMT fp32 FMA (reading R19), d <= 352 (else EUNSUPPORTED).
   Hashed once per token, shared by its k routed copies (reading R6).  n == 0 is a no-op.
   workspace: device buffer of lshmoe_hash_workspace() bytes (0 for f32 or d <= 256: may be NULL).
   It must be zero-filled before its first use and not written by anyone else afterwards: it holds
   per-tile arrival counters that every call leaves at zero, plus scratch.  A caller allocates it
   once (e.g. torch.zeros) and reuses it, on one stream at a time. */
lshmoe_status lshmoe_hash_workspace(int64_t n, int d, int q, lshmoe_dtype dtype, size_t* bytes /* [host] */);
lshmoe_status lshmoe_hash(const void* x, lshmoe_dtype dtype, int64_t n, int d,
                          const void* rotation, int q, int16_t* codes,
                          void* workspace, size_t workspace_bytes, lshmoe_stream stream);

/* ---- NEXT-2: gate + hash in one projection (reading R29) ---------------
   One tcgen05 pass over x computes the q cross-polytope codes (as lshmoe_hash) and the gate of
   Eq. 1-2: scores s = W_g x (bf16 products, fp32 accumulation), the k largest (ties to
   the smaller expert id), slots in ascending expert id, weights = softmax over the k selected
   scores.  rotation_gate [q*d + E, d] bf16 = the q rotations followed by the E rows of W_g.
   Outputs: codes int16 [n, q]; zeta int32 [n, k]; gate_weight float [n, k].  bf16 only; E <= 256
   (d <= 256: E <= d), k <= 8.  Workspace as lshmoe_hash's.  Scores within 1e-5 (relative) of the
   k-th/(k+1)-th boundary are near-ties that may resolve differently from exact arithmetic. */
lshmoe_status lshmoe_gate_hash(const void* x, int64_t n, int d, const void* rotation_gate, int q, int num_experts,
                               int k, int16_t* codes, int32_t* zeta, float* gate_weight, void* workspace,
                               size_t workspace_bytes, lshmoe_stream stream);

/* ---- NEXT-2 fp8 option: cross-polytope hash on e4m3 operands (reading R28) ---
   Eq. 3's argmax is invariant to a positive scale of x and, per hash function, of R_j, so both are
   scaled by the largest power of two that keeps their max magnitude <= 448 and rounded to e4m3
   (RNE); the codes are Eq. 3 on those values, computed on kind::f8f6f4 tensor cores (exact e4m3
   products, fp32 accumulation).  This is a different hash of x than lshmoe_hash's (decisions within
   the e4m3 rounding of a tie may differ) and halves the rotation's tensor-core time.
   lshmoe_rotation_e4m3: [host] out q*d*d bytes, from the fp32 lshmoe_rotation of the same seed.
   lshmoe_quantize_e4m3: x bf16 [n, d] -> x8 [n, d] bytes, per-row power-of-two scale; d % 64 == 0.
   lshmoe_hash_e4m3: codes int16 [n, q] from x8 and R8 (device); workspace as lshmoe_hash's. */
lshmoe_status lshmoe_rotation_e4m3(int d, int q, uint64_t rotation_seed, uint8_t* out /* [host] */);
lshmoe_status lshmoe_quantize_e4m3(const void* x, int64_t n, int d, uint8_t* x8, lshmoe_stream stream);
lshmoe_status lshmoe_hash_e4m3(const uint8_t* x8, int64_t n, int d, const uint8_t* rotation8, int q, int16_t* codes,
                               void* workspace, size_t workspace_bytes, lshmoe_stream stream);

/* ---- NEXT-4: structured pseudo-random rotation (Eq. 3's R) ---------------
   Reading R30: x is zero-padded to d' = 1024 and rotated by R_j = H D3_j H D2_j H D1_j (H the
   unnormalised Sylvester Hadamard matrix of order 1024, D_r,j random +-1 diagonals); the code is
   Eq. 3's signed argmax over the 1024 outputs: code_tj = sign(y_i*) (i* + 1), i* in [0, 1024),
   ties to the smallest i, a zero winner '+'.  Codes feed lshmoe_compress like lshmoe_hash's.
   lshmoe_hd3_signs: [host] out [q][3][32] uint32: bit (i % 32) of word (j*3 + r)*32 + i/32 is 1 iff
     D_(r+1),j[i] = -1, where that is bit 63 of SplitMix64 output r*1024 + i + 1 of the stream seeded
     with rotation_seed ^ (0xD1B54A32D192ED03 * (j+1)).  Pure host function, deterministic.
   lshmoe_hash_hd3: x [n, d] dtype (device), signs [q][3][32] (device copy of the above) -> codes
     int16 [n, q].  Three fast Walsh-Hadamard transforms per hash in fp32 on the CUDA cores (no
     tensor cores); the result differs from exact arithmetic only where the oracle's top-two margin
     is below ~1e-5 (reported as near-ties).  Requires d <= 1024, d % 8 == 0 (bf16) / % 4 (f32). */
lshmoe_status lshmoe_hd3_signs(int q, uint64_t rotation_seed, uint32_t* out /* [host] */);
lshmoe_status lshmoe_hash_hd3(const void* x, lshmoe_dtype dtype, int64_t n, int d, const uint32_t* signs, int q,
                              int16_t* codes, lshmoe_stream stream);

/* ---- NEXT-3: spherical-plane (SP) hash, the paper's other evaluated family (§4.5) --
   The paper gives no construction; SPEC's sign-bit reading (reading R26): hash
   function j owns the b unit normals in rows j*b .. j*b+b-1 of `normals`, and
     code_tj = sum_{i<b} [normals[j*b+i] . x_t >= 0] * 2^i        (a zero dot counts as 1)
   codes int16 [n, q] in [0, 2^b), usable as lshmoe_compress's composite key exactly like CP codes.
   normals: device, dtype, row-major with lshmoe_sp_rows(q, b) >= q*b rows of d (rows past q*b
   are read but ignored; e.g. the first b rows of each lshmoe_rotation R_j, zero padded).
   bf16: tcgen05 GEMM with the sign-bit epilogue (products exact, fp32 accumulation); f32: SIMT
   fp32 FMA.  Requires 1 <= b <= 15, q*b <= 256; bf16 d % 64 == 0 (as lshmoe_hash).
   Decisions with |n.x| below 1e-5 * |n||x| are near-ties that may differ from exact arithmetic. */
int lshmoe_sp_rows(int q, int b);
lshmoe_status lshmoe_sp_hash(const void* x, lshmoe_dtype dtype, int64_t n, int d, const void* normals, int q, int b,
                             int16_t* codes, lshmoe_stream stream);

/* ---- a3-a5: group by expert, bucketize, centroid means -------------------------------------
   Bytes of device workspace lshmoe_compress needs for these sizes.  The workspace must be filled
   with 0xFF bytes once before its first use (e.g. cudaMemset(ws, 0xFF, bytes)); every call leaves
   its hash table and arrival counters back in that state, so no per-call clearing is launched.
   It must not be shared by calls in flight on different streams. */
lshmoe_status lshmoe_compress_workspace(int64_t n, int k, int num_experts, int q, int d,
                                        lshmoe_dtype dtype, size_t* bytes /* [host] out */);

/* Inputs: x [n, d] dtype; codes int16 [n, q] (from lshmoe_hash); experts (zeta) int32 [n, k].
   Outputs (capacity n*k rows — no token is ever dropped, reading R20):
     bucket      int32 [n, k]    global centroid row of routed copy (t, s)
     perm        int32 [n*k]     copy ids grouped by centroid row, ascending within a row (R8)
     row_start   int32 [n*k+1]   perm offsets of each row; the first m+1 entries are valid
     expert_rows int32 [E]       m_e = number of centroids of expert e
     num_rows    int32 [1]       m = sum_e m_e
     centroids   dtype [n*k, d]  c~ = RNE(mean) in send layout: expert-major, rows of expert e
                                 at [sum_{e'<e} m_e', ...), local bucket ids in first-appearance
                                 order of the (t, s)-ordered group (reading R7)
     centroids_f32 float [n*k, d] nullable: the fp32 means before rounding (parity tier 2)
   Bucket key = the q-tuple of codes (AND-composite, reading R4); clustering is per
   (rank, expert) group (Alg. 1 L4-L6, reading R5).  Centroid = fp32 sum in a fixed order
   scaled once by the correctly rounded reciprocal of the count (reading R10).  Stream-ordered; no
   host synchronisation.  n*k is bounded by the per-SM shared-memory staging of one perm range
   (about 2700 * SM count copies, ~400K on B200); larger calls fail with an error.
   Ordering: the gate map (experts) is read as soon as the preceding kernel on the stream signals
   its programmatic dependents, before that kernel has finished (the codes only after it has).  This
   holds for any predecessor that does not trigger dependents early, and for lshmoe_hash (it does not
   write the gate map); when the predecessor is lshmoe_gate_hash on the same stream the library waits
   for it first.  LSHMOE_EARLY_GATE=0 disables the early read. */
lshmoe_status lshmoe_compress(const void* x, lshmoe_dtype dtype, int64_t n, int d,
                              const int16_t* codes, int q,
                              const int32_t* experts, int k, int num_experts,
                              int32_t* bucket, int32_t* perm, int32_t* row_start,
                              int32_t* expert_rows, int32_t* num_rows,
                              void* centroids, float* centroids_f32,
                              void* workspace, size_t workspace_bytes, lshmoe_stream stream);

/* ---- a6/a8 communicator ----------------------------------------------------------------------
   Expert placement: rank p owns experts [p*E/w, (p+1)*E/w).  NCCL over NVLink; the
   bootstrap id travels over torch.distributed.  world == 1 needs no id (pass NULL: dispatch /
   combine are then the aliased local exchange); world == 1 WITH an id makes a one-rank NCCL comm
   whose dispatch / combine run the phase-1 code (count all-gather, host plan, self segments,
   grouped send/recv) — phase 1 exercised on one GPU.  id == NULL at world > 1 makes a comm without
   NCCL, usable only by the phase-2 calls below. */
lshmoe_status lshmoe_get_unique_id(uint8_t* id /* [host] LSHMOE_UNIQUE_ID_BYTES */);
lshmoe_status lshmoe_comm_init(const uint8_t* id /* [host] */, int world, int rank,
                               lshmoe_comm** out /* [host] */);
lshmoe_status lshmoe_comm_destroy(lshmoe_comm* comm);
/* Host-side plan of the exchange (pure host, no CUDA; used by dispatch/combine, exported so the
   w-rank layout logic can be tested without GPUs).  counts [host] int32 [world, E]: expert_rows of
   every rank.  Outputs [host]: send_off int64 [E+1] = row offset of expert e in this rank's centroid
   layout; recv_off int64 [E/w*w + 1] = row offset of segment (local expert el, source src) at
   index el*w + src in the receive layout; recv_rows int32 [E/w*w] = its row count. */
lshmoe_status lshmoe_exchange_plan(int world, int rank, int num_experts, const int32_t* counts,
                                   int64_t* send_off, int64_t* recv_off, int32_t* recv_rows);
/* The counts of the last dispatch on this comm: counts [host] int32 [world, E], entry (p, e) =
   expert_rows[e] of rank p.  Only valid at world > 1 after lshmoe_dispatch. */
lshmoe_status lshmoe_comm_last_counts(const lshmoe_comm* comm, int32_t* counts, int num_experts);

/* ---- a6: dispatch, Alg. 1 L14: send only the centroids ------------------------------
   centroids [m, d] in compress's send layout; expert_rows [E] device.  recv [recv_capacity, d]
   receives, on rank p, the rows of p's local experts ordered by (local expert, source rank,
   local bucket) (reading R24); recv_rows int32 [E/w, w] device out = rows per (local expert,
   source).  world > 1: all-gathers the counts (ncclAllGather), synchronises `stream` once to
   read them, then one grouped ncclSend/ncclRecv all-to-all-v; checks the device error word.
   world == 1 (comm may be NULL): a device-side copy bounded by the device count (skipped when
   recv == centroids; the recv_rows copy is skipped when recv_rows == expert_rows, whose [E, 1]
   layout is identical); no host synchronisation.  recv_total [host] (nullable) receives the row
   count at world > 1 (left untouched at world == 1). */
lshmoe_status lshmoe_dispatch(lshmoe_comm* comm, const void* centroids, lshmoe_dtype dtype, int d,
                              const int32_t* expert_rows, int num_experts,
                              void* recv, int64_t recv_capacity, int32_t* recv_rows,
                              int64_t* recv_total, lshmoe_stream stream);

/* ---- a7: expert FFN on the received centroids, Alg. 1 L15 [harness utility] --------
   out = W2 relu(W1 in + b1) + b2 per local expert, rows segmented by recv_rows
   [E_local, world].  W1 [E_local, d_ffn, d], b1 [E_local, d_ffn], W2 [E_local, d, d_ffn],
   b2 [E_local, d] in dtype; hidden [capacity, d_ffn] dtype is scratch; capacity >= rows
   received.  bf16: tcgen05 GEMMs, fp32 accumulation, hidden rounded to bf16; f32: SIMT. */
lshmoe_status lshmoe_expert_ffn(const void* in, lshmoe_dtype dtype, int d, int d_ffn,
                                const int32_t* recv_rows, int experts_local, int world,
                                const void* W1, const void* b1, const void* W2, const void* b2,
                                void* hidden, int64_t capacity, void* out, lshmoe_stream stream);

/* ---- a8: combine, Alg. 1 L16: exact reverse of the last dispatch on `comm` ----------
   expert_out laid out like recv; returned [m, d] receives E(c~) in the centroids' layout. */
lshmoe_status lshmoe_combine(lshmoe_comm* comm, const void* expert_out, lshmoe_dtype dtype, int d,
                             const int32_t* expert_rows, int num_experts, void* returned,
                             int64_t returned_capacity, lshmoe_stream stream);

/* ---- a6/a8 phase 2: device-initiated exchange over peer memory ------------------
   The same all-to-all as lshmoe_dispatch / lshmoe_combine (identical layouts, reading R24) without a
   host synchronisation and without NCCL on the data path: every rank owns a window holding its
   receive and returned buffers, per-epoch count mailboxes and flags; dispatch writes its counts and
   its centroid rows straight into the owners' windows (NVLink stores), combine writes the expert
   outputs straight back into the sources' returned buffers, flag handshakes (system-scope
   release/acquire) complete each call on the device.  All ranks must call dispatch_p2p /
   combine_p2p in the same order; the kernels spin until every peer has arrived, so the kernels of
   all ranks must be able to run concurrently.
   lshmoe_comm_p2p_init: allocates the window (recv_capacity / ret_capacity rows of row_bytes =
     d * sizeof(dtype), a multiple of 16; E % world == 0, world <= 8, E <= 256) and maps every
     peer's window with CUDA IPC (handles all-gathered over the comm's NCCL; collective).
   The same in three steps when the handles travel another way (e.g. torch.distributed, or a comm
   made with id == NULL at world > 1, which has no NCCL and serves phase 2 only):
   lshmoe_comm_p2p_alloc (same arguments; complete at world 1), lshmoe_comm_p2p_handle (this
   window's CUDA IPC handle, LSHMOE_P2P_HANDLE_BYTES [host] out), lshmoe_comm_p2p_open (handles
   [host] world * LSHMOE_P2P_HANDLE_BYTES, rank-major; maps every peer's window).
   lshmoe_comm_local_group: `world` comms in this process sharing one device (virtual ranks, plain
     pointers instead of IPC), for testing the protocol on one GPU; out [host] lshmoe_comm* [world],
     each released with lshmoe_comm_destroy.  Their dispatch_p2p calls must run on distinct streams.
   lshmoe_comm_destroy releases the window and unmaps the peers': every rank must be done with the
     phase-2 calls (e.g. a barrier) before any rank destroys its comm.
   lshmoe_comm_p2p_buffers: the window's recv [recv_capacity, d], returned [ret_capacity, d] and the
     device int32 recv_rows [E/w, w] written by dispatch_p2p (pointers owned by the comm).
   lshmoe_dispatch_p2p: centroids [m, d] (send layout; may be NULL when m == 0) + expert_rows [E]
     device -> every owner's recv / recv_rows.  Row capacities are the caller's contract (not checked on the device).
   lshmoe_combine_p2p: expert_out [rows received, d] in recv layout (may be NULL when no rows were
     received) -> the sources' returned
     buffers (centroid layout), for the last dispatch_p2p.  grid: CTAs per call (<= 0: two per SM, divided by w in a local
     group so that every virtual rank's kernel is resident at once).
   Capacities must be equal on every rank.  Rows that would land past a receive / returned buffer
   are dropped and flagged on the sending rank; lshmoe_comm_p2p_error synchronises `stream`, reads
   and clears the flags (value bit 0: a receive buffer overflowed, bit 1: a returned buffer) and
   returns LSHMOE_EDEVICE when any is set.  A peer that never joins a call (or falls further behind
   than the spin limit, LSHMOE_P2P_TIMEOUT_S seconds, default 300) does not hang the device: the
   waiting kernel gives up, sets value bit 2 and finishes; that call's results are invalid and
   lshmoe_comm_p2p_error returns LSHMOE_EDEVICE (no trap, so the CUDA context survives). */
lshmoe_status lshmoe_comm_p2p_init(lshmoe_comm* comm, int64_t recv_capacity, int64_t ret_capacity,
                                   int row_bytes, int num_experts);
lshmoe_status lshmoe_comm_p2p_alloc(lshmoe_comm* comm, int64_t recv_capacity, int64_t ret_capacity,
                                    int row_bytes, int num_experts);
lshmoe_status lshmoe_comm_p2p_handle(const lshmoe_comm* comm, uint8_t* handle /* [host] */);
lshmoe_status lshmoe_comm_p2p_open(lshmoe_comm* comm, const uint8_t* handles /* [host] */);
lshmoe_status lshmoe_comm_local_group(int world, int64_t recv_capacity, int64_t ret_capacity,
                                      int row_bytes, int num_experts, lshmoe_comm** out);
lshmoe_status lshmoe_comm_p2p_buffers(lshmoe_comm* comm, void** recv, void** returned,
                                      int32_t** recv_rows);
/* a3-a6 fused: lshmoe_compress whose centroid kernel also performs the phase-2 dispatch (Alg. 1 L8
   and L14, SURVEY §8(e) "stores from the centroid kernel"): it posts this rank's per-expert counts,
   reads every source's, and stores each centroid row into its owner's receive buffer as well as into
   `centroids` (restore needs them); its last CTA completes the same flag handshake as
   lshmoe_dispatch_p2p, so the receive buffer and recv_rows of comm's window are complete when it
   ends and lshmoe_combine_p2p follows as usual.  Arguments as lshmoe_compress (no fp32 copy);
   comm must have a phase-2 window for num_experts and rows of d elements.  The kernel occupies every
   SM (one CTA each) and spins on its peers, so every rank needs its own GPU: a local group at
   world > 1 (or ranks sharing a GPU under MPS) returns LSHMOE_EUNSUPPORTED — use lshmoe_compress +
   lshmoe_dispatch_p2p there.  Arguments are validated before anything is launched; only a launched
   call licenses the following lshmoe_combine_p2p. */
lshmoe_status lshmoe_compress_p2p(lshmoe_comm* comm, const void* x, lshmoe_dtype dtype, int64_t n, int d,
                                  const int16_t* codes, int q, const int32_t* experts, int k,
                                  int num_experts, int32_t* bucket, int32_t* perm, int32_t* row_start,
                                  int32_t* expert_rows, int32_t* num_rows, void* centroids,
                                  void* workspace, size_t workspace_bytes, lshmoe_stream stream);
lshmoe_status lshmoe_comm_p2p_error(lshmoe_comm* comm, int32_t* value /* [host] */, lshmoe_stream stream);
/* Peer-wait limit of this comm's phase-2 kernels, in seconds (> 0; default LSHMOE_P2P_TIMEOUT_S or
   300).  Applies to calls issued afterwards (a captured graph keeps the value it was captured with). */
lshmoe_status lshmoe_comm_p2p_set_timeout(lshmoe_comm* comm, double seconds);
lshmoe_status lshmoe_dispatch_p2p(lshmoe_comm* comm, const void* centroids, const int32_t* expert_rows,
                                  int grid, lshmoe_stream stream);
lshmoe_status lshmoe_combine_p2p(lshmoe_comm* comm, const void* expert_out, int grid,
                                 lshmoe_stream stream);

/* ---- a9: residual-based error compensation, Eq. 4-5, Alg. 1 L17-19 -------------
   y_t = sum_s g_ts * (returned[b_ts] + (x_t - centroids[b_ts])), b = bucket [n, k], g = gate_weight
   float [n, k] or NULL (g = 1, Eq. 2 unweighted, reading R13).  The residual is taken against
   the centroid as transmitted (reading R11), so identity experts restore k*x exactly.  fp32
   math, y rounded (RNE) to dtype. */
lshmoe_status lshmoe_restore(const void* x, const void* centroids, const void* returned,
                             lshmoe_dtype dtype, int64_t n, int d, const int32_t* bucket, int k,
                             const float* gate_weight, void* y, lshmoe_stream stream);

/* ---- NEXT-1: backward of the compressed path (reading R27) --------------------------------------
   The paper trains with LSH-MoE but never writes the gradient.  Reading R27: codes and
   buckets are constants, the wire rounding c~ = RNE(mean) is straight-through, and with the
   forward y_t = sum_s g_ts (o_b + x_t - c~_b), c_b = mean of the bucket's x:
     lshmoe_grad_compress  G_b = sum_{(t,s) in b} g_ts dY_t        (dL/do_b), send layout [m, d]
     (G goes to the expert's rank with lshmoe_dispatch; the expert's own backward gives
      H_b = J_E(c~_b)^T G_b; H comes back with lshmoe_combine)
     lshmoe_grad_restore   dX_t = sum_s [ g_ts dY_t + (H_b - G_b) / n_b ],
                           dg_ts = dY_t . (o_b + x_t - c~_b)
   bucket / perm / row_start are lshmoe_compress's outputs of the same forward.  Summation order of
   G is the forward's perm order (fp32 accumulation, one rounding to dtype; grad_out_f32 nullable
   keeps the fp32 sums).  Workspace: lshmoe_grad_compress_workspace(d) bytes, filled with 0xFF once
   before first use and left so by every call (arrival counters of rows cut by CTA ranges). */
/* The expert's backward for the dX path (H = J_E(c~)^T G for E(c) = W2 relu(W1 c + b1) + b2,
   weight gradients not computed): dh = (G W2) * [h > 0], H = dh W1, as two grouped GEMMs over the
   same recv_rows segments as lshmoe_expert_ffn.  W2T [E_local, d_ffn, d] = W2^T and W1T
   [E_local, d, d_ffn] = W1^T per expert (the transposed copies a training framework keeps for its
   backward; K-major for TMA); hidden = the forward's post-ReLU activations [capacity, d_ffn];
   dhidden [capacity, d_ffn] scratch; grad_in (H) [capacity, d] out.  bf16: tcgen05, fp32
   accumulation, dh rounded to bf16; f32: SIMT. */
lshmoe_status lshmoe_expert_ffn_backward(const void* grad_out, lshmoe_dtype dtype, int d, int d_ffn,
                                         const int32_t* recv_rows, int experts_local, int world,
                                         const void* W2T, const void* W1T, const void* hidden, void* dhidden,
                                         int64_t capacity, void* grad_in, lshmoe_stream stream);
lshmoe_status lshmoe_grad_compress_workspace(int d, size_t* bytes /* [host] */);
lshmoe_status lshmoe_grad_compress(const void* dy, lshmoe_dtype dtype, int64_t n, int d,
                                   const float* gate_weight /* nullable [n, k] */, const int32_t* bucket,
                                   const int32_t* perm, const int32_t* row_start, int k,
                                   void* grad_out /* [n*k, d]: rows [0, m) written */,
                                   float* grad_out_f32 /* nullable [n*k, d] */,
                                   void* workspace, size_t workspace_bytes, lshmoe_stream stream);
lshmoe_status lshmoe_grad_restore(const void* dy, const void* x, const void* centroids, const void* returned,
                                  const void* grad_c /* G [m, d] */, const void* grad_ret /* H [m, d] */,
                                  lshmoe_dtype dtype, int64_t n, int d, const int32_t* bucket,
                                  const int32_t* row_start, int k, const float* gate_weight /* nullable */,
                                  void* dx /* out [n, d] */, float* dgate /* out, nullable [n, k] fp32 */,
                                  lshmoe_stream stream);

/* ---- uncompressed expert-parallel baseline (§2.2): same machinery, no LSH ---------
   lshmoe_permute: rows of x copied into send [n*k, d] grouped by expert (ascending (t, s)
   within an expert), slot int32 [n, k] = send row of copy (t, s), expert_rows [E] = n_e.
   lshmoe_unpermute: y_t = sum_s g_ts * returned[slot_ts].  Workspace: lshmoe_compress_workspace. */
lshmoe_status lshmoe_permute(const void* x, lshmoe_dtype dtype, int64_t n, int d,
                             const int32_t* experts, int k, int num_experts,
                             int32_t* slot, int32_t* expert_rows, void* send,
                             void* workspace, size_t workspace_bytes, lshmoe_stream stream);
lshmoe_status lshmoe_unpermute(const void* returned, lshmoe_dtype dtype, int64_t n, int d,
                               const int32_t* slot, int k, const float* gate_weight, void* y,
                               lshmoe_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* LSHMOE_H_ */
