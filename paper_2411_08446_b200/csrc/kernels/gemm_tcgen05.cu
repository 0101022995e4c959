// tcgen05 tensor-core kernels (sm_100a): one warp-specialised, persistent TN-GEMM mainloop
// (TMA -> shared memory ring -> single-thread tcgen05.mma -> double-buffered TMEM accumulator)
// with two epilogues:
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
// Roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer, warps 2-5 =
// epilogue (warp w reads TMEM lanes 32*(w%4) .. +31).
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "../abi/lshmoe_internal.h"
#include "common.cuh"
#include "sm100.cuh"

namespace lshmoe {
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;                      // 64 bf16 = 128 B = one SWIZZLE_128B row
constexpr int kThreads = 192;
constexpr int kEpiWarp0 = 2;

template <int BN>
struct Cfg {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (196 * 1024) / kStageBytes > 8 ? 8 : (196 * 1024) / kStageBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct WorkItem {
  int a_row;       // first A row (token / centroid row) of the 128-row tile
  int b_row0;      // first B row (rotation / weight row) of chunk 0
  int nchunks;     // accumulator chunks of BN columns (hash: d / BN; FFN: 1)
  int valid_rows;  // rows of the tile that are real outputs
  int tag0, tag1;  // epilogue-specific (hash: m tile, j; FFN: expert, n0)
};

// ---- schedulers --------------------------------------------------------------------------------
struct HashSched {
  int n, q, d, bn;
  int m_tiles;
  __device__ void init(void*) {}
  __device__ int units() const { return m_tiles * q; }
  __device__ WorkItem get(int u) const {
    WorkItem w;
    const int mt = u / q, j = u - mt * q;      // j fastest: the q units of one token tile run together
    w.a_row = mt * BM;
    w.b_row0 = j * d;
    w.nchunks = d / bn;
    w.valid_rows = min(BM, n - mt * BM);
    w.tag0 = mt;
    w.tag1 = j;
    return w;
  }
};

constexpr int kMaxLocalExperts = 256;

struct FfnSched {
  const int32_t* recv_rows;  // [E_local, world]
  int E_local, world, N, bn;
  // smem tables, filled by init()
  int* seg_start;   // [E_local + 1]
  int* tiles_pre;   // [E_local + 1]
  __device__ void init(void* smem) {
    seg_start = reinterpret_cast<int*>(smem);
    tiles_pre = seg_start + (kMaxLocalExperts + 1);
    if (threadIdx.x == 0) {
      int rows = 0, tiles = 0;
      const int ntn = N / bn;
      for (int e = 0; e < E_local; ++e) {
        seg_start[e] = rows;
        tiles_pre[e] = tiles;
        int r = 0;
        for (int s = 0; s < world; ++s) r += recv_rows[e * world + s];
        rows += r;
        tiles += ((r + BM - 1) / BM) * ntn;
      }
      seg_start[E_local] = rows;
      tiles_pre[E_local] = tiles;
    }
    __syncthreads();
  }
  __device__ int units() const { return tiles_pre[E_local]; }
  __device__ WorkItem get(int u) const {
    int e = 0;
    while (tiles_pre[e + 1] <= u) ++e;
    const int ntn = N / bn;
    const int local = u - tiles_pre[e];
    const int mt = local / ntn, nt = local - mt * ntn;
    WorkItem w;
    w.a_row = seg_start[e] + mt * BM;
    w.b_row0 = e * N + nt * bn;
    w.nchunks = 1;
    w.valid_rows = min(BM, seg_start[e + 1] - w.a_row);
    w.tag0 = e;
    w.tag1 = nt * bn;
    return w;
  }
};

// ---- epilogues ---------------------------------------------------------------------------------
struct ArgmaxEpi {
  int16_t* codes;
  int q;
  float best;
  int bidx;
  bool bneg;
  __device__ void begin(const WorkItem&) {
    best = -1.0f;
    bidx = 0;
    bneg = false;
  }
  __device__ void chunk_begin(const WorkItem&, int) {}
  __device__ void consume(const WorkItem&, int /*row*/, const uint32_t (&r)[32], int col0) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float v = __uint_as_float(r[i]);
      const float a = fabsf(v);
      if (a > best) {           // strict: equal magnitudes keep the smaller (earlier) index
        best = a;
        bidx = col0 + i;
        bneg = v < 0.0f;        // -0.0f is not < 0: a zero winner is '+'
      }
    }
  }
  __device__ void finish(const WorkItem& w, int row) {
    if (row < w.valid_rows) {
      const int t = w.a_row + row;
      codes[static_cast<int64_t>(t) * q + w.tag1] = static_cast<int16_t>(bneg ? -(bidx + 1) : (bidx + 1));
    }
  }
};

struct BiasActEpi {
  const __nv_bfloat16* bias;  // [E_local, N]
  __nv_bfloat16* out;         // [rows, N]
  int N;
  bool relu;
  __device__ void begin(const WorkItem&) {}
  __device__ void chunk_begin(const WorkItem&, int) {}
  __device__ void consume(const WorkItem& w, int row, const uint32_t (&r)[32], int col0) {
    if (row >= w.valid_rows) return;
    const int n0 = w.tag1 + col0;
    const __nv_bfloat16* b = bias + static_cast<int64_t>(w.tag0) * N + n0;
    uint32_t packed[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float v0 = __uint_as_float(r[2 * i]) + __bfloat162float(b[2 * i]);
      float v1 = __uint_as_float(r[2 * i + 1]) + __bfloat162float(b[2 * i + 1]);
      if (relu) {
        v0 = fmaxf(v0, 0.0f);
        v1 = fmaxf(v1, 0.0f);
      }
      __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
      packed[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<int64_t>(w.a_row + row) * N + n0);
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
  }
  __device__ void finish(const WorkItem&, int) {}
};

// ---- the kernel --------------------------------------------------------------------------------
template <int BN, class Sched, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                   Sched sched, Epi epi) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ int sched_tables[2 * (kMaxLocalExperts + 1)];

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int kblocks = K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbarrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  sched.init(sched_tables);   // contains __syncthreads
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int units = sched.units();

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const WorkItem w = sched.get(u);
        for (int c = 0; c < w.nchunks; ++c) {
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
            tma_load_2d(sA + stage * C::kABytes, &tmA, &full[stage], kb * BK, w.a_row);
            tma_load_2d(sB + stage * C::kBBytes, &tmB, &full[stage], kb * BK, w.b_row0 + c * BN);
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
    // ===== MMA issuer (one thread) =====
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const WorkItem w = sched.get(u);
        for (int c = 0; c < w.nchunks; ++c) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + stage * C::kABytes);
            const uint32_t b0 = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              mma_bf16_ss(d_tmem, smem_desc_sw128(a0 + kk * 32), smem_desc_sw128(b0 + kk * 32), idesc,
                          (kb | kk) != 0);
            }
            mma_commit(&empty[stage]);          // frees the smem slot when these MMAs finish
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit(&tfull[acc]);              // accumulator ready for the epilogue
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue warps =====
    const int quad = warp % 4;
    const int row = quad * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const WorkItem w = sched.get(u);
      epi.begin(w);
      for (int c = 0; c < w.nchunks; ++c) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        epi.chunk_begin(w, c);
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN;
#pragma unroll 1
        for (int cb = 0; cb < BN / 32; ++cb) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + cb * 32, r);
          tmem_ld_wait();
          epi.consume(w, row, r, c * BN + cb * 32);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      epi.finish(w, row);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
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
int make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : cudaErrorInvalidValue;
}

template <int BN, class Sched, class Epi>
int launch_tc(const CUtensorMap& a, const CUtensorMap& b, int K, const Sched& s, const Epi& e, int grid,
              cudaStream_t st) {
  auto kern = tc_gemm_kernel<BN, Sched, Epi>;
  static bool configured = false;     // one attribute call per instantiation
  if (!configured) {
    int err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::kSmem);
    if (err) return err;
    configured = true;
  }
  kern<<<grid, kThreads, Cfg<BN>::kSmem, st>>>(a, b, K, s, e);
  count_launches(1);
  return cudaGetLastError();
}

int pick_bn(int N) { return N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : 64); }

template <class Sched, class Epi>
int launch_bn(int bn, const void* A, int64_t a_rows, const void* B, int64_t b_rows, int K, Sched s, Epi e, int grid,
              cudaStream_t st) {
  CUtensorMap ma, mb;
  int err = make_map(&ma, A, a_rows, K, BM);
  if (err) return err;
  err = make_map(&mb, B, b_rows, K, bn);
  if (err) return err;
  s.bn = bn;
  switch (bn) {
    case 256: return launch_tc<256>(ma, mb, K, s, e, grid, st);
    case 128: return launch_tc<128>(ma, mb, K, s, e, grid, st);
    default: return launch_tc<64>(ma, mb, K, s, e, grid, st);
  }
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

int launch_hash_bf16(const void* x, int64_t n, int d, const void* R, int q, int16_t* codes, void* stream) {
  HashSched s;
  s.n = static_cast<int>(n);
  s.q = q;
  s.d = d;
  s.m_tiles = static_cast<int>((n + BM - 1) / BM);
  ArgmaxEpi e;
  e.codes = codes;
  e.q = q;
  const int units = s.m_tiles * q;
  const int grid = units < device_sm_count() ? units : device_sm_count();
  return launch_bn(pick_bn(d), x, n, R, static_cast<int64_t>(q) * d, d, s, e, grid, static_cast<cudaStream_t>(stream));
}

int launch_ffn_bf16(const void* in, int d, int d_ffn, const int32_t* recv_rows, int E_local, int world,
                    const void* W1, const void* b1, const void* W2, const void* b2, void* hidden, int64_t capacity,
                    void* out, void* stream) {
  if (E_local > kMaxLocalExperts) return cudaErrorInvalidValue;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = device_sm_count();
  FfnSched s1{recv_rows, E_local, world, d_ffn, 0, nullptr, nullptr};
  BiasActEpi e1{static_cast<const __nv_bfloat16*>(b1), static_cast<__nv_bfloat16*>(hidden), d_ffn, true};
  int err = launch_bn(pick_bn(d_ffn), in, capacity, W1, static_cast<int64_t>(E_local) * d_ffn, d, s1, e1, grid, st);
  if (err) return err;
  FfnSched s2{recv_rows, E_local, world, d, 0, nullptr, nullptr};
  BiasActEpi e2{static_cast<const __nv_bfloat16*>(b2), static_cast<__nv_bfloat16*>(out), d, false};
  return launch_bn(pick_bn(d), hidden, capacity, W2, static_cast<int64_t>(E_local) * d, d_ffn, s2, e2, grid, st);
}

}  // namespace lshmoe
