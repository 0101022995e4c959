// a1: random rotation matrices R_j of the cross-polytope hash (Eq. 3, PAPER.md P:L228:
// "R is a random rotation matrix").  The paper fixes no distribution or recipe (DESIGN.md
// reading R3); this file fixes one that is bit-reproducible across implementations:
//   SplitMix64 counter stream -> Irwin-Hall(12) approximately-Gaussian G_j (no libm)
//   -> modified Gram-Schmidt over the columns of G_j in fp64, every sum left-to-right, no FMA
//      (this translation unit is compiled with -ffp-contract=off)
//   -> R_j = Q_j^T -> RNE fp64 -> fp32 (-> RNE bf16).
// Right-looking MGS: after q_i is fixed, every later column is reduced against it; the inner
// loop runs over columns j (independent, vectorisable) while the k-sum order stays sequential.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <vector>

#include "lshmoe_internal.h"

namespace lshmoe {

static inline uint64_t splitmix64_at(uint64_t state0, uint64_t i /* 1-based */) {
  uint64_t z = state0 + i * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// G (row-major d x d, G[r*d + c]) of hash j.
static void gaussian_matrix(int d, uint64_t state0, std::vector<double>& G) {
  const size_t nn = static_cast<size_t>(d) * d;
  G.resize(nn);
  const double scale = 1.0 / 9007199254740992.0;  // 2^-53
  for (size_t e = 0; e < nn; ++e) {
    double g = 0.0;
    for (int i = 0; i < 12; ++i) {
      const uint64_t z = splitmix64_at(state0, 12 * e + i + 1);
      const double u = static_cast<double>(z >> 11) * scale;
      g = (i == 0) ? u : g + u;
    }
    G[e] = g - 6.0;
  }
}

// Q (row-major, columns orthonormal) from G by right-looking modified Gram-Schmidt.
static void mgs_columns(int d, std::vector<double>& A /* in: G, destroyed */, std::vector<double>& Q) {
  Q.assign(static_cast<size_t>(d) * d, 0.0);
  std::vector<double> r(d), qi(d);
  for (int i = 0; i < d; ++i) {
    double ss = 0.0;
    for (int k = 0; k < d; ++k) {
      const double v = A[static_cast<size_t>(k) * d + i];
      const double p = v * v;
      ss = (k == 0) ? p : ss + p;
    }
    const double nrm = std::sqrt(ss);
    for (int k = 0; k < d; ++k) {
      qi[k] = A[static_cast<size_t>(k) * d + i] / nrm;
      Q[static_cast<size_t>(k) * d + i] = qi[k];
    }
    if (i + 1 == d) break;
    // r_j = sum_k qi[k] * A[k][j], sequential in k, for all j > i.
    for (int k = 0; k < d; ++k) {
      const double qk = qi[k];
      const double* row = &A[static_cast<size_t>(k) * d];
      if (k == 0) {
        for (int j = i + 1; j < d; ++j) r[j] = qk * row[j];
      } else {
        for (int j = i + 1; j < d; ++j) r[j] = r[j] + qk * row[j];
      }
    }
    for (int k = 0; k < d; ++k) {
      const double qk = qi[k];
      double* row = &A[static_cast<size_t>(k) * d];
      for (int j = i + 1; j < d; ++j) row[j] = row[j] - qk * r[j];
    }
  }
}

lshmoe_status rotation_host(int d, int q, uint64_t seed, lshmoe_dtype dtype, void* out) {
  std::vector<double> G, Q;
  const size_t nn = static_cast<size_t>(d) * d;
  for (int j = 0; j < q; ++j) {
    const uint64_t state0 = seed ^ (0x9E3779B97F4A7C15ull * static_cast<uint64_t>(j + 1));
    gaussian_matrix(d, state0, G);
    mgs_columns(d, G, Q);
    // R_j[i][k] = Q[k][i]
    if (dtype == LSHMOE_F32) {
      float* o = static_cast<float*>(out) + j * nn;
      for (int i = 0; i < d; ++i)
        for (int k = 0; k < d; ++k) o[static_cast<size_t>(i) * d + k] = static_cast<float>(Q[static_cast<size_t>(k) * d + i]);
    } else {
      uint16_t* o = static_cast<uint16_t*>(out) + j * nn;
      for (int i = 0; i < d; ++i)
        for (int k = 0; k < d; ++k)
          o[static_cast<size_t>(i) * d + k] = f32_to_bf16_rne(static_cast<float>(Q[static_cast<size_t>(k) * d + i]));
    }
  }
  return LSHMOE_OK;
}


// NEXT-2 fp8 option (reading R28): R_j (the fp32-stored rotation) scaled by the largest 2^k with
// max|R_j| * 2^k <= 448 and rounded to e4m3 (round to nearest, ties to even).
static uint8_t f32_to_e4m3_rne(float f) {   // |f| <= 448
  const double a = std::fabs(static_cast<double>(f));
  const uint8_t sign = f < 0 ? 0x80 : 0;
  if (a == 0.0) return sign;
  if (a < 0.015625) {                          // below 2^-6: subnormal grid m * 2^-9
    const double m = std::nearbyint(a * 512.0);   // ties to even (default rounding mode)
    return static_cast<uint8_t>(sign | static_cast<uint8_t>(m));   // m == 8 is the first normal (0x08)
  }
  int e;
  const double fr = std::frexp(a, &e);         // a = fr * 2^e, fr in [0.5, 1)
  int ue = e - 1;                              // a = (2 fr) * 2^ue, 2 fr in [1, 2)
  double m = std::nearbyint((2.0 * fr - 1.0) * 8.0);
  if (m == 8.0) {
    m = 0.0;
    ++ue;
  }
  return static_cast<uint8_t>(sign | static_cast<uint8_t>(((ue + 7) << 3) | static_cast<int>(m)));
}

lshmoe_status rotation_e4m3_host(int d, int q, uint64_t seed, uint8_t* out) {
  std::vector<float> R(static_cast<size_t>(q) * d * d);
  lshmoe_status st = rotation_host(d, q, seed, LSHMOE_F32, R.data());
  if (st != LSHMOE_OK) return st;
  const size_t nn = static_cast<size_t>(d) * d;
  for (int j = 0; j < q; ++j) {
    const float* Rj = R.data() + j * nn;
    float vmax = 0.0f;
    for (size_t i = 0; i < nn; ++i) vmax = std::max(vmax, std::fabs(Rj[i]));
    int k = 0;
    if (vmax > 0.0f) {
      int e;
      const double fr = std::frexp(static_cast<double>(vmax), &e);
      k = fr <= 0.875 ? 9 - e : 8 - e;
    }
    for (size_t i = 0; i < nn; ++i) out[j * nn + i] = f32_to_e4m3_rne(std::ldexp(Rj[i], k));
  }
  return LSHMOE_OK;
}

// NEXT-4 (reading R30): the +-1 diagonals D_1..D_3 of hash j as bit vectors over the d' = 1024
// padded coordinates.  Entry i of round r is -1 iff bit 63 of SplitMix64 output number
// r*1024 + i + 1 of the stream seeded with rotation_seed ^ (0xD1B54A32D192ED03 * (j + 1)) is set;
// out[(j*3 + r)*32 + i/32] bit i%32.
void hd3_signs_host(int q, uint64_t seed, uint32_t* out) {
  for (int j = 0; j < q; ++j) {
    const uint64_t state = seed ^ (0xD1B54A32D192ED03ull * static_cast<uint64_t>(j + 1));
    for (int r = 0; r < 3; ++r)
      for (int w = 0; w < 32; ++w) {
        uint32_t word = 0;
        for (int b = 0; b < 32; ++b) {
          const uint64_t z = splitmix64_at(state, static_cast<uint64_t>(r) * 1024 + 32 * w + b + 1);
          word |= static_cast<uint32_t>(z >> 63) << b;
        }
        out[(j * 3 + r) * 32 + w] = word;
      }
  }
}

}  // namespace lshmoe
