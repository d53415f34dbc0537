// he_rhombus.cu -- K6: the Rhombus PCMv at RLWE degree n = rhombus_degree (4096), restated from
// oracle/he_oracle_rhombus.c (same integer algorithm, so results are bit-exact):
//   (D) decompose  : hybrid key switch (dnum 2, special prime P) of the degree-N input from s to
//                    s'(X^rho), then the free X^rho split into rho RLWE-n pieces
//   (M) MVM        : coefficient-encoded inner products, pt x ct in the NTT domain, summed over pieces
//   (P) packing    : PackLWEs over the n row ciphertexts of each output piece; the automorphisms act
//                    in the NTT domain as index permutations, each followed by a Galois key switch
//   (R)(C)         : rescale by q1 and the free X^rho interleave back to degree N.
// Every stage is a batched kernel launch (all combines of a packing level at once) around the K2
// NTT; nothing runs on the host but the launch sequence.
//
// The file also holds the other key-switching paths, which share the hybrid-key machinery above:
//   - MLWE -> RLWE ring packing of the PCMM output (he_ring_pack_*: key-switch and trace methods),
//   - the slot-domain BSGS PCMM and general slot linear maps (he_slot_*: hoisted rotations with
//     gadget keys),
//   - multi-GPU shards of the PCMv (he_rhombus_run_shard / he_rhombus_combine).
// Each is restated in oracle/he_oracle_rhombus.c and bit-exact with it.
#include <algorithm>
#include <initializer_list>
#include <vector>

#include "he_common.cuh"
#include "he_internal.h"
#include "he_kernels.h"

using namespace he;

namespace {

constexpr uint64_t kStreamSecretRh = 0x5EC1000000000000ULL;
HE_HD uint64_t stream_ksk_a(uint32_t id, uint32_t i, uint32_t j) {
  return 0xC000000000000000ULL | ((uint64_t)id << 16) | ((uint64_t)i << 8) | (uint64_t)j;
}
HE_HD uint64_t stream_ksk_e(uint32_t id, uint32_t i) {
  return 0xCE00000000000000ULL | ((uint64_t)id << 16) | ((uint64_t)i << 8);
}
HE_HD uint32_t half_reverse(uint32_t x, uint32_t n, int logn) {
  return (x & (n >> 1)) | bitrev_h(x & ((n >> 1) - 1), logn - 1);
}
HE_D uint32_t barrett64(uint64_t x, uint64_t mu, uint32_t q) {  // x mod q for any x < 2^64
  const uint64_t qh = __umul64hi(x, mu);
  return csub((uint32_t)(x - qh * q), q);
}

// several same-shape NTT batches (table t[i], base d[i]) as one launch per pass (ntt_*_multi)
static cudaError_t ntt_jobs(bool inverse, std::initializer_list<const NttTable*> t, std::initializer_list<uint32_t*> d,
                            uint32_t count, uint64_t stride, cudaStream_t st) {
  const NttTable* tt[16];
  uint32_t* dd[16];
  int n = 0;
  for (const NttTable* x : t) tt[n++] = x;
  n = 0;
  for (uint32_t* x : d) dd[n++] = x;
  return inverse ? ntt_inverse_multi(tt, dd, n, count, stride, st) : ntt_forward_multi(tt, dd, n, count, stride, st);
}

struct Mods {
  uint32_t m[3];
  uint64_t mu[3];
  RngCtx rng;  // key material for the key generators (k_ksk_prep)
};
HE_D uint32_t mulmod_b(uint32_t a, uint32_t b, uint64_t mu, uint32_t q) { return barrett64((uint64_t)a * b, mu, q); }
// centred c (|c| < q 2^32) -> c mod q
HE_D uint32_t lift_b(int64_t c, uint64_t mu, uint32_t q) {
  return barrett64((uint64_t)(c + ((int64_t)q << 32)), mu, q);
}
Mods make_mods(const RingDims& R) {
  Mods M;
  M.m[0] = R.q[0];
  M.m[1] = R.q[1];
  M.m[2] = R.P;
  for (int j = 0; j < 3; ++j) M.mu[j] = (uint64_t)(((unsigned __int128)1 << 64) / M.m[j]);
  M.rng = R.rng;
  return M;
}

// ------------------------------------------------------------------ key generation
__global__ void k_small_secret(RngCtx rc, uint64_t seed, uint32_t n, uint32_t N, int32_t* s_small, int32_t* s_up) {
  const Rng key = rng_make(rc, seed, kStreamSecretRh);
  const uint32_t rho = N / n;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (i < n) s_small[i] = ternary(rng_next(key, i));
    s_up[i] = (i % rho == 0) ? ternary(rng_next(key, i / rho)) : 0;
  }
}
// sigma_k(s) on a signed secret
__global__ void k_secret_auto(const int32_t* s, uint32_t n, uint32_t k, int32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t j = ((uint64_t)i * k) % (2ull * n);
    if (j < n) out[j] = s[i];
    else out[j - n] = -s[i];
  }
}
__global__ void k_reduce_signed(const int32_t* s, uint32_t n, uint32_t q, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t v = s[i];
    out[i] = v < 0 ? q + v : (uint32_t)v;
  }
}
// alpha (uniform) and t = g * s_old + e  (coefficient form, modulus q)
__global__ void k_ksk_prep(RngCtx rc, uint64_t seed, uint32_t id, uint32_t i, uint32_t j, uint32_t q, uint32_t g,
                           const int32_t* s_old, uint32_t n, uint32_t* alpha, uint32_t* t) {
  const Rng ka = rng_make(rc, seed, stream_ksk_a(id, i, j)), ke = rng_make(rc, seed, stream_ksk_e(id, i));
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    alpha[c] = (uint32_t)(rng_next(ka, c) % q);
    const int64_t e = cbd21_d(rng_next(ke, c));
    const uint64_t gs = (uint64_t)g * from_i64(s_old[c], q) % q;
    t[c] = (uint32_t)((gs + from_i64(e, q)) % q);
  }
}
// beta = t - alpha * s_new   (NTT domain, in place in t)
__global__ void k_ksk_beta(const uint32_t* alpha, const uint32_t* s_new, uint32_t n, uint32_t q, uint32_t* t) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    t[c] = sub_mod(t[c], mul_mod(alpha[c], s_new[c], q), q);
}

// ------------------------------------------------------------------ key switching pieces (batched)
// digits of c (coefficient form, per limb [2][cnt][n]) lifted to the other moduli:
//   d_i = c_i * Qhat_i^-1 mod q_i;  D[j][i] = d_i mod m_j for j != i.  D[i][i] comes from the NTT form.
__global__ void k_modup(const uint32_t* __restrict__ c, const uint32_t* __restrict__ T, uint32_t logn, uint64_t cnt_n,
                        Mods M, uint32_t qhinv0, uint32_t qhinv1, uint32_t* __restrict__ D) {
  // D layout: [j (3)][i (2)][cnt * n];  T layout [L][cnt][2][n] (NTT form, a part = slot 0).  4 words per step.
  const uint32_t q0 = M.m[0], q1 = M.m[1], P = M.m[2];
  const uint64_t nmask = (1ull << logn) - 1;
  for (uint64_t x4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x4 < cnt_n / 4; x4 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = x4 * 4;
    const uint64_t tix = ((x >> logn) << (logn + 1)) + (x & nmask);
    const uint4 c0 = reinterpret_cast<const uint4*>(c)[x4], c1 = reinterpret_cast<const uint4*>(c + cnt_n)[x4];
    const uint4 t0 = *reinterpret_cast<const uint4*>(T + tix), t1 = *reinterpret_cast<const uint4*>(T + 2 * cnt_n + tix);
    const uint32_t d0[4] = {mulmod_b(c0.x, qhinv0, M.mu[0], q0), mulmod_b(c0.y, qhinv0, M.mu[0], q0),
                            mulmod_b(c0.z, qhinv0, M.mu[0], q0), mulmod_b(c0.w, qhinv0, M.mu[0], q0)};
    const uint32_t d1[4] = {mulmod_b(c1.x, qhinv1, M.mu[1], q1), mulmod_b(c1.y, qhinv1, M.mu[1], q1),
                            mulmod_b(c1.z, qhinv1, M.mu[1], q1), mulmod_b(c1.w, qhinv1, M.mu[1], q1)};
    auto put = [&](int slot, uint32_t a, uint32_t b, uint32_t cc, uint32_t dd) {
      reinterpret_cast<uint4*>(D + (size_t)slot * cnt_n)[x4] = make_uint4(a, b, cc, dd);
    };
    put(0 * 2 + 1, barrett64(d1[0], M.mu[0], q0), barrett64(d1[1], M.mu[0], q0), barrett64(d1[2], M.mu[0], q0),
        barrett64(d1[3], M.mu[0], q0));
    put(1 * 2 + 0, barrett64(d0[0], M.mu[1], q1), barrett64(d0[1], M.mu[1], q1), barrett64(d0[2], M.mu[1], q1),
        barrett64(d0[3], M.mu[1], q1));
    put(2 * 2 + 0, barrett64(d0[0], M.mu[2], P), barrett64(d0[1], M.mu[2], P), barrett64(d0[2], M.mu[2], P),
        barrett64(d0[3], M.mu[2], P));
    put(2 * 2 + 1, barrett64(d1[0], M.mu[2], P), barrett64(d1[1], M.mu[2], P), barrett64(d1[2], M.mu[2], P),
        barrett64(d1[3], M.mu[2], P));
    // own-modulus digits straight from the NTT form (NTT is linear mod q_i)
    put(0 * 2 + 0, mulmod_b(t0.x, qhinv0, M.mu[0], q0), mulmod_b(t0.y, qhinv0, M.mu[0], q0),
        mulmod_b(t0.z, qhinv0, M.mu[0], q0), mulmod_b(t0.w, qhinv0, M.mu[0], q0));
    put(1 * 2 + 1, mulmod_b(t1.x, qhinv1, M.mu[1], q1), mulmod_b(t1.y, qhinv1, M.mu[1], q1),
        mulmod_b(t1.z, qhinv1, M.mu[1], q1), mulmod_b(t1.w, qhinv1, M.mu[1], q1));
  }
}
// U[j] = sum_i D[j][i] * K[i][0][j],  W[j] = sum_i D[j][i] * K[i][1][j]   (NTT domain, n a power of two)
// K layout [i][part][j][n];  UW layout [j][2][cnt][n].  4 words per step.
__global__ void k_mac(const uint32_t* __restrict__ D, const uint32_t* __restrict__ K, uint32_t n, uint64_t cnt_n,
                      Mods M, uint32_t* __restrict__ UW) {
  for (uint64_t x4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x4 < cnt_n / 4; x4 += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c4 = (uint32_t)((x4 * 4) & (n - 1)) / 4;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint4 a = reinterpret_cast<const uint4*>(D + (size_t)(j * 2 + 0) * cnt_n)[x4];
      const uint4 b = reinterpret_cast<const uint4*>(D + (size_t)(j * 2 + 1) * cnt_n)[x4];
      const uint4 k00 = __ldg(reinterpret_cast<const uint4*>(K + ((size_t)(0 * 2 + 0) * 3 + j) * n) + c4);
      const uint4 k10 = __ldg(reinterpret_cast<const uint4*>(K + ((size_t)(1 * 2 + 0) * 3 + j) * n) + c4);
      const uint4 k01 = __ldg(reinterpret_cast<const uint4*>(K + ((size_t)(0 * 2 + 1) * 3 + j) * n) + c4);
      const uint4 k11 = __ldg(reinterpret_cast<const uint4*>(K + ((size_t)(1 * 2 + 1) * 3 + j) * n) + c4);
      const uint64_t mu = M.mu[j];
      const uint32_t q = M.m[j];
      auto f = [&](uint32_t d0, uint32_t d1, uint32_t x0, uint32_t x1) {
        return barrett64((uint64_t)d0 * x0 + (uint64_t)d1 * x1, mu, q);
      };
      reinterpret_cast<uint4*>(UW + (size_t)(j * 2 + 0) * cnt_n)[x4] =
          make_uint4(f(a.x, b.x, k00.x, k10.x), f(a.y, b.y, k00.y, k10.y), f(a.z, b.z, k00.z, k10.z), f(a.w, b.w, k00.w, k10.w));
      reinterpret_cast<uint4*>(UW + (size_t)(j * 2 + 1) * cnt_n)[x4] =
          make_uint4(f(a.x, b.x, k01.x, k11.x), f(a.y, b.y, k01.y, k11.y), f(a.z, b.z, k01.z, k11.z), f(a.w, b.w, k01.w, k11.w));
    }
  }
}
// ModDown, first half: centred lift of the (coefficient-form) P parts to q0, q1.  LB [j][2][cnt][n]
__global__ void k_moddown_lift(const uint32_t* __restrict__ UWP, uint64_t cnt_n, Mods M, uint32_t* __restrict__ LB) {
  const uint32_t P = M.m[2];
  for (uint64_t x4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x4 < cnt_n / 2; x4 += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(UWP)[x4];
    const uint32_t vs[4] = {v.x, v.y, v.z, v.w};
    uint32_t l0[4], l1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t c = vs[e] > P / 2 ? (int64_t)vs[e] - P : (int64_t)vs[e];
      l0[e] = lift_b(c, M.mu[0], M.m[0]);
      l1[e] = lift_b(c, M.mu[1], M.m[1]);
    }
    reinterpret_cast<uint4*>(LB)[x4] = make_uint4(l0[0], l0[1], l0[2], l0[3]);
    reinterpret_cast<uint4*>(LB + 2 * cnt_n)[x4] = make_uint4(l1[0], l1[1], l1[2], l1[3]);
  }
}

// ------------------------------------------------------------------ decompose (degree N)
__global__ void k_decomp_modup(const uint32_t* __restrict__ ct, uint32_t N, uint32_t q0, uint32_t q1, uint32_t P,
                               uint32_t qhinv0, uint32_t qhinv1, uint32_t* __restrict__ D) {
  // ct [2 limbs][2][N]; D [j][i][N] (coefficient form: all six lifts, NTT'd afterwards)
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < N; x += gridDim.x * blockDim.x) {
    const uint32_t d0 = mul_mod(ct[x], qhinv0, q0);
    const uint32_t d1 = mul_mod(ct[2 * (size_t)N + x], qhinv1, q1);
    D[0 * (size_t)N + x] = d0;            // j=0,i=0
    D[1 * (size_t)N + x] = d1 % q0;       // j=0,i=1
    D[2 * (size_t)N + x] = d0 % q1;       // j=1,i=0
    D[3 * (size_t)N + x] = d1;            // j=1,i=1
    D[4 * (size_t)N + x] = d0 % P;
    D[5 * (size_t)N + x] = d1 % P;
  }
}
// (u, w) mod q_j from UW (coefficient form, [j][2][N]), then the X^rho split:
//   pieces [L][p][2][n]:  a = u[p + rho k],  b = b_in[p + rho k] + w[p + rho k]
__global__ void k_decomp_split(const uint32_t* __restrict__ UW, const uint32_t* __restrict__ ct, uint32_t N,
                               uint32_t n, uint32_t p_in, uint32_t piece0, uint32_t q0, uint32_t q1, uint32_t P,
                               uint32_t pinv0, uint32_t pinv1, uint32_t* __restrict__ pieces) {
  const uint32_t rho = N / n;
  const uint32_t total = p_in * n;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const uint32_t p = x / n, k = x % n;
    const size_t src = piece0 + p + (size_t)rho * k;   // input piece piece0 + p of the degree-N vector
#pragma unroll
    for (int L = 0; L < 2; ++L) {
      const uint32_t q = L ? q1 : q0, pinv = L ? pinv1 : pinv0;
      int64_t up = UW[(2 * 2 + 0) * (size_t)N + src], wp = UW[(2 * 2 + 1) * (size_t)N + src];
      if (up > P / 2) up -= P;
      if (wp > P / 2) wp -= P;
      const uint32_t u = mul_mod(from_i64((int64_t)UW[(L * 2 + 0) * (size_t)N + src] - up, q), pinv, q);
      const uint32_t w = mul_mod(from_i64((int64_t)UW[(L * 2 + 1) * (size_t)N + src] - wp, q), pinv, q);
      const uint32_t b = ct[(L * 2 + 1) * (size_t)N + src];
      uint32_t* dst = pieces + (((size_t)L * p_in + p) * 2) * n;
      dst[k] = u;
      dst[n + k] = add_mod(b, w, q);
    }
  }
}

// ------------------------------------------------------------------ weights (plan)
// Windowed (split-point) plaintexts, oracle or_rhombus_pcmv_w.  Window w = n / U, U = 2^s rows per product:
//   pt_{o,j,p}(X) = w^-1 sum_{u<U} X^{u w} sum_{i<w} W~[r(o,j,u)][w p + i] X^{-h_w(i)},  r = n o + h_n(u w + j)
// Coefficient pos of pt: pos = 0 -> (u 0, h 0); pos in [1, n - w] -> u = ceil(pos / w), h = u w - pos;
// pos in (n - w, n) -> u = 0, h = n - pos, negated (X^-h = -X^{n-h}).  Leaf jl of output piece o in a
// leaf-interleaved shard (G groups, this plan's group g) is global leaf j = g + G jl.
// Wpt [L][leaf][p][n] coefficient form before the NTT.
__global__ void k_rh_weights(const double* __restrict__ W, uint32_t n_out, uint32_t n_in, uint32_t n, int logn,
                             uint32_t win, int logw, uint32_t G, uint32_t g, uint32_t p_in, uint64_t leaves, uint32_t q0,
                             uint32_t q1, uint32_t cp0, uint32_t cp1, double delta_w, uint32_t* __restrict__ out) {
  const uint64_t per_l = leaves * p_in * n;
  const uint32_t lpp = win / G;  // leaves per output piece in this plan
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < per_l; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t pos = (uint32_t)(x % n);
    const uint64_t lp = x / n;
    const uint32_t p = (uint32_t)(lp % p_in);
    const uint64_t leaf = lp / p_in;
    const uint32_t o = (uint32_t)(leaf / lpp), j = g + G * (uint32_t)(leaf % lpp);
    uint32_t u, hw;
    bool neg = false;
    if (pos == 0) {
      u = 0;
      hw = 0;
    } else if (pos <= n - win) {
      u = (pos + win - 1) >> logw;
      hw = u * win - pos;
    } else {
      u = 0;
      hw = n - pos;
      neg = true;
    }
    const uint32_t r = n * o + half_reverse(u * win + j, n, logn);
    const uint32_t col = win * p + (win < 2 ? 0u : half_reverse(hw, win, logw));
    long long wv = 0;
    if (r < n_out && col < n_in) wv = __double2ll_rn(__dmul_rn(delta_w, W[(size_t)r * n_in + col]));
#pragma unroll
    for (int L = 0; L < 2; ++L) {
      const uint32_t q = L ? q1 : q0;
      uint32_t v = mul_mod(from_i64(wv, q), L ? cp1 : cp0, q);
      if (neg && v) v = q - v;
      out[(size_t)L * per_l + lp * n + pos] = v;
    }
  }
}

// rows [L][leaf][2][n] = sum_p Wpt[L][leaf][p][.] * pieces[L][p][ab][.]   (NTT domain); 4 coefficients per
// thread (16-byte loads and stores: the kernel streams the 0.5-2 GB of plaintexts once)
__global__ void k_rh_mvm(const uint32_t* __restrict__ Wpt, const uint32_t* __restrict__ pieces, uint64_t leaves,
                         uint32_t p_in, uint32_t logn, Mods M, uint32_t* __restrict__ rows) {
  const uint32_t n = 1u << logn, L = blockIdx.y;
  const uint64_t per_l4 = (leaves << logn) >> 2;
  const uint32_t q = M.m[L];
  const uint64_t mu = M.mu[L];
  for (uint64_t y4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y4 < per_l4; y4 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t y = y4 << 2, leaf = y >> logn;
    const uint32_t c = (uint32_t)(y & (n - 1));
    const uint32_t* w = Wpt + ((size_t)L * leaves + leaf) * p_in * n + c;
    const uint32_t* pc = pieces + (size_t)L * p_in * 2 * n + c;
    uint64_t aa[4] = {0, 0, 0, 0}, ab[4] = {0, 0, 0, 0};
    for (uint32_t p = 0; p < p_in; ++p) {
      const uint4 wv = __ldcs(reinterpret_cast<const uint4*>(w + (size_t)p * n));
      const uint4 xa = __ldg(reinterpret_cast<const uint4*>(pc + (size_t)p * 2 * n));
      const uint4 xb = __ldg(reinterpret_cast<const uint4*>(pc + (size_t)p * 2 * n + n));
      const uint32_t wvs[4] = {wv.x, wv.y, wv.z, wv.w}, xas[4] = {xa.x, xa.y, xa.z, xa.w}, xbs[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        aa[e] += (uint64_t)wvs[e] * xas[e];
        ab[e] += (uint64_t)wvs[e] * xbs[e];
      }
      if ((p & 7) == 7) {  // keep the sums below 2^64: 8 products < 2^63
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          aa[e] = barrett64(aa[e], mu, q);
          ab[e] = barrett64(ab[e], mu, q);
        }
      }
    }
    uint32_t* dst = rows + (((size_t)L * leaves + leaf) * 2) * n + c;
    reinterpret_cast<uint4*>(dst)[0] = make_uint4(barrett64(aa[0], mu, q), barrett64(aa[1], mu, q),
                                                  barrett64(aa[2], mu, q), barrett64(aa[3], mu, q));
    reinterpret_cast<uint4*>(dst + n)[0] = make_uint4(barrett64(ab[0], mu, q), barrett64(ab[1], mu, q),
                                                      barrett64(ab[2], mu, q), barrett64(ab[3], mu, q));
  }
}

// ------------------------------------------------------------------ packing level
// A [L][cnt_in][2][n] -> Ut into An [L][cnt_out][2][n]; T = sigma(E - M O) [L][cnt_out][2][n];
// C = copy of T's a part [L][cnt_out][n] for the INTT.  One CTA per (limb, combine, a/b): E - M O is
// built in shared memory with coalesced global reads, then permuted out of it.
__global__ void __launch_bounds__(512) k_pack_comb1(const uint32_t* __restrict__ A, uint32_t cnt_in, uint32_t half,
                                                    uint32_t n, const uint32_t* __restrict__ mono /* [2][n] */,
                                                    const uint32_t* __restrict__ perm, Mods M,
                                                    uint32_t* __restrict__ An, uint32_t* __restrict__ T,
                                                    uint32_t* __restrict__ C) {
  extern __shared__ uint32_t sd[];  // [n]  E - M O
  const uint32_t cnt_out = cnt_in / 2;
  const uint32_t idx = blockIdx.x, ab = blockIdx.y, L = blockIdx.z;
  const uint32_t o = idx / half, s_ = idx % half;
  const uint32_t e_i = o * 2 * half + s_, o_i = e_i + half;
  const uint32_t q = M.m[L];
  const uint64_t mu = M.mu[L];
  const uint4* Eb = reinterpret_cast<const uint4*>(A + (((size_t)L * cnt_in + e_i) * 2 + ab) * n);
  const uint4* Ob = reinterpret_cast<const uint4*>(A + (((size_t)L * cnt_in + o_i) * 2 + ab) * n);
  const uint4* ml = reinterpret_cast<const uint4*>(mono + (size_t)L * n);
  uint4* un = reinterpret_cast<uint4*>(An + (((size_t)L * cnt_out + idx) * 2 + ab) * n);
  // 4 coefficients per thread and step: 16-byte global and shared accesses
  for (uint32_t c4 = threadIdx.x; c4 < n / 4; c4 += blockDim.x) {
    const uint4 e = Eb[c4], od = Ob[c4], mm = __ldg(ml + c4);
    const uint32_t mo0 = mulmod_b(od.x, mm.x, mu, q), mo1 = mulmod_b(od.y, mm.y, mu, q);
    const uint32_t mo2 = mulmod_b(od.z, mm.z, mu, q), mo3 = mulmod_b(od.w, mm.w, mu, q);
    un[c4] = make_uint4(add_mod(e.x, mo0, q), add_mod(e.y, mo1, q), add_mod(e.z, mo2, q), add_mod(e.w, mo3, q));
    reinterpret_cast<uint4*>(sd)[c4] =
        make_uint4(sub_mod(e.x, mo0, q), sub_mod(e.y, mo1, q), sub_mod(e.z, mo2, q), sub_mod(e.w, mo3, q));
  }
  __syncthreads();
  uint4* t = reinterpret_cast<uint4*>(T + (((size_t)L * cnt_out + idx) * 2 + ab) * n);
  uint4* cc = reinterpret_cast<uint4*>(C + ((size_t)L * cnt_out + idx) * n);
  const uint4* pp = reinterpret_cast<const uint4*>(perm);
  for (uint32_t c4 = threadIdx.x; c4 < n / 4; c4 += blockDim.x) {
    const uint4 pc = __ldg(pp + c4);
    const uint4 v = make_uint4(sd[pc.x], sd[pc.y], sd[pc.z], sd[pc.w]);
    t[c4] = v;
    if (ab == 0) cc[c4] = v;
  }
}
// An += (u, T_b + w) with u = (U - LB_u) P^-1, w = (W - LB_w) P^-1   (NTT domain)
__global__ void k_pack_comb2(const uint32_t* __restrict__ UW, const uint32_t* __restrict__ LB,
                             const uint32_t* __restrict__ T, uint32_t cnt, uint32_t logn, Mods M, uint32_t pinv0,
                             uint32_t pinv1, uint32_t* __restrict__ An) {
  const uint32_t n = 1u << logn, L = blockIdx.y;
  const uint64_t cnt_n = (uint64_t)cnt << logn;
  const uint32_t q = M.m[L], pinv = L ? pinv1 : pinv0;
  const uint64_t mu = M.mu[L];
  const uint4* U = reinterpret_cast<const uint4*>(UW + (L * 2 + 0) * cnt_n);
  const uint4* W = reinterpret_cast<const uint4*>(UW + (L * 2 + 1) * cnt_n);
  const uint4* LU = reinterpret_cast<const uint4*>(LB + (L * 2 + 0) * cnt_n);
  const uint4* LW = reinterpret_cast<const uint4*>(LB + (L * 2 + 1) * cnt_n);
  for (uint64_t y4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y4 < cnt_n / 4; y4 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t y = y4 * 4, idx = y >> logn;
    const uint32_t c = (uint32_t)(y & (n - 1));
    const uint4 u4 = U[y4], w4 = W[y4], lu = LU[y4], lw = LW[y4];
    uint4* dst = reinterpret_cast<uint4*>(An + (((size_t)L * cnt + idx) * 2) * n + c);
    const uint4 tb = *reinterpret_cast<const uint4*>(T + (((size_t)L * cnt + idx) * 2 + 1) * n + c);
    const uint4 a0 = dst[0], b0 = dst[n / 4];
    auto ua = [&](uint32_t uu, uint32_t ll, uint32_t acc) {
      return add_mod(acc, mulmod_b(sub_mod(uu, ll, q), pinv, mu, q), q);
    };
    auto wb = [&](uint32_t ww, uint32_t ll, uint32_t t, uint32_t acc) {
      return add_mod(acc, add_mod(t, mulmod_b(sub_mod(ww, ll, q), pinv, mu, q), q), q);
    };
    dst[0] = make_uint4(ua(u4.x, lu.x, a0.x), ua(u4.y, lu.y, a0.y), ua(u4.z, lu.z, a0.z), ua(u4.w, lu.w, a0.w));
    dst[n / 4] = make_uint4(wb(w4.x, lw.x, tb.x, b0.x), wb(w4.y, lw.y, tb.y, b0.y), wb(w4.z, lw.z, tb.z, b0.z),
                            wb(w4.w, lw.w, tb.w, b0.w));
  }
}
// shard output (level 1, no rescale), composed: out [L][ab][N], piece o at o0 + o + rho k (zeros elsewhere)
__global__ void k_rh_compose_l1(const uint32_t* __restrict__ A, uint32_t p_out, uint32_t o0, uint32_t n, uint32_t N,
                                uint32_t* __restrict__ out) {
  const uint32_t rho = N / n;
  const uint64_t per_l = (uint64_t)p_out * 2 * n;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < 2 * per_l; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t L = (uint32_t)(x / per_l);
    const uint64_t r = x % per_l;
    const uint32_t k = (uint32_t)(r % n), ab = (uint32_t)((r / n) % 2), o = (uint32_t)(r / (2ull * n));
    out[((size_t)L * 2 + ab) * N + o0 + o + (size_t)rho * k] = A[x];
  }
}
// leaf-interleaved shards: roots [G][L][p_out][2][n] (each shard's packed subtree roots, NTT domain)
// -> A [L][p_out G][2][n] with root (o, g) at o G + g, the order the top log2 G packing levels pair
__global__ void k_rh_gather_roots(const uint32_t* __restrict__ roots, uint32_t G, uint32_t p_out, uint32_t n,
                                  uint32_t* __restrict__ A) {
  const uint64_t per = (uint64_t)2 * p_out * 2 * n;  // one shard's words
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < per * G; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t g = (uint32_t)(x / per);
    const uint64_t r = x % per;
    const uint32_t c = (uint32_t)(r % (2ull * n));
    const uint64_t lo = r / (2ull * n);
    const uint32_t o = (uint32_t)(lo % p_out), L = (uint32_t)(lo / p_out);
    A[(((uint64_t)L * p_out * G + (uint64_t)o * G + g) * 2) * n + c] = roots[x];
  }
}
// sum of shard outputs mod q_L, then rescale by q1:  parts [count][2 limbs][2][N] -> out [2][N]
__global__ void k_rh_combine(const uint32_t* __restrict__ parts, uint32_t count, uint32_t N, uint32_t q0, uint32_t q1,
                             uint32_t q1inv, uint32_t q1invp, uint32_t* __restrict__ out) {
  const size_t per = (size_t)4 * N;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < 2 * N; x += gridDim.x * blockDim.x) {
    uint32_t s0 = 0, s1 = 0;
    for (uint32_t i = 0; i < count; ++i) {
      s0 = add_mod(s0, parts[i * per + x], q0);
      s1 = add_mod(s1, parts[i * per + 2 * (size_t)N + x], q1);
    }
    uint32_t t;
    if (s1 > (q1 >> 1)) t = csub(s0 + (q1 - s1), q0);
    else t = sub_mod(s0, s1, q0);
    out[x] = shoup_mul(t, q1inv, q1invp, q0);
  }
}
// rescale by q1 and compose: out[ab][o + rho k]  (A coefficient form [L][p_out][2][n])
__global__ void k_rh_rescale_compose(const uint32_t* __restrict__ A, uint32_t p_out, uint32_t n, uint32_t N,
                                     uint32_t q0, uint32_t q1, uint32_t q1inv, uint32_t q1invp, uint32_t* __restrict__ out) {
  const uint32_t rho = N / n;
  const uint64_t per_l = (uint64_t)p_out * 2 * n;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < per_l; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = (uint32_t)(x % n);
    const uint32_t ab = (uint32_t)((x / n) % 2);
    const uint32_t o = (uint32_t)(x / (2ull * n));
    const uint32_t x0 = A[x], x1 = A[per_l + x];
    uint32_t t;
    if (x1 > (q1 >> 1)) t = csub(x0 + (q1 - x1), q0);
    else t = sub_mod(x0, x1, q0);
    out[(size_t)ab * N + o + (size_t)rho * k] = shoup_mul(t, q1inv, q1invp, q0);
  }
}

inline dim3 grid_for(uint64_t work, int threads = 256) {
  uint64_t b = (work + threads - 1) / threads;
  if (b > 148ull * 64) b = 148ull * 64;
  if (b == 0) b = 1;
  return dim3((unsigned)b);
}

int ilog2_u(uint32_t x) { return ilog2_h(x); }

}  // namespace

// ======================================================================== plan / C ABI
// A plan covers the window w (split point s = log2(n / w)) and, for leaf-interleaved multi-GPU shards,
// the leaves j = g + G jl of every output piece (G = 1: all of them).
struct he_rhombus_plan {
  const he_context* ctx;
  uint32_t n_out, n_in, p_in, p_out, n, N, logn;
  uint32_t win, logw, split;  // window w = n >> split
  uint32_t G, logG, g;        // leaf groups (shards) and this plan's group
  const uint32_t* wpt;        // caller-owned [2][leaves][p_in][n] NTT domain
  uint32_t* tables;           // owned: perm [logn][n], mono [logn][2][n]
  Mods M;
  uint32_t qhinv[2], pinv[2], q1inv, q1invp;
};

static uint64_t leaves_of(const he_rhombus_plan* p) { return (uint64_t)p->p_out * (p->win / p->G); }

// Hybrid key-switching key from s_old to s_new (degree deg; moduli q0, q1, P), NTT domain:
//   ksk[i][0][j] = alpha (uniform),  ksk[i][1][j] = g_{i,j} s_old + e - alpha s_new   (oracle or_ksk_gen)
static he_status make_ksk_dev(const Mods& M, uint64_t seed, uint32_t id, const int32_t* s_old, const int32_t* s_new,
                              uint32_t deg, const NttTable* tabs, uint32_t* ksk, cudaStream_t st) {
  uint32_t* snew = nullptr;  // s_new NTT per modulus [3][deg]
  HE_CUDA(cudaMallocAsync(&snew, 3ull * deg * sizeof(uint32_t), st), "alloc");
  for (int j = 0; j < 3; ++j) {
    k_reduce_signed<<<grid_for(deg), 256, 0, st>>>(s_new, deg, M.m[j], snew + (size_t)j * deg);
    HE_CUDA(ntt_forward(tabs[j], snew + (size_t)j * deg, 1, deg, st), "NTT(s_new)");
  }
  for (uint32_t i = 0; i < 2; ++i)
    for (uint32_t j = 0; j < 3; ++j) {
      const uint32_t q = M.m[j];
      // g_{i,j} = P * Qhat_i mod q_j for j == i, else 0  (Qhat_0 = q1, Qhat_1 = q0)
      const uint32_t g = (j == i) ? (uint32_t)((uint64_t)(M.m[2] % q) * (M.m[1 - i] % q) % q) : 0u;
      uint32_t* alpha = ksk + ((size_t)(i * 2 + 0) * 3 + j) * deg;
      uint32_t* beta = ksk + ((size_t)(i * 2 + 1) * 3 + j) * deg;
      k_ksk_prep<<<grid_for(deg), 256, 0, st>>>(M.rng, seed, id, i, j, q, g, s_old, deg, alpha, beta);
      HE_CUDA(ntt_forward(tabs[j], alpha, 1, deg, st), "NTT(alpha)");
      HE_CUDA(ntt_forward(tabs[j], beta, 1, deg, st), "NTT(t)");
      k_ksk_beta<<<grid_for(deg), 256, 0, st>>>(alpha, snew + (size_t)j * deg, deg, q, beta);
    }
  cudaFreeAsync(snew, st);
  return HE_OK;
}

extern "C" he_status he_rhombus_keygen(const he_context* c, uint64_t seed, const int32_t* s_dev, int32_t* s_small_dev,
                                       int32_t* s_up_dev, uint32_t* s_up_ntt_dev, uint32_t* ksk_dec_dev,
                                       uint32_t* gal_dev, void* stream) {
  if (!c || !s_dev || !s_small_dev || !s_up_dev || !s_up_ntt_dev || !ksk_dec_dev || !gal_dev)
    return fail(HE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N, n = c->R.n_rh;
  const int logn = ilog2_u(n);
  const Mods M = make_mods(c->R);
  k_small_secret<<<grid_for(N), 256, 0, st>>>(c->R.rng, seed, n, N, s_small_dev, s_up_dev);
  for (int L = 0; L < 2; ++L) {
    uint32_t* dst = s_up_ntt_dev + (size_t)L * N;
    k_reduce_signed<<<grid_for(N), 256, 0, st>>>(s_up_dev, N, M.m[L], dst);
    HE_CUDA(ntt_forward(c->ntt[L], dst, 1, N, st), "NTT(s_up)");
  }
  auto make_ksk = [&](uint32_t id, const int32_t* s_old, const int32_t* s_new, uint32_t deg, const NttTable* tabs,
                      uint32_t* ksk) { return make_ksk_dev(M, seed, id, s_old, s_new, deg, tabs, ksk, st); };
  he_status s = make_ksk(0, s_dev, s_up_dev, N, c->ntt, ksk_dec_dev);
  if (s) return s;
  int32_t* sk = nullptr;
  HE_CUDA(cudaMallocAsync(&sk, n * sizeof(int32_t), st), "alloc");
  for (int lv = 1; lv <= logn; ++lv) {
    const uint32_t k = (1u << lv) + 1;
    k_secret_auto<<<grid_for(n), 256, 0, st>>>(s_small_dev, n, k, sk);
    s = make_ksk(1 + lv, sk, s_small_dev, n, c->ntt_rh, gal_dev + (size_t)(lv - 1) * 12 * n);
    if (s) break;
  }
  cudaFreeAsync(sk, st);
  if (s) return s;
  return cudaGetLastError() == cudaSuccess ? HE_OK : fail(HE_ECUDA, "rhombus keygen launch failed");
}

// shape checks shared by the weight / plan entry points
static he_status rh_shape(const he_context* c, uint32_t n_out, uint32_t n_in, uint32_t win, uint32_t G, uint32_t g,
                          uint32_t* p_in, uint32_t* p_out) {
  if (!c) return fail(HE_EINVAL, "null argument");
  if (!n_out || !n_in) return fail(HE_EINVAL, "empty weight matrix");
  const uint32_t n = c->R.n_rh, rho = c->R.N / n;
  if (win == 0 || win > n || (win & (win - 1)))
    return fail(HE_EINVAL, "window %u must be a power of two in [1, %u]", win, n);
  if (G == 0 || (G & (G - 1)) || G > win || g >= G)
    return fail(HE_EINVAL, "leaf groups %u (group %u) must be a power of two <= the window %u", G, g, win);
  *p_in = (n_in + win - 1) / win;
  *p_out = (n_out + n - 1) / n;
  if (*p_in > rho || *p_out > rho)
    return fail(HE_EINVAL, "dim mismatch: vector dims (%u, %u) exceed %u pieces (input window %u, output %u)", n_out,
                n_in, rho, win, n);
  return HE_OK;
}

extern "C" he_status he_rhombus_weight_bytes_w(const he_context* c, uint32_t n_out, uint32_t n_in, uint32_t window,
                                               uint32_t groups, uint64_t* bytes) {
  uint32_t p_in, p_out;
  he_status s = rh_shape(c, n_out, n_in, window, groups, 0, &p_in, &p_out);
  if (s) return s;
  if (!bytes) return fail(HE_EINVAL, "null argument");
  *bytes = 2ull * p_out * (window / groups) * p_in * c->R.n_rh * sizeof(uint32_t);
  return HE_OK;
}

extern "C" he_status he_rhombus_weight_bytes(const he_context* c, uint32_t n_out, uint32_t n_in, uint64_t* bytes) {
  if (!c) return fail(HE_EINVAL, "null argument");
  return he_rhombus_weight_bytes_w(c, n_out, n_in, c->R.n_rh, 1, bytes);
}

extern "C" he_status he_rhombus_encode_weights_w(const he_context* c, const double* w_dev, uint32_t n_out,
                                                 uint32_t n_in, uint32_t window, uint32_t groups, uint32_t group,
                                                 uint32_t* wpt_dev, void* stream) {
  uint32_t p_in, p_out;
  he_status s = rh_shape(c, n_out, n_in, window, groups, group, &p_in, &p_out);
  if (s) return s;
  if (!w_dev || !wpt_dev) return fail(HE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t n = c->R.n_rh;
  const uint64_t leaves = (uint64_t)p_out * (window / groups);
  const Mods M = make_mods(c->R);
  const uint32_t cp0 = (uint32_t)powmod_h(window, M.m[0] - 2, M.m[0]);
  const uint32_t cp1 = (uint32_t)powmod_h(window, M.m[1] - 2, M.m[1]);
  k_rh_weights<<<grid_for(leaves * p_in * n), 256, 0, st>>>(w_dev, n_out, n_in, n, ilog2_u(n), window,
                                                            ilog2_u(window), groups, group, p_in, leaves, M.m[0],
                                                            M.m[1], cp0, cp1, (double)M.m[1], wpt_dev);
  for (int L = 0; L < 2; ++L)
    HE_CUDA(ntt_forward(c->ntt_rh[L], wpt_dev + (size_t)L * leaves * p_in * n, (uint32_t)(leaves * p_in), n, st),
            "NTT(weights)");
  return HE_OK;
}

extern "C" he_status he_rhombus_encode_weights(const he_context* c, const double* w_dev, uint32_t n_out, uint32_t n_in,
                                               uint32_t* wpt_dev, void* stream) {
  if (!c) return fail(HE_EINVAL, "null argument");
  return he_rhombus_encode_weights_w(c, w_dev, n_out, n_in, c->R.n_rh, 1, 0, wpt_dev, stream);
}

extern "C" he_status he_rhombus_plan_create_w(const he_context* c, const uint32_t* wpt_dev, uint32_t n_out,
                                              uint32_t n_in, uint32_t window, uint32_t groups, uint32_t group,
                                              he_rhombus_plan** out) {
  uint32_t p_in, p_out;
  he_status s = rh_shape(c, n_out, n_in, window, groups, group, &p_in, &p_out);
  if (s) return s;
  if (!wpt_dev || !out) return fail(HE_EINVAL, "null argument");
  he_rhombus_plan* p = new (std::nothrow) he_rhombus_plan();
  if (!p) return fail(HE_ENOMEM, "out of host memory");
  p->ctx = c;
  p->n = c->R.n_rh;
  p->N = c->R.N;
  p->logn = (uint32_t)ilog2_u(p->n);
  p->n_out = n_out;
  p->n_in = n_in;
  p->p_in = p_in;
  p->p_out = p_out;
  p->win = window;
  p->logw = (uint32_t)ilog2_u(window);
  p->split = p->logn - p->logw;
  p->G = groups;
  p->logG = (uint32_t)ilog2_u(groups);
  p->g = group;
  p->wpt = wpt_dev;
  p->M = make_mods(c->R);
  for (int i = 0; i < 2; ++i) {
    const uint32_t qi = p->M.m[i];
    p->qhinv[i] = (uint32_t)powmod_h(p->M.m[1 - i] % qi, qi - 2, qi);
    p->pinv[i] = (uint32_t)powmod_h(p->M.m[2] % qi, qi - 2, qi);
  }
  p->q1inv = (uint32_t)powmod_h(p->M.m[1] % p->M.m[0], p->M.m[0] - 2, p->M.m[0]);
  p->q1invp = shoup_pre(p->q1inv, p->M.m[0]);
  // NTT-domain automorphism permutations and monomials X^{n/2^l}: output c of the forward
  // transform holds p(psi^{2 brv(c) + 1})
  const uint32_t n = p->n, logn = p->logn;
  std::vector<uint32_t> h((size_t)logn * n * 3);
  uint32_t* perm = h.data();
  uint32_t* mono = h.data() + (size_t)logn * n;
  for (uint32_t lv = 1; lv <= logn; ++lv) {
    const uint64_t k = (1u << lv) + 1;
    for (uint32_t cc = 0; cc < n; ++cc) {
      const uint64_t e = 2ull * bitrev_h(cc, (int)logn) + 1;
      const uint64_t ek = (e * k) % (2ull * n);
      perm[(size_t)(lv - 1) * n + cc] = bitrev_h((uint32_t)((ek - 1) / 2), (int)logn);
    }
    for (int L = 0; L < 2; ++L) {
      const uint32_t q = p->M.m[L];
      // psi: the root the NTT tables use (same search as ntt_table_init)
      uint64_t psi = 0;
      for (uint64_t g = 2; g < q; ++g) {
        uint64_t cand = powmod_h(g, (q - 1) / (2ull * n), q);
        if (powmod_h(cand, n, q) == q - 1) {
          psi = cand;
          break;
        }
      }
      const uint64_t ex = n >> lv;
      for (uint32_t cc = 0; cc < n; ++cc) {
        const uint64_t e = 2ull * bitrev_h(cc, (int)logn) + 1;
        mono[((size_t)(lv - 1) * 2 + L) * n + cc] = (uint32_t)powmod_h(psi, (e * ex) % (2ull * n), q);
      }
    }
  }
  if (cudaMalloc(&p->tables, h.size() * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemcpy(p->tables, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    delete p;
    return fail(HE_ECUDA, "rhombus tables");
  }
  *out = p;
  return HE_OK;
}

extern "C" he_status he_rhombus_plan_create(const he_context* c, const uint32_t* wpt_dev, uint32_t n_out, uint32_t n_in,
                                            he_rhombus_plan** out) {
  if (!c) return fail(HE_EINVAL, "null argument");
  return he_rhombus_plan_create_w(c, wpt_dev, n_out, n_in, c->R.n_rh, 1, 0, out);
}

extern "C" he_status he_rhombus_plan_info(const he_rhombus_plan* p, uint32_t* info) {
  if (!p || !info) return fail(HE_EINVAL, "null argument");
  info[0] = p->win;
  info[1] = p->split;
  info[2] = p->G;
  info[3] = p->g;
  info[4] = p->p_in;
  info[5] = p->p_out;
  info[6] = (uint32_t)leaves_of(p);
  return HE_OK;
}

extern "C" he_status he_rhombus_plan_destroy(he_rhombus_plan* p) {
  if (p) {
    if (p->tables) cudaFree(p->tables);
    delete p;
  }
  return HE_OK;
}

// workspace carve-up (words); the packing buffers hold max(leaves, p_out G) ciphertexts (the finish
// of a leaf-interleaved shard packs p_out G roots)
struct RhWs {
  uint32_t *pieces, *A0, *A1, *T, *C, *D, *UW, *LB, *dD, *dUW;
};
static uint64_t rh_ws_words(const he_rhombus_plan* p, RhWs* w, uint32_t* base) {
  const uint64_t n = p->n, N = p->N;
  const uint64_t cap = std::max<uint64_t>(leaves_of(p), (uint64_t)p->p_out * p->G);
  const uint64_t c1 = std::max<uint64_t>(cap / 2, 1);
  uint64_t off = 0;
  auto take = [&](uint32_t*& ptr, uint64_t words) {
    if (w) ptr = base + off;
    off += (words + 63) & ~63ull;
  };
  RhWs dummy;
  RhWs& r = w ? *w : dummy;
  take(r.pieces, 2ull * p->p_in * 2 * n);
  take(r.A0, 2ull * cap * 2 * n);
  take(r.A1, 2ull * c1 * 2 * n);
  take(r.T, 2ull * c1 * 2 * n);
  take(r.C, 2ull * c1 * n);
  take(r.D, 6ull * c1 * n);
  take(r.UW, 6ull * c1 * n);
  take(r.LB, 4ull * c1 * n);
  take(r.dD, 6ull * N);
  take(r.dUW, 6ull * N);
  return off;
}

extern "C" he_status he_rhombus_workspace_bytes(const he_rhombus_plan* p, uint64_t* bytes) {
  if (!p || !bytes) return fail(HE_EINVAL, "null argument");
  *bytes = rh_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  return HE_OK;
}

// PackLWEs levels lv_first..lv_last over cnt ciphertexts (A in w.A0, NTT domain); level lv combines
// E + X^{n/2^lv} O + sigma_{2^lv + 1}(E - X^{n/2^lv} O) with O the leaf n/2^lv further on -- which, in a
// leaf-interleaved shard holding every G-th leaf, is (n/2^lv)/G positions further in A (stride = G).
// Returns the buffer holding the result.
static he_status rh_pack(const he_rhombus_plan* p, const RhWs& w, const uint32_t* gal, uint32_t cnt, uint32_t lv_first,
                         uint32_t lv_last, uint32_t stride, uint32_t** result, cudaStream_t st) {
  const he_context* c = p->ctx;
  const uint32_t n = p->n;
  uint32_t* A = w.A0;
  uint32_t* An = w.A1;
  const uint32_t* perm_base = p->tables;
  const uint32_t* mono_base = p->tables + (size_t)p->logn * n;
  for (uint32_t lv = lv_first; lv <= lv_last; ++lv) {
    const uint32_t cnt_out = cnt / 2, half = (n >> lv) / stride;
    const uint64_t cn = (uint64_t)cnt_out * n;
    k_pack_comb1<<<dim3(cnt_out, 2, 2), 512, n * sizeof(uint32_t), st>>>(
        A, cnt, half, n, mono_base + (size_t)(lv - 1) * 2 * n, perm_base + (size_t)(lv - 1) * n, p->M, An, w.T, w.C);
    const NttTable *t0 = &c->ntt_rh[0], *t1 = &c->ntt_rh[1], *t2 = &c->ntt_rh[2];
    HE_CUDA(ntt_jobs(true, {t0, t1}, {w.C, w.C + cn}, cnt_out, n, st), "INTT(T_a)");
    k_modup<<<grid_for(cn), 256, 0, st>>>(w.C, w.T, p->logn, cn, p->M, p->qhinv[0], p->qhinv[1], w.D);
    HE_CUDA(ntt_jobs(false, {t0, t1, t2, t2}, {w.D + (0 * 2 + 1) * cn, w.D + (1 * 2 + 0) * cn, w.D + 4 * cn, w.D + 5 * cn},
                     cnt_out, n, st), "NTT(digits)");
    k_mac<<<grid_for(cn), 256, 0, st>>>(w.D, gal + (size_t)(lv - 1) * 12 * n, n, cn, p->M, w.UW);
    HE_CUDA(ntt_inverse(c->ntt_rh[2], w.UW + 2 * 2 * cn, 2 * cnt_out, n, st), "INTT(U_P, W_P)");
    k_moddown_lift<<<grid_for(2 * cn), 256, 0, st>>>(w.UW + 2 * 2 * cn, cn, p->M, w.LB);
    HE_CUDA(ntt_jobs(false, {t0, t1}, {w.LB, w.LB + 2 * cn}, 2 * cnt_out, n, st), "NTT(lift)");
    {
      dim3 g = grid_for(cn / 4);
      g.y = 2;
      k_pack_comb2<<<g, 256, 0, st>>>(w.UW, w.LB, w.T, cnt_out, p->logn, p->M, p->pinv[0], p->pinv[1], An);
    }
    // ping-pong: outputs alternate A1, A0, A1, ... (each level's output fits the other buffer)
    uint32_t* tmp = A;
    A = An;
    An = tmp;
    cnt = cnt_out;
  }
  *result = A;
  return HE_OK;
}

static he_status rh_check_run(const he_rhombus_plan* p, const uint32_t* ct_in, uint32_t level, const uint32_t* ksk_dec,
                              const uint32_t* gal, const void* out, const void* ws_dev, uint64_t ws_bytes) {
  if (!p) return fail(HE_EINVAL, "null plan");
  if (level < 1) return fail(HE_ENEEDS_BOOTSTRAP, "pcmv needs one level");
  if (level != 1) return fail(HE_EINVAL, "the Rhombus PCMv runs at level 1 (got %u)", level);
  if (!ct_in || !ksk_dec || !gal || !out || !ws_dev) return fail(HE_EINVAL, "null argument");
  const uint64_t need = rh_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  if (ws_bytes < need)
    return fail(HE_EINVAL, "workspace too small (%llu < %llu)", (unsigned long long)ws_bytes, (unsigned long long)need);
  return HE_OK;
}

// (D) decompose + (M) products + the packing levels this plan owns; the packed ciphertexts stay in
// the workspace (NTT domain, [L][p_out][2][n]) at *packed.
static he_status rh_front(const he_rhombus_plan* p, const uint32_t* ct_in, const uint32_t* ksk_dec, const uint32_t* gal,
                          const RhWs& w, uint32_t piece0, uint32_t** packed, cudaStream_t st) {
  const he_context* c = p->ctx;
  const uint32_t n = p->n, N = p->N, q0 = p->M.m[0], q1 = p->M.m[1], P = p->M.m[2];
  // (D) decompose: key switch the a part at degree N, then split
  k_decomp_modup<<<grid_for(N), 256, 0, st>>>(ct_in, N, q0, q1, P, p->qhinv[0], p->qhinv[1], w.dD);
  HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1], &c->ntt[2]}, {w.dD, w.dD + 2ull * N, w.dD + 4ull * N}, 2, N, st),
          "NTT(digits)");
  k_mac<<<grid_for(N), 256, 0, st>>>(w.dD, ksk_dec, N, N, p->M, w.dUW);
  HE_CUDA(ntt_jobs(true, {&c->ntt[0], &c->ntt[1], &c->ntt[2]}, {w.dUW, w.dUW + 2ull * N, w.dUW + 4ull * N}, 2, N, st),
          "INTT(U,W)");
  k_decomp_split<<<grid_for((uint64_t)p->p_in * n), 256, 0, st>>>(w.dUW, ct_in, N, n, p->p_in, piece0, q0, q1, P,
                                                                   p->pinv[0], p->pinv[1], w.pieces);
  HE_CUDA(ntt_jobs(false, {&c->ntt_rh[0], &c->ntt_rh[1]}, {w.pieces, w.pieces + (size_t)p->p_in * 2 * n}, p->p_in * 2, n,
                   st), "NTT(pieces)");
  // (M) leaf ciphertexts: U = n / w inner products each
  const uint64_t leaves = leaves_of(p);
  {
    dim3 g = grid_for(leaves * n / 4);
    g.y = 2;
    k_rh_mvm<<<g, 256, 0, st>>>(p->wpt, w.pieces, leaves, p->p_in, p->logn, p->M, w.A0);
  }
  // (P) this plan's PackLWEs levels: s+1 .. log2 n - log2 G
  return rh_pack(p, w, gal, (uint32_t)leaves, p->split + 1, p->logn - p->logG, p->G, packed, st);
}

static void rh_count(const he_rhombus_plan* p, he_ledger* ledger, int rescale) {
  if (!ledger) return;
  ledger->pc_mults += (int64_t)leaves_of(p) * p->p_in;
  ledger->ct_rotations += (int64_t)(p->win / p->G - 1) * p->p_out;
  ledger->rescales += rescale;
}

static he_status rhombus_run_impl(const he_rhombus_plan* p, const uint32_t* ct_in, uint32_t level,
                                  const uint32_t* ksk_dec, const uint32_t* gal, uint32_t* out, void* ws_dev,
                                  uint64_t ws_bytes, void* stream, he_ledger* ledger, uint32_t piece0, int shard,
                                  uint32_t opiece0) {
  he_status s = rh_check_run(p, ct_in, level, ksk_dec, gal, out, ws_dev, ws_bytes);
  if (s) return s;
  if (p->G != 1)
    return fail(HE_EINVAL, "a leaf-interleaved shard plan (%u groups) runs through he_rhombus_run_subtree", p->G);
  if (shard && (piece0 + p->p_in > p->N / p->n || opiece0 + p->p_out > p->N / p->n))
    return fail(HE_EINVAL, "shard pieces [%u, %u) in / [%u, %u) out exceed the %u pieces of one ciphertext", piece0,
                piece0 + p->p_in, opiece0, opiece0 + p->p_out, p->N / p->n);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t n = p->n, N = p->N, q0 = p->M.m[0], q1 = p->M.m[1];
  RhWs w;
  rh_ws_words(p, &w, (uint32_t*)ws_dev);
  uint32_t* A = nullptr;
  s = rh_front(p, ct_in, ksk_dec, gal, w, piece0, &A, st);
  if (s) return s;
  // (R) + (C)
  const uint32_t cnt = p->p_out;
  HE_CUDA(ntt_jobs(true, {&p->ctx->ntt_rh[0], &p->ctx->ntt_rh[1]}, {A, A + (size_t)cnt * 2 * n}, cnt * 2, n, st),
          "INTT(packed)");
  if (shard) {
    HE_CUDA(cudaMemsetAsync(out, 0, 4ull * N * sizeof(uint32_t), st), "memset");
    k_rh_compose_l1<<<grid_for((uint64_t)cnt * 4 * n), 256, 0, st>>>(A, cnt, opiece0, n, N, out);
  } else {
    HE_CUDA(cudaMemsetAsync(out, 0, 2ull * N * sizeof(uint32_t), st), "memset");
    k_rh_rescale_compose<<<grid_for((uint64_t)cnt * 2 * n), 256, 0, st>>>(A, cnt, n, N, q0, q1, p->q1inv, p->q1invp, out);
  }
  HE_CUDA(cudaGetLastError(), "rhombus launch");
  rh_count(p, ledger, shard ? 0 : 1);
  return HE_OK;
}

extern "C" he_status he_rhombus_run(const he_rhombus_plan* p, const uint32_t* ct_in, uint32_t level,
                                    const uint32_t* ksk_dec, const uint32_t* gal, uint32_t* out, void* ws_dev,
                                    uint64_t ws_bytes, void* stream, he_ledger* ledger) {
  return rhombus_run_impl(p, ct_in, level, ksk_dec, gal, out, ws_dev, ws_bytes, stream, ledger, 0, 0, 0);
}

extern "C" he_status he_rhombus_run_shard(const he_rhombus_plan* p, const uint32_t* ct_in, uint32_t level,
                                          const uint32_t* ksk_dec, const uint32_t* gal, uint32_t piece0,
                                          uint32_t opiece0, uint32_t* out_l1, void* ws_dev, uint64_t ws_bytes,
                                          void* stream, he_ledger* ledger) {
  return rhombus_run_impl(p, ct_in, level, ksk_dec, gal, out_l1, ws_dev, ws_bytes, stream, ledger, piece0, 1, opiece0);
}

extern "C" he_status he_rhombus_run_subtree(const he_rhombus_plan* p, const uint32_t* ct_in, uint32_t level,
                                            const uint32_t* ksk_dec, const uint32_t* gal, uint32_t* roots_out,
                                            void* ws_dev, uint64_t ws_bytes, void* stream, he_ledger* ledger) {
  he_status s = rh_check_run(p, ct_in, level, ksk_dec, gal, roots_out, ws_dev, ws_bytes);
  if (s) return s;
  cudaStream_t st = (cudaStream_t)stream;
  RhWs w;
  rh_ws_words(p, &w, (uint32_t*)ws_dev);
  uint32_t* A = nullptr;
  s = rh_front(p, ct_in, ksk_dec, gal, w, 0, &A, st);
  if (s) return s;
  HE_CUDA(cudaMemcpyAsync(roots_out, A, 2ull * p->p_out * 2 * p->n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st),
          "roots");
  rh_count(p, ledger, 0);
  return HE_OK;
}

extern "C" he_status he_rhombus_finish(const he_rhombus_plan* p, const uint32_t* roots, const uint32_t* gal,
                                       uint32_t* out, void* ws_dev, uint64_t ws_bytes, void* stream,
                                       he_ledger* ledger) {
  if (!p) return fail(HE_EINVAL, "null plan");
  if (!roots || !gal || !out || !ws_dev) return fail(HE_EINVAL, "null argument");
  const uint64_t need = rh_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  if (ws_bytes < need)
    return fail(HE_EINVAL, "workspace too small (%llu < %llu)", (unsigned long long)ws_bytes, (unsigned long long)need);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t n = p->n, N = p->N, G = p->G, cnt = p->p_out;
  RhWs w;
  rh_ws_words(p, &w, (uint32_t*)ws_dev);
  k_rh_gather_roots<<<grid_for(4ull * cnt * n * G), 256, 0, st>>>(roots, G, cnt, n, w.A0);
  uint32_t* A = nullptr;
  he_status s = rh_pack(p, w, gal, cnt * G, p->logn - p->logG + 1, p->logn, 1, &A, st);
  if (s) return s;
  HE_CUDA(ntt_jobs(true, {&p->ctx->ntt_rh[0], &p->ctx->ntt_rh[1]}, {A, A + (size_t)cnt * 2 * n}, cnt * 2, n, st),
          "INTT(packed)");
  HE_CUDA(cudaMemsetAsync(out, 0, 2ull * N * sizeof(uint32_t), st), "memset");
  k_rh_rescale_compose<<<grid_for((uint64_t)cnt * 2 * n), 256, 0, st>>>(A, cnt, n, N, p->M.m[0], p->M.m[1], p->q1inv,
                                                                         p->q1invp, out);
  HE_CUDA(cudaGetLastError(), "rhombus finish");
  if (ledger) {
    ledger->ct_rotations += (int64_t)(G - 1) * cnt;
    ledger->rescales += 1;
  }
  return HE_OK;
}

extern "C" he_status he_rhombus_combine(const he_context* c, const uint32_t* parts, uint32_t count, uint32_t* out,
                                        void* stream, he_ledger* ledger) {
  if (!c || !parts || !out) return fail(HE_EINVAL, "null argument");
  if (count == 0) return fail(HE_EINVAL, "no shard outputs to combine");
  const uint32_t q0 = c->R.q[0], q1 = c->R.q[1];
  const uint32_t q1inv = (uint32_t)powmod_h(q1 % q0, q0 - 2, q0);
  k_rh_combine<<<grid_for(2ull * c->R.N), 256, 0, (cudaStream_t)stream>>>(parts, count, c->R.N, q0, q1, q1inv,
                                                                           shoup_pre(q1inv, q0), out);
  HE_CUDA(cudaGetLastError(), "rhombus combine");
  if (ledger) ledger->rescales += 1;
  return HE_OK;
}

// ======================================================================== MLWE -> RLWE ring packing
// SURVEY.md §8f1; restated from oracle/he_oracle_rhombus.c (or_ring_pack), bit-exact.  The leaves are
// the level-1 PCMM products C_y (he_pcmm_run_level1): A_y[k m - j] = a'_y[j][m], B_y[k m] = b'_y[m],
// scaled by k^-1.  PackLWEs over the subring Z[X^k] runs the K6 packing level at degree N: level l
// combines E + X^{k/2^l} O + sigma_g(E - X^{k/2^l} O), g = 1 + 2^l d, with one hybrid Galois key
// switch per combine; log2 k levels turn each k-row block into one RLWE ciphertext, then rescale.
namespace {

// leaves a part [L][cnt][2][N] (coefficient form) from the MLWE-layout words raw_a [L][n_out][k][d]:
// one CTA per (32 positions m, row, limb): transposing tile [j][m] in smem, coalesced on both sides
__global__ void __launch_bounds__(256) k_rp_leaves_a(const uint32_t* __restrict__ raw_a, uint64_t limb_stride,
                                                     uint32_t y0, uint32_t d, uint32_t k, uint32_t N, uint32_t cnt,
                                                     uint32_t kinv0, uint32_t kinvp0, uint32_t kinv1, uint32_t kinvp1,
                                                     uint32_t q0, uint32_t q1, uint32_t* __restrict__ leaves) {
  __shared__ uint32_t tile[256 * 33];  // [j][m], k <= 256
  const uint32_t m0 = blockIdx.x * 32, yl = blockIdx.y, L = blockIdx.z;
  const uint32_t q = L ? q1 : q0, kinv = L ? kinv1 : kinv0, kinvp = L ? kinvp1 : kinvp0;
  const uint32_t* src = raw_a + L * limb_stride + (size_t)(y0 + yl) * N + m0;
  for (uint32_t i = threadIdx.x; i < 32 * k; i += blockDim.x) tile[(i >> 5) * 33 + (i & 31)] = src[(size_t)d * (i >> 5) + (i & 31)];
  __syncthreads();
  uint32_t* dst = leaves + (((size_t)L * cnt + yl) * 2 + 0) * N;
  for (uint32_t i = threadIdx.x; i < 32 * k; i += blockDim.x) {
    const uint32_t mm = i / k, j = k - 1 - (i % k);
    uint32_t v = tile[j * 33 + mm];
    int64_t c = (int64_t)k * (m0 + mm) - j;
    if (c < 0) {
      c += N;
      v = v ? q - v : 0;
    }
    dst[c] = shoup_mul(v, kinv, kinvp, q);
  }
}
// leaves b part: B_y[c] = b'_y[c / k] for c = 0 mod k, else 0;  raw_b [L][n_out/k][N] (RLWE order)
__global__ void k_rp_leaves_b(const uint32_t* __restrict__ raw_b, uint64_t limb_stride, uint32_t y0, uint32_t k,
                              uint32_t logN, uint32_t cnt, uint32_t kinv0, uint32_t kinvp0, uint32_t kinv1,
                              uint32_t kinvp1, uint32_t q0, uint32_t q1, uint32_t* __restrict__ leaves) {
  const uint32_t N = 1u << logN, L = blockIdx.y;
  const uint32_t q = L ? q1 : q0, kinv = L ? kinv1 : kinv0, kinvp = L ? kinvp1 : kinvp0;
  const uint64_t total = (uint64_t)cnt << logN;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t yl = (uint32_t)(x >> logN), c = (uint32_t)(x & (N - 1)), y = y0 + yl;
    uint32_t v = 0;
    if (c % k == 0) v = shoup_mul(raw_b[L * limb_stride + (size_t)(y / k) * N + (y % k) + c], kinv, kinvp, q);
    leaves[(((size_t)L * cnt + yl) * 2 + 1) * N + c] = v;
  }
}
// packing level at degree N (no smem staging: the polynomial does not fit), see k_pack_comb1
__global__ void k_rp_comb1(const uint32_t* __restrict__ A, uint32_t cnt_in, uint32_t half, uint32_t logN,
                           const uint32_t* __restrict__ mono /* [2][N] */, const uint32_t* __restrict__ perm, Mods M,
                           uint32_t* __restrict__ An, uint32_t* __restrict__ T, uint32_t* __restrict__ C) {
  const uint32_t N = 1u << logN, ab = blockIdx.y, L = blockIdx.z, cnt_out = cnt_in / 2;
  const uint32_t q = M.m[L];
  const uint64_t mu = M.mu[L];
  const uint32_t* ml = mono + (size_t)L * N;
  const uint64_t total = (uint64_t)cnt_out << logN;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t idx = (uint32_t)(x >> logN), c = (uint32_t)(x & (N - 1));
    const uint32_t o = idx / half, s_ = idx % half;
    const uint32_t e_i = o * 2 * half + s_, o_i = e_i + half;
    const uint32_t* Eb = A + (((size_t)L * cnt_in + e_i) * 2 + ab) * N;
    const uint32_t* Ob = A + (((size_t)L * cnt_in + o_i) * 2 + ab) * N;
    const uint32_t e = Eb[c], mo = mulmod_b(Ob[c], ml[c], mu, q);
    An[(((size_t)L * cnt_out + idx) * 2 + ab) * N + c] = add_mod(e, mo, q);
    const uint32_t pc = perm[c];
    const uint32_t v = sub_mod(Eb[pc], mulmod_b(Ob[pc], ml[pc], mu, q), q);
    T[(((size_t)L * cnt_out + idx) * 2 + ab) * N + c] = v;
    if (ab == 0) C[((size_t)L * cnt_out + idx) * N + c] = v;
  }
}
// rescale by q1: A [L][nb][2][N] coefficient form -> out [nb][2][N]
__global__ void k_rp_rescale(const uint32_t* __restrict__ A, uint64_t per_l, uint32_t q0, uint32_t q1, uint32_t q1inv,
                             uint32_t q1invp, uint32_t* __restrict__ out) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < per_l; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x0 = A[x], x1 = A[per_l + x];
    uint32_t t;
    if (x1 > (q1 >> 1)) t = csub(x0 + (q1 - x1), q0);
    else t = sub_mod(x0, x1, q0);
    out[x] = shoup_mul(t, q1inv, q1invp, q0);
  }
}

// ---- MLWE -> RLWE key-switch packing (default method; oracle or_mlwe_to_rlwe)
// digits of alpha_j (alpha_j[t + k m] = a'_{kY+t}[j][m]) for a chunk of (j, Y) pairs, coefficient form,
// lifted to all three moduli:  D [mod][i][cnt][N], index jj * Yc + Y.  One CTA per (32 positions m, pair):
// the [t][m] tile is transposed through smem so both the reads and the writes are coalesced.
__global__ void __launch_bounds__(256) k_ms_digits(const uint32_t* __restrict__ raw_a, uint32_t n_out, uint32_t Y0,
                                                   uint32_t j0, uint32_t Yc, uint32_t cnt, uint32_t d, uint32_t k,
                                                   uint32_t N, Mods M, uint32_t qh0, uint32_t qh0p, uint32_t qh1,
                                                   uint32_t qh1p, uint32_t* __restrict__ D) {
  __shared__ uint32_t tile[256 * 33];  // [t][m], k <= 256
  const uint32_t m0 = blockIdx.x * 32, idx = blockIdx.y, jj = idx / Yc, Y = idx % Yc, j = j0 + jj;
  const size_t plane = (size_t)cnt * N;
  for (uint32_t L = 0; L < 2; ++L) {
    const uint32_t* src = raw_a + ((size_t)L * n_out + (size_t)(Y0 + Y) * k) * N + (size_t)d * j + m0;
    for (uint32_t i = threadIdx.x; i < 32 * k; i += blockDim.x) tile[(i >> 5) * 33 + (i & 31)] = src[(size_t)(i >> 5) * N + (i & 31)];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 32 * k; i += blockDim.x) {
      const uint32_t mm = i / k, t = i % k;
      const size_t c = (size_t)idx * N + t + (size_t)k * (m0 + mm);
      const uint32_t v = tile[t * 33 + mm];
      // own-limb digit d_L = alpha * Qhat_L^-1 mod q_L, then its residues mod the other two moduli
      const uint32_t dg = L ? shoup_mul(v, qh1, qh1p, M.m[1]) : shoup_mul(v, qh0, qh0p, M.m[0]);
#pragma unroll
      for (int mod = 0; mod < 3; ++mod)
        D[(size_t)(mod * 2 + L) * plane + c] = (mod == (int)L) ? dg : barrett64(dg, M.mu[mod], M.m[mod]);
    }
    __syncthreads();
  }
}
// UW [mod][part][Yc][N] += sum_jj sum_i D^[mod][i][jj Yc + Y] * K_{j0+jj}[i][part][mod]   (NTT domain)
// one thread per (frequency, block, modulus): contiguous streams per warp; the key words are shared by
// the Yc blocks through L1/L2
constexpr int kMsMaxYc = 16;
__global__ void __launch_bounds__(256) k_ms_mac(const uint32_t* __restrict__ D, const uint32_t* __restrict__ K,
                                                uint32_t jc, uint32_t Yc, uint32_t logN, Mods M,
                                                uint32_t* __restrict__ UW) {
  const uint32_t N = 1u << logN, mod = blockIdx.y;
  const uint64_t x4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;  // (Y * N + f) / 4: 4 frequencies per thread
  if (x4 >= ((uint64_t)Yc << logN) / 4) return;
  const uint32_t f4 = (uint32_t)((x4 * 4) & (N - 1)) / 4;
  const uint32_t q = mod == 0 ? M.m[0] : (mod == 1 ? M.m[1] : M.m[2]);
  const uint64_t mu = mod == 0 ? M.mu[0] : (mod == 1 ? M.mu[1] : M.mu[2]);
  const size_t plane4 = (size_t)jc * Yc * N / 4, yn4 = (size_t)Yc * N / 4, n4 = N / 4;
  const uint4* d0 = reinterpret_cast<const uint4*>(D) + (size_t)(mod * 2 + 0) * plane4 + x4;
  const uint4* d1 = reinterpret_cast<const uint4*>(D) + (size_t)(mod * 2 + 1) * plane4 + x4;
  uint64_t au[4] = {0, 0, 0, 0}, aw[4] = {0, 0, 0, 0};
  for (uint32_t jj = 0; jj < jc; ++jj) {
    const uint4* Kj = reinterpret_cast<const uint4*>(K + (size_t)jj * 12 * N) + f4;
    const uint4 x0 = __ldcs(d0 + jj * yn4), x1 = __ldcs(d1 + jj * yn4);
    const uint4 k00 = __ldg(Kj + ((0 * 2 + 0) * 3 + mod) * n4), k10 = __ldg(Kj + ((1 * 2 + 0) * 3 + mod) * n4);
    const uint4 k01 = __ldg(Kj + ((0 * 2 + 1) * 3 + mod) * n4), k11 = __ldg(Kj + ((1 * 2 + 1) * 3 + mod) * n4);
    const uint32_t a0[4] = {x0.x, x0.y, x0.z, x0.w}, a1[4] = {x1.x, x1.y, x1.z, x1.w};
    const uint32_t u0[4] = {k00.x, k00.y, k00.z, k00.w}, u1[4] = {k10.x, k10.y, k10.z, k10.w};
    const uint32_t w0[4] = {k01.x, k01.y, k01.z, k01.w}, w1[4] = {k11.x, k11.y, k11.z, k11.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      au[e] += (uint64_t)a0[e] * u0[e] + (uint64_t)a1[e] * u1[e];
      aw[e] += (uint64_t)a0[e] * w0[e] + (uint64_t)a1[e] * w1[e];
    }
    if (jj & 1) {  // two products of < 2^60 per step: reduce every second step (< 2^63)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        au[e] = barrett64(au[e], mu, q);
        aw[e] = barrett64(aw[e], mu, q);
      }
    }
  }
  uint4* U = reinterpret_cast<uint4*>(UW) + (size_t)(mod * 2 + 0) * yn4 + x4;
  uint4* W = reinterpret_cast<uint4*>(UW) + (size_t)(mod * 2 + 1) * yn4 + x4;
  const uint4 uo = *U, wo = *W;
  *U = make_uint4(add_mod(uo.x, barrett64(au[0], mu, q), q), add_mod(uo.y, barrett64(au[1], mu, q), q),
                  add_mod(uo.z, barrett64(au[2], mu, q), q), add_mod(uo.w, barrett64(au[3], mu, q), q));
  *W = make_uint4(add_mod(wo.x, barrett64(aw[0], mu, q), q), add_mod(wo.y, barrett64(aw[1], mu, q), q),
                  add_mod(wo.z, barrett64(aw[2], mu, q), q), add_mod(wo.w, barrett64(aw[3], mu, q), q));
}
// ModDown of the summed (U, W) (coefficient form), b += composed b', rescale by q1 -> out [Y][2][N]
__global__ void k_ms_finish(const uint32_t* __restrict__ UW, const uint32_t* __restrict__ raw_b, uint32_t blocks,
                            uint32_t Y0, uint32_t Yc, uint32_t logN, Mods M, uint32_t pinv0, uint32_t pinv1,
                            uint32_t q1inv, uint32_t q1invp, uint32_t* __restrict__ out) {
  const uint32_t N = 1u << logN, P = M.m[2], q0 = M.m[0], q1 = M.m[1];
  const uint64_t per = (uint64_t)Yc << logN;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < per; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t Y = (uint32_t)(x >> logN), c = (uint32_t)(x & (N - 1));
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint32_t vp = UW[(size_t)(2 * 2 + part) * per + x];
      const int64_t cp = vp > P / 2 ? (int64_t)vp - P : (int64_t)vp;
      uint32_t v[2];
#pragma unroll
      for (int L = 0; L < 2; ++L) {
        const uint32_t q = M.m[L];
        v[L] = mulmod_b(sub_mod(UW[(size_t)(L * 2 + part) * per + x], lift_b(cp, M.mu[L], q), q), L ? pinv1 : pinv0,
                        M.mu[L], q);
        if (part) v[L] = add_mod(v[L], raw_b[((size_t)L * blocks + Y0 + Y) * N + c], q);
      }
      uint32_t t;
      if (v[1] > (q1 >> 1)) t = csub(v[0] + (q1 - v[1]), q0);
      else t = sub_mod(v[0], v[1], q0);
      out[((size_t)(Y0 + Y) * 2 + part) * N + c] = shoup_mul(t, q1inv, q1invp, q0);
    }
  }
}
// s^_j = s_j(X^k): s^_j[c] = s[j + c] for c = 0 mod k, else 0
__global__ void k_ms_component(const int32_t* s, uint32_t N, uint32_t k, uint32_t j, int32_t* out) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x)
    out[c] = (c % k == 0) ? s[j + c] : 0;
}

// ---- one-digit MLWE -> RLWE key switching with two special primes (method HE_RING_PACK_KEYSWITCH1; oracle
// or_mlwe_to_rlwe1): the digit of alpha_j is alpha_j itself (mod Q = q0 q1), its centred value lifted to
// P1 = P and P2, and the keys encrypt P1 P2 s_j(X^k) modulo Q P1 P2 -- 4 NTT'd planes per (block, j) instead of
// 2 digits x 3 moduli, 8 key planes per component instead of 12.
struct Mods4 {
  uint32_t m[4];   // q0, q1, P1, P2
  uint64_t mu[4];
};
// D [mod 4][cnt][N]: alpha mod q0, alpha mod q1 (the residues themselves) and [alpha]_Q mod P1, P2.  One CTA per
// (16 positions m, pair): both limbs' [t][m] tiles through smem (pitch 17), 4 consecutive t per thread -> 16-byte
// stores of every plane.
constexpr int kMs1M = 16;
__global__ void __launch_bounds__(256) k_ms1_digits(const uint32_t* __restrict__ raw_a, uint32_t n_out, uint32_t Y0,
                                                    uint32_t j0, uint32_t Yc, uint32_t cnt, uint32_t d, uint32_t k,
                                                    uint32_t N, Mods4 M, uint32_t q0inv_q1, uint32_t* __restrict__ D) {
  __shared__ uint32_t tile[2][256 * (kMs1M + 1)];  // [limb][t][m], k <= 256
  const uint32_t m0 = blockIdx.x * kMs1M, idx = blockIdx.y, jj = idx / Yc, Y = idx % Yc, j = j0 + jj;
  const size_t plane = (size_t)cnt * N;
  for (uint32_t L = 0; L < 2; ++L) {
    const uint32_t* src = raw_a + ((size_t)L * n_out + (size_t)(Y0 + Y) * k) * N + (size_t)d * j + m0;
    for (uint32_t i = threadIdx.x; i < kMs1M * k; i += blockDim.x)
      tile[L][(i / kMs1M) * (kMs1M + 1) + (i % kMs1M)] = src[(size_t)(i / kMs1M) * N + (i % kMs1M)];
  }
  __syncthreads();
  const uint32_t q0 = M.m[0], q1 = M.m[1];
  const uint64_t Q = (uint64_t)q0 * q1;
  const uint32_t k4 = k / 4;
  for (uint32_t i = threadIdx.x; i < kMs1M * k4; i += blockDim.x) {
    const uint32_t mm = i / k4, t0 = 4 * (i % k4);
    uint32_t o[4][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t a0 = tile[0][(t0 + e) * (kMs1M + 1) + mm], a1 = tile[1][(t0 + e) * (kMs1M + 1) + mm];
      // CRT: alpha = a0 + q0 ((a1 - a0) q0^-1 mod q1) in [0, Q), centred
      const uint32_t tq = mulmod_b(sub_mod(a1, barrett64(a0, M.mu[1], q1), q1), q0inv_q1, M.mu[1], q1);
      const uint64_t al = (uint64_t)a0 + (uint64_t)q0 * tq;
      const int64_t ac = al > Q / 2 ? (int64_t)al - (int64_t)Q : (int64_t)al;
      o[0][e] = a0;
      o[1][e] = a1;
      o[2][e] = lift_b(ac, M.mu[2], M.m[2]);
      o[3][e] = lift_b(ac, M.mu[3], M.m[3]);
    }
    const size_t c = (size_t)idx * N + t0 + (size_t)k * (m0 + mm);
#pragma unroll
    for (int mod = 0; mod < 4; ++mod)
      *reinterpret_cast<uint4*>(D + mod * plane + c) = make_uint4(o[mod][0], o[mod][1], o[mod][2], o[mod][3]);
  }
}
// The same digits with the outer (cols) stages of K2's forward NTT fused in, for N = 16 x 4096 and k = 256: the
// 16-point column c of plane alpha_j holds coefficients c + 4096 v = t + 256 (m0 + 16 v) (t = c % 256,
// m0 = c / 256), i.e. the positions m = m0 mod 16 of ONE a' row segment -- so a CTA that stages 32 whole row
// segments a'[t][j][0 .. 255] (both limbs, 1 KB each, coalesced) owns 512 complete columns. Per column: CRT
// lift to P1, P2, then the 16-point merged-twiddle CT transform of each modulus exactly as ntt_fwd_cols<16>
// does it (same butterflies, same lazy [0, 4q) outputs), 128-byte stores per (modulus, v). The rows pass then
// runs as usual (ntt_forward(..., rows_only)). Saves the digit planes' HBM round trip between the two kernels.
constexpr int kMs1T = 32;                 // rows t per CTA
constexpr int kMs1Pitch = 257;            // smem words per staged row segment (conflict-free column gathers)
HE_D void ct_bf_rp(uint32_t& x, uint32_t& y, uint2 w, uint32_t q2, uint32_t q) {  // = he_ntt.cu ct_bf
  const uint32_t a = min(x, x - q2);
  const uint32_t t = y * w.x - __umulhi(y, w.y) * q;
  x = a + t;
  y = a + q2 - t;
}
// the 16-point cols transform of canonical inputs (< q): twiddles are kernel parameters (constant-bank operands,
// no loads), and the first stage skips the x correction (x < q already)
HE_D void cols16_store(uint32_t (&x)[16], const uint2 (&tw)[16], uint32_t q, uint32_t* dst) {
  const uint32_t q2 = 2 * q;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t a = x[u], y = x[u + 8];
    const uint32_t t = y * tw[1].x - __umulhi(y, tw[1].y) * q;
    x[u] = a + t;
    x[u + 8] = a + q2 - t;
  }
#pragma unroll
  for (int m = 2, t = 4; m < 16; m <<= 1, t >>= 1) {
#pragma unroll
    for (int i = 0; i < m; ++i) {
#pragma unroll
      for (int u = 0; u < t; ++u) ct_bf_rp(x[2 * i * t + u], x[2 * i * t + u + t], tw[m + i], q2, q);
    }
  }
#pragma unroll
  for (int v = 0; v < 16; ++v) dst[(size_t)4096 * v] = x[v];
}
struct Ms1Tw {
  uint2 tw[4][16];      // forward twiddles (W, Shoup) 0 .. 15 of q0, q1, P1, P2 at N = 2^16 (NttTable::fw16)
  // 32-bit CRT constants: floor(2^32 / q1); q0^-1 mod q1 (Shoup); per special prime i: q0 mod P_i (Shoup), Q mod P_i
  uint32_t m1, w01, w01p, c[2], cp[2], qp[2];
  uint64_t Q;
};
__global__ void __launch_bounds__(256, 3) k_ms1_digits_cols(const uint32_t* __restrict__ raw_a, uint32_t n_out,
                                                            uint32_t Y0, uint32_t j0, uint32_t Yc, uint32_t cnt,
                                                            Mods4 M, uint32_t q0inv_q1, Ms1Tw T,
                                                            uint32_t* __restrict__ D) {
  extern __shared__ uint32_t seg[];   // [limb][kMs1T rows t][kMs1Pitch]
  constexpr uint32_t k = 256, d = 256, N = 65536;
  const uint32_t t0 = blockIdx.x * kMs1T, idx = blockIdx.y, jj = idx / Yc, Y = idx % Yc, j = j0 + jj;
  for (uint32_t L = 0; L < 2; ++L) {
    const uint32_t* src = raw_a + ((size_t)L * n_out + (size_t)(Y0 + Y) * k + t0) * N + (size_t)d * j;
    for (uint32_t i = threadIdx.x; i < kMs1T * d / 4; i += blockDim.x) {
      // a warp access = 4 rows x 128 B; stores hit banks r + 4 m4 (+ e): all 32 distinct
      const uint32_t w = i >> 5, ln = i & 31, r = (w & 7) * 4 + (ln >> 3), m4 = (w >> 3) * 8 + (ln & 7);
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src + (size_t)r * N) + m4);
      uint32_t* o = seg + (L * kMs1T + r) * kMs1Pitch + 4 * m4;
      o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
    }
  }
  __syncthreads();
  const uint32_t q0 = M.m[0], q1 = M.m[1];
  const uint64_t Q = (uint64_t)q0 * q1;
  const size_t plane = (size_t)cnt * N;
  // thread -> (t = lane, m0 = warp + 8 i): the 32 lanes of a warp gather 32 rows (banks t * 257 = t mod 32).
  // Moduli in sequence (q0, q1 straight from the staged words, then P1, P2 via the CRT lift) to stay at 3 CTAs/SM
  const uint32_t t = threadIdx.x & 31;
  for (uint32_t m0 = threadIdx.x >> 5; m0 < 16; m0 += blockDim.x >> 5) {
    const uint32_t* s0 = seg + t * kMs1Pitch + m0;
    const uint32_t* s1 = seg + (kMs1T + t) * kMs1Pitch + m0;
    const size_t c = (size_t)idx * N + t0 + t + (size_t)k * m0;
    uint32_t x[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = s0[16 * v];
    cols16_store(x, T.tw[0], q0, D + c);
#pragma unroll
    for (int v = 0; v < 16; ++v) x[v] = s1[16 * v];
    cols16_store(x, T.tw[1], q1, D + plane + c);
    uint32_t x3[16];
#pragma unroll
    for (int v = 0; v < 16; ++v) {
      // CRT: alpha = a0 + q0 tq, tq = (a1 - a0) q0^-1 mod q1, in [0, Q), centred (= k_ms1_digits) -- in 32-bit
      // pieces: [alpha]_Q mod P = (a0 mod P) + (q0 mod P) tq - (Q mod P if alpha > Q/2), all mod P
      const uint32_t a0 = s0[16 * v], a1 = s1[16 * v];
      const uint32_t r = a0 - __umulhi(a0, T.m1) * q1;   // a0 < 2^30: Barrett remainder in [0, 2 q1)
      const uint32_t dd = a1 + 2 * q1 - r;               // = a1 - a0 mod q1, in (0, 3 q1): Shoup takes any u32
      uint32_t tq = dd * T.w01 - __umulhi(dd, T.w01p) * q1;
      tq = min(tq, tq - q1);                              // [0, q1)
      // alpha = a0 + q0 tq > Q / 2 (Q, q0, q1 odd)  <=>  tq > (q1 - 1) / 2, or tq == (q1 - 1) / 2 and a0 > q0 / 2
      const uint32_t h1 = q1 >> 1;
      const bool neg = tq > h1 || (tq == h1 && a0 > (q0 >> 1));
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint32_t P = M.m[2 + i];
        // (a0 mod P) + (q0 mod P) tq + (P - (Q mod P) if negative): [0, P) + [0, 2P) + [0, P) < 4P < 2^32
        uint32_t u = min(a0, a0 - P) + (tq * T.c[i] - __umulhi(tq, T.cp[i]) * P) + (neg ? P - T.qp[i] : 0u);
        u = min(u, u - 2 * P);
        u = min(u, u - P);
        if (i == 0) x[v] = u;
        else x3[v] = u;
      }
    }
    cols16_store(x, T.tw[2], M.m[2], D + 2 * plane + c);
    cols16_store(x3, T.tw[3], M.m[3], D + 3 * plane + c);
  }
}
// UW [mod][part][Yc][N] += sum_jj D^[mod][jj Yc + Y] * K_{j0+jj}[part][mod]   (NTT domain; 4 frequencies per thread)
__global__ void __launch_bounds__(256) k_ms1_mac(const uint32_t* __restrict__ D, const uint32_t* __restrict__ K,
                                                 uint32_t jc, uint32_t Yc, uint32_t logN, Mods4 M,
                                                 uint32_t* __restrict__ UW) {
  const uint32_t N = 1u << logN, mod = blockIdx.y;
  const uint64_t x4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (x4 >= ((uint64_t)Yc << logN) / 4) return;
  const uint32_t f4 = (uint32_t)((x4 * 4) & (N - 1)) / 4;
  const uint32_t q = M.m[mod];
  const uint64_t mu = M.mu[mod];
  const size_t plane4 = (size_t)jc * Yc * N / 4, yn4 = (size_t)Yc * N / 4, n4 = N / 4;
  const uint4* d0 = reinterpret_cast<const uint4*>(D) + (size_t)mod * plane4 + x4;
  uint64_t au[4] = {0, 0, 0, 0}, aw[4] = {0, 0, 0, 0};
#pragma unroll 8
  for (uint32_t jj = 0; jj < jc; ++jj) {
    const uint4* Kj = reinterpret_cast<const uint4*>(K + (size_t)jj * 8 * N) + f4;
    const uint4 x = __ldcs(d0 + jj * yn4);
    const uint4 ku = __ldg(Kj + (0 * 4 + mod) * n4), kw = __ldg(Kj + (1 * 4 + mod) * n4);
    const uint32_t a[4] = {x.x, x.y, x.z, x.w}, u[4] = {ku.x, ku.y, ku.z, ku.w}, w[4] = {kw.x, kw.y, kw.z, kw.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      au[e] += (uint64_t)a[e] * u[e];
      aw[e] += (uint64_t)a[e] * w[e];
    }
    if ((jj & 7) == 7) {  // products < 2^60: reduce every 8 steps (< 2^63)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        au[e] = barrett64(au[e], mu, q);
        aw[e] = barrett64(aw[e], mu, q);
      }
    }
  }
  uint4* U = reinterpret_cast<uint4*>(UW) + (size_t)(mod * 2 + 0) * yn4 + x4;
  uint4* W = reinterpret_cast<uint4*>(UW) + (size_t)(mod * 2 + 1) * yn4 + x4;
  const uint4 uo = *U, wo = *W;
  *U = make_uint4(add_mod(uo.x, barrett64(au[0], mu, q), q), add_mod(uo.y, barrett64(au[1], mu, q), q),
                  add_mod(uo.z, barrett64(au[2], mu, q), q), add_mod(uo.w, barrett64(au[3], mu, q), q));
  *W = make_uint4(add_mod(wo.x, barrett64(aw[0], mu, q), q), add_mod(wo.y, barrett64(aw[1], mu, q), q),
                  add_mod(wo.z, barrett64(aw[2], mu, q), q), add_mod(wo.w, barrett64(aw[3], mu, q), q));
}
// The same MAC with each thread owning 2 frequencies of kMacY output blocks: every key pair is loaded once per
// (component, frequency) and used for kMacY blocks (k_ms1_mac re-reads the keys once per block from L2).
constexpr uint32_t kMacY = 8;
template <bool LAZY_IN>
__global__ void __launch_bounds__(256) k_ms1_mac_y(const uint32_t* __restrict__ D, const uint32_t* __restrict__ K,
                                                   uint32_t jc, uint32_t Yc, uint32_t logN, Mods4 M,
                                                   uint32_t* __restrict__ UW) {
  const uint32_t N = 1u << logN, mod = blockIdx.z, y0 = blockIdx.y * kMacY;
  const uint32_t f2 = blockIdx.x * blockDim.x + threadIdx.x;   // frequencies 2 f2, 2 f2 + 1
  const uint32_t q = M.m[mod];
  const uint64_t mu = M.mu[mod];
  const size_t plane2 = (size_t)jc * Yc * N / 2, n2 = N / 2;
  const uint2* d0 = reinterpret_cast<const uint2*>(D) + (size_t)mod * plane2 + (size_t)y0 * n2 + f2;
  uint64_t au[kMacY][2], aw[kMacY][2];
#pragma unroll
  for (uint32_t y = 0; y < kMacY; ++y) au[y][0] = au[y][1] = aw[y][0] = aw[y][1] = 0;
#pragma unroll 2
  for (uint32_t jj = 0; jj < jc; ++jj) {
    const uint2* Kj = reinterpret_cast<const uint2*>(K + (size_t)jj * 8 * N) + f2;
    const uint2 ku = __ldg(Kj + (0 * 4 + mod) * n2), kw = __ldg(Kj + (1 * 4 + mod) * n2);
#pragma unroll
    for (uint32_t y = 0; y < kMacY; ++y) {
      uint2 x = __ldcs(d0 + ((size_t)jj * Yc + y) * n2);
      if (LAZY_IN) {   // digit NTT outputs left in [0, 4 q) by the rows pass -> [0, 2 q): with the keys < q and
        // the reduction every 8 steps, 8 (2 q) q + q < 2^64 for q < 2^30
        x.x = min(x.x, x.x - 2 * q), x.y = min(x.y, x.y - 2 * q);
      }
      au[y][0] += (uint64_t)x.x * ku.x;
      au[y][1] += (uint64_t)x.y * ku.y;
      aw[y][0] += (uint64_t)x.x * kw.x;
      aw[y][1] += (uint64_t)x.y * kw.y;
    }
    if ((jj & 7) == 7) {  // products < 2^60: reduce every 8 steps (< 2^63)
#pragma unroll
      for (uint32_t y = 0; y < kMacY; ++y)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          au[y][e] = barrett64(au[y][e], mu, q);
          aw[y][e] = barrett64(aw[y][e], mu, q);
        }
    }
  }
  const size_t yn2 = (size_t)Yc * n2;
#pragma unroll
  for (uint32_t y = 0; y < kMacY; ++y) {
    uint2* U = reinterpret_cast<uint2*>(UW) + (size_t)(mod * 2 + 0) * yn2 + (size_t)(y0 + y) * n2 + f2;
    uint2* W = reinterpret_cast<uint2*>(UW) + (size_t)(mod * 2 + 1) * yn2 + (size_t)(y0 + y) * n2 + f2;
    const uint2 uo = *U, wo = *W;
    *U = make_uint2(add_mod(uo.x, barrett64(au[y][0], mu, q), q), add_mod(uo.y, barrett64(au[y][1], mu, q), q));
    *W = make_uint2(add_mod(wo.x, barrett64(aw[y][0], mu, q), q), add_mod(wo.y, barrett64(aw[y][1], mu, q), q));
  }
}
// ModDown by P1 P2 of the summed (U, W) (coefficient form; [x]_P centred by CRT), b += composed b', rescale by q1
__global__ void k_ms1_finish(const uint32_t* __restrict__ UW, const uint32_t* __restrict__ raw_b, uint32_t blocks,
                             uint32_t Y0, uint32_t Yc, uint32_t logN, Mods4 M, uint32_t p1inv_p2, uint32_t pinv0,
                             uint32_t pinv1, uint32_t q1inv, uint32_t q1invp, uint32_t* __restrict__ out) {
  const uint32_t N = 1u << logN, q0 = M.m[0], q1 = M.m[1], P1 = M.m[2], P2 = M.m[3];
  const uint64_t per = (uint64_t)Yc << logN, PP = (uint64_t)P1 * P2;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < per; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t Y = (uint32_t)(x >> logN), c = (uint32_t)(x & (N - 1));
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint32_t v1 = UW[(size_t)(2 * 2 + part) * per + x], v2 = UW[(size_t)(3 * 2 + part) * per + x];
      const uint32_t tq = mulmod_b(sub_mod(v2, barrett64(v1, M.mu[3], P2), P2), p1inv_p2, M.mu[3], P2);
      const uint64_t xp = (uint64_t)v1 + (uint64_t)P1 * tq;   // [x]_{P1 P2} in [0, P1 P2)
      const bool neg = xp > PP / 2;
      const uint64_t mag = neg ? PP - xp : xp;
      uint32_t v[2];
#pragma unroll
      for (int L = 0; L < 2; ++L) {
        const uint32_t q = M.m[L];
        uint32_t r = barrett64(mag, M.mu[L], q);
        if (neg && r) r = q - r;                                   // [x]_P mod q
        v[L] = mulmod_b(sub_mod(UW[(size_t)(L * 2 + part) * per + x], r, q), L ? pinv1 : pinv0, M.mu[L], q);
        if (part) v[L] = add_mod(v[L], raw_b[((size_t)L * blocks + Y0 + Y) * N + c], q);
      }
      uint32_t t;
      if (v[1] > (q1 >> 1)) t = csub(v[0] + (q1 - v[1]), q0);
      else t = sub_mod(v[0], v[1], q0);
      out[((size_t)(Y0 + Y) * 2 + part) * N + c] = shoup_mul(t, q1inv, q1invp, q0);
    }
  }
}
// the second special prime of method KEYSWITCH1: the largest prime < 2^30, 1 mod 2N, not q0, q1 or P
static bool is_prime_h(uint64_t n) {
  if (n < 2) return false;
  for (uint64_t p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull})
    if (n % p == 0) return n == p;
  uint64_t dd = n - 1;
  int sh = 0;
  while (!(dd & 1)) dd >>= 1, ++sh;
  for (uint64_t a : {2ull, 3ull, 5ull, 7ull, 11ull}) {
    uint64_t x = powmod_h(a, dd, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < sh && comp; ++r) {
      x = (unsigned __int128)x * x % n;
      if (x == n - 1) comp = false;
    }
    if (comp) return false;
  }
  return true;
}
uint32_t ring_pack_p2(const RingDims& R) {
  const uint64_t two_n = 2ull * R.N;
  for (uint64_t cc = ((1ull << 30) - 1) / two_n; cc > 0; --cc) {
    const uint64_t p = cc * two_n + 1;
    if (p >= (1ull << 30) || p == R.q[0] || p == R.q[1] || p == R.P) continue;
    if (is_prime_h(p)) return (uint32_t)p;
  }
  return 0;
}

uint64_t find_psi(uint32_t q, uint32_t n) {  // the root ntt_table_init uses
  for (uint64_t g = 2; g < q; ++g) {
    const uint64_t cand = powmod_h(g, (q - 1) / (2ull * n), q);
    if (powmod_h(cand, n, q) == q - 1) return cand;
  }
  return 0;
}

}  // namespace

struct he_ring_pack_plan {
  const he_context* ctx;
  int method;        // HE_RING_PACK_KEYSWITCH (0), HE_RING_PACK_TRACE (1) or HE_RING_PACK_KEYSWITCH1 (2)
  NttTable ntt_p2{};  // KEYSWITCH1: degree-N tables of the second special prime
  Mods4 M4{};
  uint32_t q0inv_q1 = 0, p1inv_p2 = 0, ppinv[2] = {0, 0};
  uint32_t jc;       // keyswitch: components j per pass
  uint32_t n_out, blocks, chunk, d, k, N, logN, logk;
  uint32_t* tables;  // owned: perm [logk][N], mono [logk][2][N]
  Mods M;
  uint32_t qhinv[2], pinv[2], q1inv, q1invp, kinv[2], kinvp[2];
};

static uint64_t ring_pack_key_words(const he_context* c, int method) {
  if (method == HE_RING_PACK_KEYSWITCH1) return (uint64_t)c->R.k * 8ull * c->R.N;   // [k][2][4][N]
  const uint64_t n_keys = method == HE_RING_PACK_TRACE ? (uint64_t)ilog2_u(c->R.k) : (uint64_t)c->R.k;
  return n_keys * 12ull * c->R.N;
}
static bool rp_method_ok(int m) {
  return m == HE_RING_PACK_KEYSWITCH || m == HE_RING_PACK_TRACE || m == HE_RING_PACK_KEYSWITCH1;
}
static Mods4 make_mods4(const RingDims& R, uint32_t P2) {
  Mods4 M;
  M.m[0] = R.q[0];
  M.m[1] = R.q[1];
  M.m[2] = R.P;
  M.m[3] = P2;
  for (int j = 0; j < 4; ++j) M.mu[j] = (uint64_t)(((unsigned __int128)1 << 64) / M.m[j]);
  return M;
}
extern "C" he_status he_ring_pack_special2(const he_context* c, uint32_t* p2) {
  if (!c || !p2) return fail(HE_EINVAL, "null argument");
  *p2 = ring_pack_p2(c->R);
  return *p2 ? HE_OK : fail(HE_EINVAL, "no second special prime below 2^30 for N = %u", c->R.N);
}
extern "C" he_status he_ring_pack_key_bytes(const he_context* c, int method, uint64_t* bytes) {
  if (!c || !bytes) return fail(HE_EINVAL, "null argument");
  if (!rp_method_ok(method)) return fail(HE_EINVAL, "unknown method %d", method);
  *bytes = ring_pack_key_words(c, method) * sizeof(uint32_t);
  return HE_OK;
}

extern "C" he_status he_ring_pack_keygen(const he_context* c, int method, uint64_t seed, const int32_t* s_dev,
                                         uint32_t* keys_dev, void* stream) {
  if (!c || !s_dev || !keys_dev) return fail(HE_EINVAL, "null argument");
  if (!rp_method_ok(method)) return fail(HE_EINVAL, "unknown method %d", method);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N, d = c->R.d, k = c->R.k;
  const int logk = ilog2_u(k);
  const Mods M = make_mods(c->R);
  int32_t* sk = nullptr;
  HE_CUDA(cudaMallocAsync(&sk, N * sizeof(int32_t), st), "alloc");
  he_status s = HE_OK;
  if (method == HE_RING_PACK_KEYSWITCH1) {
    // keys [j][part (alpha, beta)][mod (q0, q1, P1, P2)][N], NTT domain: beta = -alpha s + e + P1 P2 s_j(X^k)
    // mod q0, q1 (0 mod P1, P2); key id 0x300 + j, one digit (i = 0)
    const uint32_t P2 = ring_pack_p2(c->R);
    if (!P2) s = fail(HE_EINVAL, "no second special prime");
    NttTable t2{};
    uint32_t* snew = nullptr;
    if (!s && ntt_table_init(t2, N, P2) != cudaSuccess) s = fail(HE_ECUDA, "P2 tables");
    if (!s && cudaMallocAsync(&snew, 4ull * N * sizeof(uint32_t), st) != cudaSuccess) s = fail(HE_ENOMEM, "alloc");
    const Mods4 M4 = make_mods4(c->R, P2);
    const NttTable* tab[4] = {&c->ntt[0], &c->ntt[1], &c->ntt[2], &t2};
    for (int mi = 0; mi < 4 && !s; ++mi) {
      k_reduce_signed<<<grid_for(N), 256, 0, st>>>(s_dev, N, M4.m[mi], snew + (size_t)mi * N);
      if (ntt_forward(*tab[mi], snew + (size_t)mi * N, 1, N, st) != cudaSuccess) s = fail(HE_ECUDA, "NTT(s)");
    }
    for (uint32_t j = 0; j < k && !s; ++j) {
      k_ms_component<<<grid_for(N), 256, 0, st>>>(s_dev, N, k, j, sk);
      for (int mi = 0; mi < 4 && !s; ++mi) {
        const uint32_t q = M4.m[mi];
        const uint32_t g = mi < 2 ? (uint32_t)((uint64_t)(c->R.P % q) * (P2 % q) % q) : 0u;
        uint32_t* alpha = keys_dev + ((size_t)j * 8 + 0 * 4 + mi) * N;
        uint32_t* beta = keys_dev + ((size_t)j * 8 + 1 * 4 + mi) * N;
        k_ksk_prep<<<grid_for(N), 256, 0, st>>>(M.rng, seed, 0x300 + j, 0, (uint32_t)mi, q, g, sk, N, alpha, beta);
        if (ntt_forward(*tab[mi], alpha, 1, N, st) != cudaSuccess || ntt_forward(*tab[mi], beta, 1, N, st) != cudaSuccess)
          s = fail(HE_ECUDA, "NTT(key)");
        k_ksk_beta<<<grid_for(N), 256, 0, st>>>(alpha, snew + (size_t)mi * N, N, q, beta);
      }
    }
    if (snew) cudaFreeAsync(snew, st);
    cudaStreamSynchronize(st);
    ntt_table_free(t2);
  } else if (method == HE_RING_PACK_TRACE) {
    for (int lv = 1; lv <= logk && !s; ++lv) {  // sigma_g(s) -> s, g = 1 + 2^l d
      k_secret_auto<<<grid_for(N), 256, 0, st>>>(s_dev, N, (d << lv) + 1, sk);
      s = make_ksk_dev(M, seed, 0x100 + lv, sk, s_dev, N, c->ntt, keys_dev + (size_t)(lv - 1) * 12 * N, st);
    }
  } else {
    for (uint32_t j = 0; j < k && !s; ++j) {     // s_j(X^k) -> s
      k_ms_component<<<grid_for(N), 256, 0, st>>>(s_dev, N, k, j, sk);
      s = make_ksk_dev(M, seed, 0x200 + j, sk, s_dev, N, c->ntt, keys_dev + (size_t)j * 12 * N, st);
    }
  }
  cudaFreeAsync(sk, st);
  if (s) return s;
  return cudaGetLastError() == cudaSuccess ? HE_OK : fail(HE_ECUDA, "ring pack keygen launch failed");
}

extern "C" he_status he_ring_pack_plan_create(const he_context* c, uint32_t n_out, int method,
                                              he_ring_pack_plan** out) {
  if (!c || !out) return fail(HE_EINVAL, "null argument");
  if (!rp_method_ok(method)) return fail(HE_EINVAL, "unknown method %d", method);
  const uint32_t k = c->R.k;
  if (n_out == 0 || n_out % k) return fail(HE_EINVAL, "n_out (%u) must be a positive multiple of k = %u", n_out, k);
  if (k > 256 || c->R.d % 32) return fail(HE_EINVAL, "ring packing needs k <= 256 and d a multiple of 32");
  if (method == HE_RING_PACK_KEYSWITCH1 && k % 4) return fail(HE_EINVAL, "keyswitch1 packing needs k %% 4 == 0");
  he_ring_pack_plan* p = new (std::nothrow) he_ring_pack_plan();
  if (!p) return fail(HE_ENOMEM, "out of host memory");
  p->ctx = c;
  p->method = method;
  p->n_out = n_out;
  p->d = c->R.d;
  p->k = k;
  p->N = c->R.N;
  p->logN = (uint32_t)ilog2_u(p->N);
  p->logk = (uint32_t)ilog2_u(k);
  p->blocks = n_out / k;
  static const int env_chunk = getenv("HE_RP_CHUNK") ? atoi(getenv("HE_RP_CHUNK")) : 0;  // blocks per pass
  static const int env_jc = getenv("HE_MS_JC") ? atoi(getenv("HE_MS_JC")) : 0;       // components per pass
  if (method == HE_RING_PACK_TRACE) {
    p->chunk = env_chunk > 0 ? (uint32_t)env_chunk : 8;
  } else {   // both key-switch methods
    p->chunk = env_chunk > 0 && env_chunk <= kMsMaxYc ? (uint32_t)env_chunk : kMsMaxYc;
    p->jc = env_jc > 0 ? (uint32_t)env_jc : 32;  // measured: 4 -> 14.6, 16 -> 11.8, 32 -> 11.0, 64 -> 10.8 ms
    if (p->jc > k) p->jc = k;
    while (k % p->jc) --p->jc;
  }
  if (p->chunk > p->blocks) p->chunk = p->blocks;
  p->M = make_mods(c->R);
  for (int i = 0; i < 2; ++i) {
    const uint32_t qi = p->M.m[i];
    p->qhinv[i] = (uint32_t)powmod_h(p->M.m[1 - i] % qi, qi - 2, qi);
    p->pinv[i] = (uint32_t)powmod_h(p->M.m[2] % qi, qi - 2, qi);
    p->kinv[i] = (uint32_t)powmod_h(k, qi - 2, qi);
    p->kinvp[i] = shoup_pre(p->kinv[i], qi);
  }
  p->q1inv = (uint32_t)powmod_h(p->M.m[1] % p->M.m[0], p->M.m[0] - 2, p->M.m[0]);
  p->q1invp = shoup_pre(p->q1inv, p->M.m[0]);
  if (method == HE_RING_PACK_KEYSWITCH1) {
    const uint32_t P2 = ring_pack_p2(c->R);
    if (!P2 || ntt_table_init(p->ntt_p2, c->R.N, P2) != cudaSuccess) {
      delete p;
      return fail(HE_EINVAL, "no NTT-friendly second special prime for N = %u", c->R.N);
    }
    p->M4 = make_mods4(c->R, P2);
    const uint32_t q0 = p->M4.m[0], q1 = p->M4.m[1], P1 = p->M4.m[2];
    p->q0inv_q1 = (uint32_t)powmod_h(q0 % q1, q1 - 2, q1);
    p->p1inv_p2 = (uint32_t)powmod_h(P1 % P2, P2 - 2, P2);
    for (int i = 0; i < 2; ++i) {
      const uint32_t qi = p->M4.m[i];
      p->ppinv[i] = (uint32_t)powmod_h((uint64_t)(P1 % qi) * (P2 % qi) % qi, qi - 2, qi);
    }
  }
  // NTT-domain tables at degree N: output c of the forward transform holds p(psi^{2 brv(c) + 1})
  const uint32_t N = p->N, logN = p->logN, logk = p->logk;
  std::vector<uint32_t> h((size_t)logk * N * 3);
  uint32_t* perm = h.data();
  uint32_t* mono = h.data() + (size_t)logk * N;
  std::vector<uint32_t> pw(2ull * N);
  for (int L = 0; L < 2; ++L) {
    const uint32_t q = p->M.m[L];
    const uint64_t psi = find_psi(q, N);
    if (!psi) {
      delete p;
      return fail(HE_EINVAL, "q%d is not NTT-friendly at degree %u", L, N);
    }
    uint64_t acc = 1;
    for (uint64_t e = 0; e < 2ull * N; ++e, acc = acc * psi % q) pw[e] = (uint32_t)acc;
    for (uint32_t lv = 1; lv <= logk; ++lv) {
      const uint64_t ex = k >> lv;  // X^{k / 2^l}
      for (uint32_t cc = 0; cc < N; ++cc) {
        const uint64_t e = 2ull * bitrev_h(cc, (int)logN) + 1;
        mono[((size_t)(lv - 1) * 2 + L) * N + cc] = pw[(e * ex) % (2ull * N)];
      }
    }
  }
  for (uint32_t lv = 1; lv <= logk; ++lv) {
    const uint64_t g = ((uint64_t)p->d << lv) + 1;
    for (uint32_t cc = 0; cc < N; ++cc) {
      const uint64_t e = 2ull * bitrev_h(cc, (int)logN) + 1;
      const uint64_t eg = (e * g) % (2ull * N);
      perm[(size_t)(lv - 1) * N + cc] = bitrev_h((uint32_t)((eg - 1) / 2), (int)logN);
    }
  }
  if (cudaMalloc(&p->tables, h.size() * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemcpy(p->tables, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    delete p;
    return fail(HE_ECUDA, "ring pack tables");
  }
  *out = p;
  return HE_OK;
}

extern "C" he_status he_ring_pack_plan_destroy(he_ring_pack_plan* p) {
  if (p) {
    if (p->tables) cudaFree(p->tables);
    ntt_table_free(p->ntt_p2);
    delete p;
  }
  return HE_OK;
}

struct RpWs {
  uint32_t *A0, *A1, *T, *C, *D, *UW, *LB;
};
static uint64_t rp_ws_words(const he_ring_pack_plan* p, RpWs* w, uint32_t* base) {
  const uint64_t N = p->N, cnt = (uint64_t)p->chunk * p->k, c1 = cnt / 2;
  uint64_t off = 0;
  auto take = [&](uint32_t*& ptr, uint64_t words) {
    if (w) ptr = base + off;
    off += (words + 63) & ~63ull;
  };
  RpWs dummy;
  RpWs& r = w ? *w : dummy;
  if (p->method == HE_RING_PACK_KEYSWITCH) {  // D [3][2][jc * Yc][N], UW [3][2][Yc][N]
    take(r.D, 6ull * p->jc * p->chunk * N);
    take(r.UW, 6ull * p->chunk * N);
    return off;
  }
  if (p->method == HE_RING_PACK_KEYSWITCH1) {  // D [4][jc * Yc][N], UW [4][2][Yc][N]
    take(r.D, 4ull * p->jc * p->chunk * N);
    take(r.UW, 8ull * p->chunk * N);
    return off;
  }
  take(r.A0, 2ull * cnt * 2 * N);
  take(r.A1, 2ull * c1 * 2 * N);
  take(r.T, 2ull * c1 * 2 * N);
  take(r.C, 2ull * c1 * N);
  take(r.D, 6ull * c1 * N);
  take(r.UW, 6ull * c1 * N);
  take(r.LB, 4ull * c1 * N);
  return off;
}

extern "C" he_status he_ring_pack_workspace_bytes(const he_ring_pack_plan* p, uint64_t* bytes) {
  if (!p || !bytes) return fail(HE_EINVAL, "null argument");
  *bytes = rp_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  return HE_OK;
}

extern "C" he_status he_ring_pack_run(const he_ring_pack_plan* p, const uint32_t* raw_b, const uint32_t* raw_a,
                                      const uint32_t* gal, uint32_t* out, void* ws_dev, uint64_t ws_bytes,
                                      void* stream, he_ledger* ledger) {
  if (!p) return fail(HE_EINVAL, "null plan");
  if (!raw_b || !raw_a || !gal || !out || !ws_dev) return fail(HE_EINVAL, "null argument");
  const uint64_t need = rp_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  if (ws_bytes < need)
    return fail(HE_EINVAL, "workspace too small (%llu < %llu)", (unsigned long long)ws_bytes, (unsigned long long)need);
  cudaStream_t st = (cudaStream_t)stream;
  const he_context* c = p->ctx;
  const uint32_t N = p->N, k = p->k, d = p->d, q0 = p->M.m[0], q1 = p->M.m[1];
  RpWs w;
  rp_ws_words(p, &w, (uint32_t*)ws_dev);
  if (p->method == HE_RING_PACK_KEYSWITCH) {
    const uint32_t qh0p = shoup_pre(p->qhinv[0], q0), qh1p = shoup_pre(p->qhinv[1], q1);
    for (uint32_t Y0 = 0; Y0 < p->blocks; Y0 += p->chunk) {
      const uint32_t Yc = (p->blocks - Y0 < p->chunk) ? p->blocks - Y0 : p->chunk;
      const uint32_t cnt = p->jc * Yc;
      HE_CUDA(cudaMemsetAsync(w.UW, 0, 6ull * Yc * N * sizeof(uint32_t), st), "memset");
      for (uint32_t j0 = 0; j0 < k; j0 += p->jc) {
        k_ms_digits<<<dim3(d / 32, cnt), 256, 0, st>>>(raw_a, p->n_out, Y0, j0, Yc, cnt, d, k, N, p->M, p->qhinv[0],
                                                      qh0p, p->qhinv[1], qh1p, w.D);
        HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1], &c->ntt[2]},
                         {w.D, w.D + 2ull * cnt * N, w.D + 4ull * cnt * N}, 2 * cnt, N, st), "NTT(digits)");
        k_ms_mac<<<dim3((unsigned)(((uint64_t)Yc * N / 4 + 255) / 256), 3), 256, 0, st>>>(w.D, gal + (size_t)j0 * 12 * N, p->jc,
                                                                                   Yc, p->logN, p->M, w.UW);
      }
      HE_CUDA(ntt_jobs(true, {&c->ntt[0], &c->ntt[1], &c->ntt[2]}, {w.UW, w.UW + 2ull * Yc * N, w.UW + 4ull * Yc * N},
                       2 * Yc, N, st), "INTT(U, W)");
      k_ms_finish<<<grid_for((uint64_t)Yc * N), 256, 0, st>>>(w.UW, raw_b, p->blocks, Y0, Yc, p->logN, p->M, p->pinv[0],
                                                               p->pinv[1], p->q1inv, p->q1invp, out);
    }
    HE_CUDA(cudaGetLastError(), "ring pack launch");
    if (ledger) ledger->rescales += p->blocks;  // k key switches per block, no rotations
    return HE_OK;
  }
  if (p->method == HE_RING_PACK_KEYSWITCH1) {
    const NttTable* tab[4] = {&c->ntt[0], &c->ntt[1], &c->ntt[2], &p->ntt_p2};
    // Llama ring (N = 2^16, k = d = 256): digits fused with the NTT's cols pass; HE_RP_UNFUSED=1 keeps the
    // separate kernels (the path every other ring size takes) for A/B checks
    const bool fused = getenv("HE_RP_UNFUSED") == nullptr && N == 65536 && k == 256 && d == 256;
    const size_t fused_smem = (size_t)2 * kMs1T * kMs1Pitch * sizeof(uint32_t);
    Ms1Tw tw4;
    for (int mod = 0; mod < 4; ++mod)
      for (int i = 0; i < 16; ++i) tw4.tw[mod][i] = tab[mod]->fw16[i];
    {
      const uint32_t q0m = p->M4.m[0], q1m = p->M4.m[1];
      tw4.m1 = (uint32_t)(0x100000000ull / q1m);
      tw4.w01 = p->q0inv_q1;
      tw4.w01p = shoup_pre(p->q0inv_q1, q1m);
      tw4.Q = (uint64_t)q0m * q1m;
      for (int i = 0; i < 2; ++i) {
        const uint32_t P = p->M4.m[2 + i];
        tw4.c[i] = q0m % P;
        tw4.cp[i] = shoup_pre(tw4.c[i], P);
        tw4.qp[i] = (uint32_t)(tw4.Q % P);
      }
    }
    if (fused)
      HE_CUDA(cudaFuncSetAttribute(k_ms1_digits_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem),
              "smem attribute");
    for (uint32_t Y0 = 0; Y0 < p->blocks; Y0 += p->chunk) {
      const uint32_t Yc = (p->blocks - Y0 < p->chunk) ? p->blocks - Y0 : p->chunk;
      const uint32_t cnt = p->jc * Yc;
      HE_CUDA(cudaMemsetAsync(w.UW, 0, 8ull * Yc * N * sizeof(uint32_t), st), "memset");
      for (uint32_t j0 = 0; j0 < k; j0 += p->jc) {
        if (fused) {   // digits + the NTT's outer stages in one pass over a' (k_ms1_digits_cols)
          k_ms1_digits_cols<<<dim3(k / kMs1T, cnt), 256, fused_smem, st>>>(raw_a, p->n_out, Y0, j0, Yc, cnt, p->M4,
                                                                          p->q0inv_q1, tw4, w.D);
        } else {
          k_ms1_digits<<<dim3(d / kMs1M, cnt), 256, 0, st>>>(raw_a, p->n_out, Y0, j0, Yc, cnt, d, k, N, p->M4,
                                                             p->q0inv_q1, w.D);
        }
        // the MAC over 8 blocks reduces its inputs itself (free in a memory-bound kernel), so the rows pass
        // skips its final reduction; HE_RP_NTT_REDUCE=1 keeps it there (A/B)
        static const bool ntt_reduce = getenv("HE_RP_NTT_REDUCE") != nullptr;
        const bool mac_y = Yc % kMacY == 0 && getenv("HE_RP_MAC4") == nullptr;
        const bool lazy = mac_y && !ntt_reduce;
        {
          uint32_t* dd[4] = {w.D, w.D + (size_t)cnt * N, w.D + 2ull * cnt * N, w.D + 3ull * cnt * N};
          HE_CUDA(ntt_forward_multi(tab, dd, 4, cnt, N, st, fused, !lazy), "NTT(digits)");
        }
        if (mac_y) {
          auto mac = lazy ? k_ms1_mac_y<true> : k_ms1_mac_y<false>;
          mac<<<dim3((unsigned)(N / 2 / 256), Yc / kMacY, 4), 256, 0, st>>>(w.D, gal + (size_t)j0 * 8 * N, p->jc, Yc,
                                                                         p->logN, p->M4, w.UW);
        } else {
          k_ms1_mac<<<dim3((unsigned)(((uint64_t)Yc * N / 4 + 255) / 256), 4), 256, 0, st>>>(
              w.D, gal + (size_t)j0 * 8 * N, p->jc, Yc, p->logN, p->M4, w.UW);
        }
      }
      {
        uint32_t* dd[4] = {w.UW, w.UW + 2ull * Yc * N, w.UW + 4ull * Yc * N, w.UW + 6ull * Yc * N};
        HE_CUDA(ntt_inverse_multi(tab, dd, 4, 2 * Yc, N, st), "INTT(U, W)");
      }
      k_ms1_finish<<<grid_for((uint64_t)Yc * N), 256, 0, st>>>(w.UW, raw_b, p->blocks, Y0, Yc, p->logN, p->M4,
                                                                p->p1inv_p2, p->ppinv[0], p->ppinv[1], p->q1inv,
                                                                p->q1invp, out);
    }
    HE_CUDA(cudaGetLastError(), "ring pack launch");
    if (ledger) ledger->rescales += p->blocks;
    return HE_OK;
  }
  const uint32_t* perm_base = p->tables;
  const uint32_t* mono_base = p->tables + (size_t)p->logk * N;
  for (uint32_t b0 = 0; b0 < p->blocks; b0 += p->chunk) {
    const uint32_t nb = (p->blocks - b0 < p->chunk) ? p->blocks - b0 : p->chunk;
    uint32_t cnt = nb * k;
    const uint32_t y0 = b0 * k;
    k_rp_leaves_a<<<dim3(d / 32, cnt, 2), 256, 0, st>>>(raw_a, (uint64_t)p->n_out * N, y0, d, k, N, cnt, p->kinv[0],
                                                         p->kinvp[0], p->kinv[1], p->kinvp[1], q0, q1, w.A0);
    {
      dim3 g = grid_for((uint64_t)cnt * N);
      g.y = 2;
      k_rp_leaves_b<<<g, 256, 0, st>>>(raw_b, (uint64_t)p->blocks * N, y0, k, p->logN, cnt, p->kinv[0], p->kinvp[0],
                                       p->kinv[1], p->kinvp[1], q0, q1, w.A0);
    }
    for (int L = 0; L < 2; ++L)
      HE_CUDA(ntt_forward(c->ntt[L], w.A0 + (size_t)L * cnt * 2 * N, cnt * 2, N, st), "NTT(leaves)");
    uint32_t* A = w.A0;
    uint32_t* An = w.A1;
    for (uint32_t lv = 1; lv <= p->logk; ++lv) {
      const uint32_t cnt_out = cnt / 2, half = k >> lv;
      const uint64_t cn = (uint64_t)cnt_out * N;
      {
        dim3 g = grid_for(cn);
        g.y = 2;
        g.z = 2;
        k_rp_comb1<<<g, 256, 0, st>>>(A, cnt, half, p->logN, mono_base + (size_t)(lv - 1) * 2 * N,
                                      perm_base + (size_t)(lv - 1) * N, p->M, An, w.T, w.C);
      }
      for (int L = 0; L < 2; ++L) HE_CUDA(ntt_inverse(c->ntt[L], w.C + (size_t)L * cn, cnt_out, N, st), "INTT(T_a)");
      k_modup<<<grid_for(cn), 256, 0, st>>>(w.C, w.T, p->logN, cn, p->M, p->qhinv[0], p->qhinv[1], w.D);
      HE_CUDA(ntt_forward(c->ntt[0], w.D + (0 * 2 + 1) * cn, cnt_out, N, st), "NTT(d1 mod q0)");
      HE_CUDA(ntt_forward(c->ntt[1], w.D + (1 * 2 + 0) * cn, cnt_out, N, st), "NTT(d0 mod q1)");
      HE_CUDA(ntt_forward(c->ntt[2], w.D + (2 * 2 + 0) * cn, 2 * cnt_out, N, st), "NTT(d mod P)");
      k_mac<<<grid_for(cn), 256, 0, st>>>(w.D, gal + (size_t)(lv - 1) * 12 * N, N, cn, p->M, w.UW);
      HE_CUDA(ntt_inverse(c->ntt[2], w.UW + 2 * 2 * cn, 2 * cnt_out, N, st), "INTT(U_P, W_P)");
      k_moddown_lift<<<grid_for(2 * cn), 256, 0, st>>>(w.UW + 2 * 2 * cn, cn, p->M, w.LB);
      HE_CUDA(ntt_forward(c->ntt[0], w.LB, 2 * cnt_out, N, st), "NTT(lift q0)");
      HE_CUDA(ntt_forward(c->ntt[1], w.LB + 2 * cn, 2 * cnt_out, N, st), "NTT(lift q1)");
      {
        dim3 g = grid_for(cn / 4);
        g.y = 2;
        k_pack_comb2<<<g, 256, 0, st>>>(w.UW, w.LB, w.T, cnt_out, p->logN, p->M, p->pinv[0], p->pinv[1], An);
      }
      uint32_t* tmp = A;
      A = An;
      An = (lv == 1) ? w.A0 : tmp;
      cnt = cnt_out;
    }
    // cnt == nb: INTT and rescale into out [b0 ..][2][N]
    for (int L = 0; L < 2; ++L)
      HE_CUDA(ntt_inverse(c->ntt[L], A + (size_t)L * nb * 2 * N, nb * 2, N, st), "INTT(packed)");
    k_rp_rescale<<<grid_for((uint64_t)nb * 2 * N), 256, 0, st>>>(A, (uint64_t)nb * 2 * N, q0, q1, p->q1inv, p->q1invp,
                                                                  out + (size_t)b0 * 2 * N);
  }
  HE_CUDA(cudaGetLastError(), "ring pack launch");
  if (ledger) {
    ledger->ct_rotations += (int64_t)(k - 1) * p->blocks;
    ledger->rescales += p->blocks;
  }
  return HE_OK;
}

// ======================================================================== slot-domain BSGS PCMM (§8f3)
// hesim pcmm_bsgs (matmul.py:165-176) on real CKKS ciphertexts at degree N; restated from
// oracle/he_oracle_rhombus.c (or_slot_pcmm), bit-exact.  Ciphertexts live in the NTT domain between
// steps; a left slot rotation by r is X -> X^(5^r) (an index permutation of NTT values) plus a
// hybrid key switch of the lifted digits (hoisted: the digits of the input are formed and
// transformed once for all b - 1 baby rotations).
namespace {

// Gadget key switching for the slot rotations (oracle or_ksk_gen_gadget): each RNS digit d_i is split
// into kSdSub = 2 sub-digits of kSdBits = 15 bits, so the key-switching noise is ~2^15 below the plain
// dnum-2 key's -- the baby rotations act on the input at scale Delta = 2^26.  Sub-digits are < 2^15,
// i.e. the same value under every modulus: D [mod][t = i kSdSub + h][N] (coefficient form).
constexpr int kSdSub = 2;
constexpr int kSdBits = 15;
constexpr int kSdT = 2 * kSdSub;   // digit polys per modulus
// Batched over z = blockIdx.z sources (all baby rotations, or all giant groups, in one launch).
// digits of source z: a-part at a + z * as (limb stride ls) -> D [mod][z][t][N]  (cnt sources)
__global__ void k_sd_digits(const uint32_t* __restrict__ a, uint64_t as, uint64_t ls, uint32_t N, uint32_t cnt, Mods M,
                            uint32_t qh0, uint32_t qh0p, uint32_t qh1, uint32_t qh1p, uint32_t* __restrict__ D) {
  const uint32_t z = blockIdx.z;
  const uint32_t* src = a + z * as;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < N; x += gridDim.x * blockDim.x) {
    const uint32_t dg[2] = {shoup_mul(src[x], qh0, qh0p, M.m[0]), shoup_mul(src[ls + x], qh1, qh1p, M.m[1])};
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int h = 0; h < kSdSub; ++h) {
        const uint32_t v = (dg[i] >> (kSdBits * h)) & ((1u << kSdBits) - 1u);
#pragma unroll
        for (int mod = 0; mod < 3; ++mod) D[(((size_t)mod * cnt + z) * kSdT + i * kSdSub + h) * N + x] = v;
      }
  }
}
// plain dnum-2 digits: D^ [mod][z][i < 2][N] = d_i mod m_mod, d_i = [a_i (q/q_i)^-1]_{q_i}
__global__ void k_sd_digits_plain(const uint32_t* __restrict__ a, uint64_t as, uint64_t ls, uint32_t N, uint32_t cnt,
                                  Mods M, uint32_t qh0, uint32_t qh0p, uint32_t qh1, uint32_t qh1p,
                                  uint32_t* __restrict__ D) {
  const uint32_t z = blockIdx.z;
  const uint32_t* src = a + z * as;
  for (uint32_t x4 = blockIdx.x * blockDim.x + threadIdx.x; x4 < N / 4; x4 += gridDim.x * blockDim.x) {
    const uint4 a0 = reinterpret_cast<const uint4*>(src)[x4], a1 = reinterpret_cast<const uint4*>(src + ls)[x4];
    const uint32_t v0[4] = {a0.x, a0.y, a0.z, a0.w}, v1[4] = {a1.x, a1.y, a1.z, a1.w};
    uint32_t dg[2][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      dg[0][e] = shoup_mul(v0[e], qh0, qh0p, M.m[0]);
      dg[1][e] = shoup_mul(v1[e], qh1, qh1p, M.m[1]);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int mod = 0; mod < 3; ++mod) {
        const uint32_t q = M.m[mod];
        const uint64_t mu = M.mu[mod];
        uint32_t r[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) r[e] = barrett64(dg[i][e], mu, q);
        reinterpret_cast<uint4*>(D + (((size_t)mod * cnt + z) * 2 + i) * N)[x4] = make_uint4(r[0], r[1], r[2], r[3]);
      }
  }
}
// rotation z: UW [mod][z][part][N] = sum_t D^[mod][dz][t][perm_z c] K_z[t][part][mod][c]   (dz = hoist ? 0 : z)
template <int T>   // digits per key: kSdT (gadget keys) or 2 (plain dnum-2 keys, 12N words)
__global__ void k_sd_mac_t(const uint32_t* __restrict__ D, uint32_t dcnt, int hoist, const uint32_t* __restrict__ perms,
                           const uint32_t* __restrict__ K, uint32_t N, uint32_t cnt, Mods M, uint32_t* __restrict__ UW) {
  const uint32_t mod = blockIdx.y, z = blockIdx.z, dz = hoist ? 0 : z;
  const uint32_t q = mod == 0 ? M.m[0] : (mod == 1 ? M.m[1] : M.m[2]);
  const uint64_t mu = mod == 0 ? M.mu[0] : (mod == 1 ? M.mu[1] : M.mu[2]);
  const uint32_t* perm = perms + (size_t)z * N;
  const uint32_t* Kz = K + (size_t)z * T * 6 * N;
  const uint32_t* Dz = D + ((size_t)mod * dcnt + dz) * T * N;
  for (uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x; c4 < N / 4; c4 += gridDim.x * blockDim.x) {
    const uint4 pv = reinterpret_cast<const uint4*>(perm)[c4];   // 4 coefficients per thread, 16-byte I/O
    const uint32_t pc[4] = {pv.x, pv.y, pv.z, pv.w};
    uint64_t u[4] = {0, 0, 0, 0}, w[4] = {0, 0, 0, 0};   // T products < 2^60 each
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const uint4 ku = reinterpret_cast<const uint4*>(Kz + (size_t)((t * 2 + 0) * 3 + mod) * N)[c4];
      const uint4 kw = reinterpret_cast<const uint4*>(Kz + (size_t)((t * 2 + 1) * 3 + mod) * N)[c4];
      const uint32_t kus[4] = {ku.x, ku.y, ku.z, ku.w}, kws[4] = {kw.x, kw.y, kw.z, kw.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t dv = Dz[(size_t)t * N + pc[e]];
        u[e] += dv * kus[e];
        w[e] += dv * kws[e];
      }
    }
    reinterpret_cast<uint4*>(UW + (((size_t)mod * cnt + z) * 2 + 0) * N)[c4] =
        make_uint4(barrett64(u[0], mu, q), barrett64(u[1], mu, q), barrett64(u[2], mu, q), barrett64(u[3], mu, q));
    reinterpret_cast<uint4*>(UW + (((size_t)mod * cnt + z) * 2 + 1) * N)[c4] =
        make_uint4(barrett64(w[0], mu, q), barrett64(w[1], mu, q), barrett64(w[2], mu, q), barrett64(w[3], mu, q));
  }
}
// lazy form of k_sd_mac for the baby steps of cc ciphertexts (one key read serves all; 6.3 MB per rotation):
// each rotation written straight as the PQ-basis ct (U, W + P sigma(b^)) -- no ModDown, no UW round trip;
// digits D^ [mod][ct][t][N], NTT'd cts X [ct][L][ab][N], rotation z of ct -> out + ct os + z 6N
__global__ void k_sd_mac_lazy_multi(const uint32_t* __restrict__ D, uint32_t cc, const uint32_t* __restrict__ perms,
                                    const uint32_t* __restrict__ K, const uint32_t* __restrict__ X, uint32_t N, Mods M,
                                    uint32_t* __restrict__ out, uint64_t os) {
  const uint32_t mod = blockIdx.y, z = blockIdx.z;
  const uint32_t q = mod == 0 ? M.m[0] : (mod == 1 ? M.m[1] : M.m[2]);
  const uint64_t mu = mod == 0 ? M.mu[0] : (mod == 1 ? M.mu[1] : M.mu[2]);
  const uint32_t pm = M.m[2] % q;
  const uint32_t* perm = perms + (size_t)z * N;
  const uint32_t* Kz = K + (size_t)z * 24 * N;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    const uint32_t pc = perm[c];
    uint32_t ku[kSdT], kw[kSdT];
#pragma unroll
    for (int t = 0; t < kSdT; ++t) {
      ku[t] = Kz[(size_t)((t * 2 + 0) * 3 + mod) * N + c];
      kw[t] = Kz[(size_t)((t * 2 + 1) * 3 + mod) * N + c];
    }
    for (uint32_t ct = 0; ct < cc; ++ct) {
      const uint32_t* Dz = D + ((size_t)mod * cc + ct) * kSdT * N;
      uint64_t u = 0, w = 0;
#pragma unroll
      for (int t = 0; t < kSdT; ++t) {
        const uint64_t dv = Dz[(size_t)t * N + pc];
        u += dv * ku[t];
        w += dv * kw[t];
      }
      uint32_t* o = out + ct * os + (size_t)z * 6 * N + (size_t)mod * 2 * N;
      o[c] = barrett64(u, mu, q);
      const uint32_t wr = barrett64(w, mu, q);
      o[N + c] = mod < 2 ? add_mod(wr, mulmod_b(X[(size_t)ct * 4 * N + mod * 2 * N + N + pc], pm, mu, q), q) : wr;
    }
  }
}
// rotated ct z (NTT domain) [L][ab][N] at out + z * os: a = (U - LB_u) P^-1, b = sigma(b^_z) + (W - LB_w) P^-1
// (LB [L][z][part][N]; b^_z at bh + z * bs, limb stride bls)
__global__ void k_sd_combine(const uint32_t* __restrict__ UW, const uint32_t* __restrict__ LB,
                             const uint32_t* __restrict__ bh, uint64_t bs, uint64_t bls,
                             const uint32_t* __restrict__ perms, uint32_t N, uint32_t cnt, Mods M, uint32_t pinv0,
                             uint32_t pinv1, uint32_t* __restrict__ out, uint64_t os) {
  const uint32_t L = blockIdx.y, z = blockIdx.z, q = M.m[L], pinv = L ? pinv1 : pinv0;
  const uint64_t mu = M.mu[L];
  const uint32_t* perm = perms + (size_t)z * N;
  const uint32_t* U = UW + (((size_t)L * cnt + z) * 2) * N;
  const uint32_t* lb = LB + (((size_t)L * cnt + z) * 2) * N;
  const uint32_t* b = bh + z * bs + L * bls;
  uint32_t* o = out + z * os + (size_t)L * 2 * N;
  for (uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x; c4 < N / 4; c4 += gridDim.x * blockDim.x) {
    const uint4 uu = reinterpret_cast<const uint4*>(U)[c4], lu = reinterpret_cast<const uint4*>(lb)[c4];
    const uint4 uw = reinterpret_cast<const uint4*>(U + N)[c4], lw = reinterpret_cast<const uint4*>(lb + N)[c4];
    const uint4 pc = reinterpret_cast<const uint4*>(perm)[c4];
    reinterpret_cast<uint4*>(o)[c4] =
        make_uint4(mulmod_b(sub_mod(uu.x, lu.x, q), pinv, mu, q), mulmod_b(sub_mod(uu.y, lu.y, q), pinv, mu, q),
                   mulmod_b(sub_mod(uu.z, lu.z, q), pinv, mu, q), mulmod_b(sub_mod(uu.w, lu.w, q), pinv, mu, q));
    reinterpret_cast<uint4*>(o + N)[c4] =
        make_uint4(add_mod(b[pc.x], mulmod_b(sub_mod(uw.x, lw.x, q), pinv, mu, q), q),
                   add_mod(b[pc.y], mulmod_b(sub_mod(uw.y, lw.y, q), pinv, mu, q), q),
                   add_mod(b[pc.z], mulmod_b(sub_mod(uw.z, lw.z, q), pinv, mu, q), q),
                   add_mod(b[pc.w], mulmod_b(sub_mod(uw.w, lw.w, q), pinv, mu, q), q));
  }
}
// inner_z [L][ab][N] = sum_{i < b} pt[i + z b][L] * baby[i][L][ab]   (NTT domain), z = giant group
__global__ void k_sd_inner(const uint32_t* __restrict__ baby, const uint32_t* __restrict__ pts, uint32_t b, uint32_t N,
                           Mods M, uint32_t* __restrict__ inner) {
  const uint32_t L = blockIdx.y, j = blockIdx.z, q = M.m[L];
  const uint64_t mu = M.mu[L];
  for (uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x; c4 < N / 4; c4 += gridDim.x * blockDim.x) {
    uint64_t aa[4] = {0, 0, 0, 0}, ab[4] = {0, 0, 0, 0};   // 4 coefficients per thread: 16-byte accesses
    for (uint32_t i = 0; i < b; ++i) {
      const uint4 p = __ldg(reinterpret_cast<const uint4*>(pts + ((size_t)(i + j * b) * 2 + L) * N) + c4);
      const uint4 x = reinterpret_cast<const uint4*>(baby + ((size_t)i * 4 + L * 2) * N)[c4];
      const uint4 y = reinterpret_cast<const uint4*>(baby + ((size_t)i * 4 + L * 2 + 1) * N)[c4];
      const uint32_t ps[4] = {p.x, p.y, p.z, p.w}, xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        aa[e] = barrett64(aa[e] + (uint64_t)ps[e] * xs[e], mu, q);
        ab[e] = barrett64(ab[e] + (uint64_t)ps[e] * ys[e], mu, q);
      }
    }
    reinterpret_cast<uint4*>(inner + ((size_t)j * 4 + L * 2 + 0) * N)[c4] =
        make_uint4((uint32_t)aa[0], (uint32_t)aa[1], (uint32_t)aa[2], (uint32_t)aa[3]);
    reinterpret_cast<uint4*>(inner + ((size_t)j * 4 + L * 2 + 1) * N)[c4] =
        make_uint4((uint32_t)ab[0], (uint32_t)ab[1], (uint32_t)ab[2], (uint32_t)ab[3]);
  }
}
// the same sums for JG giant groups per thread (2 coefficients per thread): each baby word is read once per JG
// groups instead of once per group (StC: b = 256 baby cts = 268 MB, re-read g = 128 times without this);
// products < 2^60 accumulate lazily, reduced every 8 terms
template <int JG>
__global__ void k_sd_inner_g(const uint32_t* __restrict__ baby, const uint32_t* __restrict__ pts, uint32_t b,
                             uint32_t g, uint32_t N, Mods M, uint32_t* __restrict__ inner) {
  const uint32_t L = blockIdx.y, j0 = blockIdx.z * JG, q = M.m[L];
  const uint64_t mu = M.mu[L];
  for (uint32_t c2 = blockIdx.x * blockDim.x + threadIdx.x; c2 < N / 2; c2 += gridDim.x * blockDim.x) {
    uint64_t acc[JG][4];
#pragma unroll
    for (int jj = 0; jj < JG; ++jj)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[jj][e] = 0;
    for (uint32_t i = 0; i < b; ++i) {
      const uint2 x = reinterpret_cast<const uint2*>(baby + ((size_t)i * 4 + L * 2) * N)[c2];
      const uint2 y = reinterpret_cast<const uint2*>(baby + ((size_t)i * 4 + L * 2 + 1) * N)[c2];
#pragma unroll
      for (int jj = 0; jj < JG; ++jj) {
        if (j0 + jj < g) {
          const uint2 p = __ldg(reinterpret_cast<const uint2*>(pts + ((size_t)(i + (j0 + jj) * b) * 2 + L) * N) + c2);
          acc[jj][0] += (uint64_t)p.x * x.x;
          acc[jj][1] += (uint64_t)p.y * x.y;
          acc[jj][2] += (uint64_t)p.x * y.x;
          acc[jj][3] += (uint64_t)p.y * y.y;
        }
      }
      if ((i & 7) == 7) {
#pragma unroll
        for (int jj = 0; jj < JG; ++jj)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[jj][e] = barrett64(acc[jj][e], mu, q);
      }
    }
#pragma unroll
    for (int jj = 0; jj < JG; ++jj) {
      if (j0 + jj < g) {
        uint32_t* o = inner + ((size_t)(j0 + jj) * 4 + L * 2) * N;
        reinterpret_cast<uint2*>(o)[c2] = make_uint2(barrett64(acc[jj][0], mu, q), barrett64(acc[jj][1], mu, q));
        reinterpret_cast<uint2*>(o + N)[c2] = make_uint2(barrett64(acc[jj][2], mu, q), barrett64(acc[jj][3], mu, q));
      }
    }
  }
}
// the products for CT ciphertexts at once (big maps, e.g. SlotToCoeffs: 32 768 plaintexts = 17 GiB): a CTA owns 32
// coefficients of one limb, stages the CT baby sets of that tile in shared memory ([ct][i][lane][a, b] pairs,
// CT b 256 B) and streams every plaintext word of the tile exactly once, using it for all CT ciphertexts; warp w
// runs the groups 2w, 2w + 1 (+32 ...), 16 plaintext terms per group loaded ahead.  q < 2^30: products < 2^60,
// so 8 of them plus a folded sum (< 2^62 + 2^32) stay below 2^64 -- one 32-bit fold per 8 terms, one
// Barrett reduction per group
constexpr int kSdTile = 32;
constexpr int kSdSharedThreads = 512;   // 16 warps; 256 threads with 32 terms ahead measured 7% slower
template <int CT, int U, int GW = 2>   // GW giant groups per warp
__global__ void __launch_bounds__(kSdSharedThreads, 1)
    k_sd_inner_s(const uint32_t* __restrict__ baby, uint64_t baby_cs, const uint32_t* __restrict__ pts, uint32_t b,
                 uint32_t g, uint32_t N, uint32_t nl, Mods M, uint32_t* __restrict__ inner, uint64_t inner_cs,
                 uint32_t ib, uint32_t bn, int accumulate) {
  // baby terms i in [ib, ib + bn) of the b per group; accumulate: add the sums already in inner (second half)
  extern __shared__ __align__(16) uint32_t sbaby[];
  const uint32_t L = blockIdx.y, c0 = blockIdx.x * kSdTile, q = M.m[L];
  const uint64_t mu = M.mu[L];
  const uint32_t r32 = (uint32_t)((1ull << 32) % q);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // stage: row r = ct bn + i holds 32 (a, b) pairs; 8 threads per row, 4 coefficients each
  for (uint32_t r = threadIdx.x >> 3; r < CT * bn; r += blockDim.x >> 3) {
    const uint32_t ct = r / bn, i = ib + r % bn, t = threadIdx.x & 7;
    const uint32_t* src = baby + ct * baby_cs + ((size_t)i * nl + L) * 2 * N + c0;
    const uint4 va = reinterpret_cast<const uint4*>(src)[t];
    const uint4 vb = reinterpret_cast<const uint4*>(src + N)[t];
    uint4* dst = reinterpret_cast<uint4*>(sbaby + (size_t)r * 2 * kSdTile) + 2 * t;
    dst[0] = make_uint4(va.x, vb.x, va.y, vb.y);
    dst[1] = make_uint4(va.z, vb.z, va.w, vb.w);
  }
  __syncthreads();
  const size_t tstride = (size_t)nl * N;   // words between consecutive terms
  const uint2* sl = reinterpret_cast<const uint2*>(sbaby) + lane;
  for (uint32_t j0 = warp * GW; j0 < g; j0 += GW * (blockDim.x >> 5)) {
    const uint32_t* Pg[GW];
#pragma unroll
    for (int h = 0; h < GW; ++h)   // groups past g re-read group j0 (their sums are not stored)
      Pg[h] = pts + (((size_t)(j0 + h < g ? j0 + h : j0) * b + ib) * nl + L) * N + c0 + lane;
    uint64_t acc[GW][CT][2];
#pragma unroll
    for (int h = 0; h < GW; ++h)
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) acc[h][ct][0] = acc[h][ct][1] = 0;
    for (uint32_t i0 = 0; i0 < bn; i0 += U) {
      uint32_t pv[GW][U];
#pragma unroll
      for (int h = 0; h < GW; ++h) {
        const uint32_t* a = Pg[h] + (size_t)i0 * tstride;
#pragma unroll
        for (int u = 0; u < U; ++u) pv[h][u] = __ldg(a + u * tstride);
      }
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) {
        const uint2* sr = sl + (size_t)(ct * bn + i0) * kSdTile;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint2 xy = sr[u * kSdTile];
#pragma unroll
          for (int h = 0; h < GW; ++h) {
            acc[h][ct][0] += (uint64_t)pv[h][u] * xy.x;
            acc[h][ct][1] += (uint64_t)pv[h][u] * xy.y;
          }
          if ((u & 7) == 7) {   // fold: hi 2^32 + lo == hi (2^32 mod q) + lo  (< 2^62 + 2^32; 8 more fit)
#pragma unroll
            for (int h = 0; h < GW; ++h)
#pragma unroll
              for (int ab = 0; ab < 2; ++ab)
                acc[h][ct][ab] = (uint64_t)(uint32_t)(acc[h][ct][ab] >> 32) * r32 + (uint32_t)acc[h][ct][ab];
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < GW; ++h) {
      if (j0 + h >= g) break;
#pragma unroll
      for (int ct = 0; ct < CT; ++ct)
#pragma unroll
        for (int ab = 0; ab < 2; ++ab) {
          const uint32_t v = barrett64(acc[h][ct][ab], mu, q);
          uint32_t* o = inner + ct * inner_cs + (((size_t)(j0 + h) * nl + L) * 2 + ab) * N + c0 + lane;
          *o = accumulate ? add_mod(v, *o, q) : v;
        }
    }
  }
}
// acc [L][ab][N] = inner_0 + sum_{z < cnt} rot_z
__global__ void k_sd_accumulate(const uint32_t* __restrict__ inner0, const uint32_t* __restrict__ rot, uint32_t cnt,
                                uint32_t N, Mods M, uint32_t* __restrict__ acc) {
  const uint32_t L = blockIdx.y, q = M.m[L];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < 2 * N; x += gridDim.x * blockDim.x) {
    uint32_t v = inner0[(size_t)L * 2 * N + x];
    for (uint32_t z = 0; z < cnt; ++z) v = add_mod(v, rot[(size_t)z * 4 * N + (size_t)L * 2 * N + x], q);
    acc[(size_t)L * 2 * N + x] = v;
  }
}
// signed int64 plaintext polys [count][N] -> [count][2 limbs][N] residues (NTT'd afterwards)
__global__ void k_sd_reduce_pts(const int64_t* __restrict__ pt, uint64_t total, uint32_t logN, uint32_t nl, Mods M,
                                uint32_t* __restrict__ out) {
  const uint32_t N = 1u << logN;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = x >> logN;
    const uint32_t c = (uint32_t)(x & (N - 1));
    const int64_t v = pt[x];
    for (uint32_t L = 0; L < nl; ++L) {
      const int64_t r = v % (int64_t)M.m[L];
      out[(k * nl + L) * N + c] = (uint32_t)(r < 0 ? r + M.m[L] : r);
    }
  }
}
// lazy ModDown (hoisted BSGS; baby rotations from k_sd_mac_lazy_multi):
// baby'_0 = P ct (q0, q1), 0 mod P
__global__ void k_sd_lazy_baby0(const uint32_t* __restrict__ X, uint32_t N, Mods M, uint32_t* __restrict__ out) {
  const uint32_t mod = blockIdx.y, q = M.m[mod];
  const uint64_t mu = M.mu[mod];
  const uint32_t pm = M.m[2] % q;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < 2 * N; c += gridDim.x * blockDim.x)
    out[(size_t)mod * 2 * N + c] = mod < 2 ? mulmod_b(X[(size_t)mod * 2 * N + c], pm, mu, q) : 0u;
}
// ModDown of the g group sums [j][3][ab][N] (P part already inverse-NTT'd): LB [L][j][ab][N] = centred lift
// (4 words per thread, Barrett lift)
__global__ void k_sd_lazy_lift(const uint32_t* __restrict__ X, uint32_t g, uint32_t N, Mods M, uint32_t* __restrict__ LB) {
  const uint32_t P = M.m[2];
  const uint64_t tot4 = 2ull * g * N / 4, n4 = 2ull * N / 4;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < tot4; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = x / n4, r = x % n4;
    const uint4 v = reinterpret_cast<const uint4*>(X + j * 6 * N + 4ull * N)[r];
    const uint32_t vs[4] = {v.x, v.y, v.z, v.w};
    uint32_t l0[4], l1[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t c = vs[e] > P / 2 ? (int64_t)vs[e] - P : (int64_t)vs[e];
      l0[e] = lift_b(c, M.mu[0], M.m[0]);
      l1[e] = lift_b(c, M.mu[1], M.m[1]);
    }
    reinterpret_cast<uint4*>(LB)[x] = make_uint4(l0[0], l0[1], l0[2], l0[3]);
    reinterpret_cast<uint4*>(LB + 2ull * g * N)[x] = make_uint4(l1[0], l1[1], l1[2], l1[3]);
  }
}
// inner_j [L][ab][N] = (X_L - LB_L) P^-1 mod q_L  (NTT domain; Q layout [j][4N] for the giant step)
__global__ void k_sd_lazy_down(const uint32_t* __restrict__ X, const uint32_t* __restrict__ LB, uint32_t g,
                               uint32_t N, Mods M, uint32_t pinv0, uint32_t pinv1, uint32_t* __restrict__ out) {
  const uint32_t L = blockIdx.y, q = M.m[L], pinv = L ? pinv1 : pinv0;
  const uint64_t mu = M.mu[L], tot4 = 2ull * g * N / 4, n4 = 2ull * N / 4;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < tot4; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = x / n4, r = x % n4;
    const uint4 a = reinterpret_cast<const uint4*>(X + j * 6 * N + (uint64_t)L * 2 * N)[r];
    const uint4 l = reinterpret_cast<const uint4*>(LB + (uint64_t)L * 2 * g * N)[x];
    reinterpret_cast<uint4*>(out + j * 4 * N + (uint64_t)L * 2 * N)[r] =
        make_uint4(mulmod_b(sub_mod(a.x, l.x, q), pinv, mu, q), mulmod_b(sub_mod(a.y, l.y, q), pinv, mu, q),
                   mulmod_b(sub_mod(a.z, l.z, q), pinv, mu, q), mulmod_b(sub_mod(a.w, l.w, q), pinv, mu, q));
  }
}

}  // namespace

struct he_slot_pcmm_plan {
  const he_context* ctx;
  uint32_t d, b, g, N, logN;
  const uint32_t* pts;   // caller-owned [d][2][N] NTT domain
  uint32_t* perms;       // owned [b - 1 + g - 1][N]
  Mods M;
  uint32_t qhinv[2], qhinvp[2], pinv[2], q1inv, q1invp;
  uint32_t chunk;        // ciphertexts per shared-plaintext pass (1: per-ct kernels; 2-3: k_sd_inner_s)
  uint32_t shared;       // products through k_sd_inner_s
  uint32_t halves;       // baby range split (shared kernel runs once per half, accumulating)
  uint32_t lazy;         // lazy ModDown: baby rotations kept mod PQ, pts carry 3 moduli, one ModDown per group
  uint32_t plain_giant;  // giant rotations with plain dnum-2 keys (lazy only: their noise lands at Delta q1)
};

// gadget key (layout [t][part][mod][deg], t = i kSdSub + h), NTT domain; streams use t as the digit index
static he_status make_ksk_gadget_dev(const Mods& M, uint64_t seed, uint32_t id, const int32_t* s_old,
                                     const int32_t* s_new, uint32_t deg, const NttTable* tabs, uint32_t* ksk,
                                     cudaStream_t st) {
  uint32_t* snew = nullptr;
  HE_CUDA(cudaMallocAsync(&snew, 3ull * deg * sizeof(uint32_t), st), "alloc");
  for (int j = 0; j < 3; ++j) {
    k_reduce_signed<<<grid_for(deg), 256, 0, st>>>(s_new, deg, M.m[j], snew + (size_t)j * deg);
    HE_CUDA(ntt_forward(tabs[j], snew + (size_t)j * deg, 1, deg, st), "NTT(s_new)");
  }
  for (uint32_t t = 0; t < (uint32_t)kSdT; ++t) {
    const uint32_t i = t / kSdSub, h = t % kSdSub;
    for (uint32_t j = 0; j < 3; ++j) {
      const uint32_t q = M.m[j];
      uint32_t g = 0;
      if (j == i)
        g = (uint32_t)((uint64_t)((uint64_t)(M.m[2] % q) * (M.m[1 - i] % q) % q) * powmod_h(2, (uint64_t)kSdBits * h, q) % q);
      uint32_t* alpha = ksk + ((size_t)(t * 2 + 0) * 3 + j) * deg;
      uint32_t* beta = ksk + ((size_t)(t * 2 + 1) * 3 + j) * deg;
      k_ksk_prep<<<grid_for(deg), 256, 0, st>>>(M.rng, seed, id, t, j, q, g, s_old, deg, alpha, beta);
      HE_CUDA(ntt_forward(tabs[j], alpha, 1, deg, st), "NTT(alpha)");
      HE_CUDA(ntt_forward(tabs[j], beta, 1, deg, st), "NTT(t)");
      k_ksk_beta<<<grid_for(deg), 256, 0, st>>>(alpha, snew + (size_t)j * deg, deg, q, beta);
    }
  }
  cudaFreeAsync(snew, st);
  return HE_OK;
}

extern "C" he_status he_slot_rotation_keygen(const he_context* c, uint64_t seed, const int32_t* s_dev,
                                             const int32_t* steps, uint32_t n_steps, uint32_t* keys_dev,
                                             void* stream) {
  if (!c || !s_dev || !steps || (!keys_dev && n_steps)) return fail(HE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N;
  const Mods M = make_mods(c->R);
  int32_t* sk = nullptr;
  HE_CUDA(cudaMallocAsync(&sk, N * sizeof(int32_t), st), "alloc");
  he_status s = HE_OK;
  for (uint32_t t = 0; t < n_steps && !s; ++t) {
    const uint32_t r = (uint32_t)(((int64_t)steps[t] % (N / 2) + N / 2) % (N / 2));
    const uint32_t g = (uint32_t)powmod_h(5, r, 2ull * N);
    k_secret_auto<<<grid_for(N), 256, 0, st>>>(s_dev, N, g, sk);
    s = make_ksk_gadget_dev(M, seed, 0x10000 + r, sk, s_dev, N, c->ntt, keys_dev + (size_t)t * 24 * N, st);
  }
  cudaFreeAsync(sk, st);
  if (s) return s;
  return cudaGetLastError() == cudaSuccess ? HE_OK : fail(HE_ECUDA, "rotation keygen launch failed");
}

// plain dnum-2 rotation keys sigma_{5^r}(s) -> s ([n][2][2][3][N], NTT), for the giant steps of lazy plans
extern "C" he_status he_slot_rotation_keygen_plain(const he_context* c, uint64_t seed, const int32_t* s_dev,
                                                   const int32_t* steps, uint32_t n_steps, uint32_t* keys_dev,
                                                   void* stream) {
  if (!c || !s_dev || !steps || (!keys_dev && n_steps)) return fail(HE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N;
  const Mods M = make_mods(c->R);
  int32_t* sk = nullptr;
  HE_CUDA(cudaMallocAsync(&sk, N * sizeof(int32_t), st), "alloc");
  he_status s = HE_OK;
  for (uint32_t t = 0; t < n_steps && !s; ++t) {
    const uint32_t r = (uint32_t)(((int64_t)steps[t] % (N / 2) + N / 2) % (N / 2));
    const uint32_t g = (uint32_t)powmod_h(5, r, 2ull * N);
    k_secret_auto<<<grid_for(N), 256, 0, st>>>(s_dev, N, g, sk);
    s = make_ksk_dev(M, seed, 0x30000 + r, sk, s_dev, N, c->ntt, keys_dev + (size_t)t * 12 * N, st);
  }
  cudaFreeAsync(sk, st);
  if (s) return s;
  return cudaGetLastError() == cudaSuccess ? HE_OK : fail(HE_ECUDA, "rotation keygen launch failed");
}

extern "C" he_status he_slot_pcmm_encode_pts(const he_context* c, const int64_t* pt_dev, uint32_t count,
                                             uint32_t* pts_ntt_dev, void* stream) {
  if (!c || !pt_dev || !pts_ntt_dev) return fail(HE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N;
  const Mods M = make_mods(c->R);
  k_sd_reduce_pts<<<grid_for((uint64_t)count * N), 256, 0, st>>>(pt_dev, (uint64_t)count * N, (uint32_t)ilog2_u(N), 2u,
                                                                   M, pts_ntt_dev);
  for (int L = 0; L < 2; ++L)
    HE_CUDA(ntt_forward(c->ntt[L], pts_ntt_dev + (size_t)L * N, count, 2ull * N, st), "NTT(pt)");
  return HE_OK;
}

extern "C" he_status he_slot_pcmm_encode_pts_ext(const he_context* c, const int64_t* pt_dev, uint32_t count,
                                                 uint32_t n_mods, uint32_t* pts_ntt_dev, void* stream) {
  if (!c || !pt_dev || !pts_ntt_dev) return fail(HE_EINVAL, "null argument");
  if (n_mods != 2 && n_mods != 3) return fail(HE_EINVAL, "n_mods must be 2 (q0, q1) or 3 (q0, q1, P)");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N;
  const Mods M = make_mods(c->R);
  k_sd_reduce_pts<<<grid_for((uint64_t)count * N), 256, 0, st>>>(pt_dev, (uint64_t)count * N, (uint32_t)ilog2_u(N),
                                                                   n_mods, M, pts_ntt_dev);
  for (uint32_t L = 0; L < n_mods; ++L)
    HE_CUDA(ntt_forward(c->ntt[L], pts_ntt_dev + (size_t)L * N, count, (uint64_t)n_mods * N, st), "NTT(pt)");
  return HE_OK;
}

// plan over rotation steps: steps[t] for the b - 1 baby and g - 1 giant rotations, in run order
static he_status slot_plan_make(const he_context* c, const uint32_t* pts_ntt_dev, uint32_t d, uint32_t b, uint32_t g,
                                const std::vector<uint64_t>& steps, he_slot_pcmm_plan** out) {
  const uint32_t N = c->R.N;
  he_slot_pcmm_plan* p = new (std::nothrow) he_slot_pcmm_plan();
  if (!p) return fail(HE_ENOMEM, "out of host memory");
  p->ctx = c;
  p->d = d;
  p->b = b;
  p->g = g;
  p->N = N;
  p->logN = (uint32_t)ilog2_u(N);
  p->pts = pts_ntt_dev;
  p->M = make_mods(c->R);
  for (int i = 0; i < 2; ++i) {
    const uint32_t qi = p->M.m[i];
    p->qhinv[i] = (uint32_t)powmod_h(p->M.m[1 - i] % qi, qi - 2, qi);
    p->qhinvp[i] = shoup_pre(p->qhinv[i], qi);
    p->pinv[i] = (uint32_t)powmod_h(p->M.m[2] % qi, qi - 2, qi);
  }
  p->q1inv = (uint32_t)powmod_h(p->M.m[1] % p->M.m[0], p->M.m[0] - 2, p->M.m[0]);
  p->q1invp = shoup_pre(p->q1inv, p->M.m[0]);
  // big maps stream their plaintexts once per up-to-3 ciphertexts (shared-memory baby tiles, CT b 256 B)
  p->chunk = 1;
  p->shared = 0;
  p->lazy = 0;
  p->plain_giant = 0;
  p->halves = 1;
  const bool shared_ok = b % 16 == 0 && N % kSdTile == 0 && p->M.m[0] < (1u << 30) && p->M.m[1] < (1u << 30);
  if (((uint64_t)b * g >= 4096 || getenv("HE_SD_SHARED")) && shared_ok && !getenv("HE_SD_PER_CT")) {
    // ciphertexts per plaintext read: as many (<= 6) as fit 200 KB of baby tiles.  HE_SD_HALVES=2 splits the
    // baby range into two accumulating passes (6 instead of 3 cts at b = 256): measured no faster -- the
    // products are issue-bound at 3 (StC: 3.1 vs 3.2 ms/ct), so it stays opt-in
    const int env_halves = getenv("HE_SD_HALVES") ? atoi(getenv("HE_SD_HALVES")) : 0;
    const uint32_t tile = 2 * kSdTile * 4;   // bytes per baby term per ct
    auto fit = [&](uint32_t h) { return std::min<uint32_t>(6, (200u * 1024) / (b / h * tile)); };
    const uint32_t h = (env_halves == 2 && b % 32 == 0) ? 2 : 1;
    if (fit(h) >= 2) {
      p->chunk = fit(h);
      p->halves = h;
      p->shared = 1;
    }
  }
  std::vector<uint32_t> h((size_t)(steps.empty() ? 1 : steps.size()) * N);
  for (size_t t = 0; t < steps.size(); ++t) {
    const uint64_t gal = powmod_h(5, steps[t] % (N / 2), 2ull * N);
    for (uint32_t cc = 0; cc < N; ++cc) {
      const uint64_t e = 2ull * bitrev_h(cc, (int)p->logN) + 1;
      h[t * N + cc] = bitrev_h((uint32_t)(((e * gal) % (2ull * N) - 1) / 2), (int)p->logN);
    }
  }
  if (cudaMalloc(&p->perms, h.size() * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemcpy(p->perms, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    delete p;
    return fail(HE_ECUDA, "slot pcmm tables");
  }
  *out = p;
  return HE_OK;
}

extern "C" he_status he_slot_pcmm_plan_create(const he_context* c, const uint32_t* pts_ntt_dev, uint32_t d, uint32_t b,
                                              uint32_t g, he_slot_pcmm_plan** out) {
  if (!c || !pts_ntt_dev || !out) return fail(HE_EINVAL, "null argument");
  if (d == 0 || b == 0 || g == 0 || b * g != d) return fail(HE_EINVAL, "split %ux%u does not cover dim %u", b, g, d);
  const uint32_t N = c->R.N;
  if ((uint64_t)d * d > N / 2 || (N / 2) % (d * d))
    return fail(HE_EINVAL, "%ux%u does not tile the %u slots (d^2 must divide N/2)", d, d, N / 2);
  std::vector<uint64_t> steps;
  for (uint32_t i = 1; i < b; ++i) steps.push_back((uint64_t)i * d);
  for (uint32_t j = 1; j < g; ++j) steps.push_back((uint64_t)j * b * d);
  return slot_plan_make(c, pts_ntt_dev, d, b, g, steps, out);
}

// general slot linear map out = rescale(sum_t pt_t * rot(ct, steps[t])), steps[0] = 0 (hesim pc_linear over
// rotated copies, slotsim.py:330-370; e.g. rope_packed, pipeline.py:291-307): the BSGS run with g = 1
extern "C" he_status he_slot_lt_plan_create(const he_context* c, const uint32_t* pts_ntt_dev, uint32_t n_terms,
                                            const int32_t* steps, he_slot_pcmm_plan** out) {
  if (!c || !pts_ntt_dev || !steps || !out) return fail(HE_EINVAL, "null argument");
  if (n_terms == 0 || steps[0] != 0) return fail(HE_EINVAL, "need >= 1 term and steps[0] == 0");
  const int64_t half = c->R.N / 2;
  std::vector<uint64_t> st;
  for (uint32_t t = 1; t < n_terms; ++t) st.push_back((uint64_t)((steps[t] % half + half) % half));
  return slot_plan_make(c, pts_ntt_dev, n_terms, n_terms, 1, st, out);
}

// general BSGS slot linear map over n = b g diagonals: baby steps i * stride (i < b), giant steps j * b * stride
// (j < g); pts in kernel order i + j b, each already rotated by -j b stride (e.g. SlotToCoeffs: stride 1, n = N/2)
extern "C" he_status he_slot_bsgs_plan_create(const he_context* c, const uint32_t* pts_ntt_dev, uint32_t b, uint32_t g,
                                              uint32_t stride, he_slot_pcmm_plan** out) {
  if (!c || !pts_ntt_dev || !out) return fail(HE_EINVAL, "null argument");
  const uint64_t half = c->R.N / 2;
  if (b == 0 || g == 0 || stride == 0 || (uint64_t)b * g * stride > half)
    return fail(HE_EINVAL, "split %ux%u with stride %u exceeds the %llu slots", b, g, stride, (unsigned long long)half);
  std::vector<uint64_t> steps;
  for (uint32_t i = 1; i < b; ++i) steps.push_back((uint64_t)i * stride);
  for (uint32_t j = 1; j < g; ++j) steps.push_back((uint64_t)j * b * stride);
  return slot_plan_make(c, pts_ntt_dev, b * g, b, g, steps, out);
}

extern "C" he_status he_slot_bsgs_plan_create_ext(const he_context* c, const uint32_t* pts_ntt_dev, uint32_t b,
                                                  uint32_t g, uint32_t stride, uint32_t flags, he_slot_pcmm_plan** out) {
  if (flags & ~(HE_SLOT_LAZY_MODDOWN | HE_SLOT_PLAIN_GIANT)) return fail(HE_EINVAL, "unknown slot plan flags 0x%x", flags);
  if ((flags & HE_SLOT_PLAIN_GIANT) && !(flags & HE_SLOT_LAZY_MODDOWN))
    return fail(HE_EINVAL, "HE_SLOT_PLAIN_GIANT needs HE_SLOT_LAZY_MODDOWN (eager plans take gadget giant keys)");
  if (!(flags & HE_SLOT_LAZY_MODDOWN)) return he_slot_bsgs_plan_create(c, pts_ntt_dev, b, g, stride, out);
  if (!c || !out) return fail(HE_EINVAL, "null argument");
  const Mods M = make_mods(c->R);
  if (b % 8 || c->R.N % kSdTile || (uint64_t)b * 2 * kSdTile * 4 > 200 * 1024 || M.m[0] >= (1u << 30) ||
      M.m[1] >= (1u << 30) || M.m[2] >= (1u << 30))
    return fail(HE_EINVAL, "lazy ModDown needs b %% 8 == 0, b <= 800 and 30-bit moduli (b = %u)", b);
  he_status s = he_slot_bsgs_plan_create(c, pts_ntt_dev, b, g, stride, out);
  if (s) return s;
  (*out)->lazy = 1;
  (*out)->shared = 1;
  (*out)->plain_giant = (flags & HE_SLOT_PLAIN_GIANT) ? 1u : 0u;
  return HE_OK;
}

extern "C" he_status he_slot_pcmm_plan_destroy(he_slot_pcmm_plan* p) {
  if (p) {
    if (p->perms) cudaFree(p->perms);
    delete p;
  }
  return HE_OK;
}

struct SdWs {
  uint32_t *D, *X, *baby, *inner, *innerq, *rot, *acc, *UW, *LB;
};
static uint64_t sd_ws_words(const he_slot_pcmm_plan* p, SdWs* w, uint32_t* base) {
  const uint64_t N = p->N, T = (p->b > p->g ? p->b : p->g), C = p->chunk;   // rotations per batched pass < T
  uint64_t off = 0;
  auto take = [&](uint32_t*& ptr, uint64_t words) {
    if (w) ptr = base + off;
    off += (words + 63) & ~63ull;
  };
  SdWs dummy;
  SdWs& r = w ? *w : dummy;
  take(r.D, 3ull * kSdT * T * N);
  take(r.X, 4 * N * C);
  const uint64_t cw = p->lazy ? 6 : 4;   // words per N of a baby / group ct (3 moduli when lazy)
  take(r.baby, cw * p->b * N * C);
  take(r.inner, cw * p->g * N * C);
  take(r.innerq, p->lazy ? 4ull * p->g * N : 0);
  take(r.rot, 4ull * T * N);
  take(r.acc, 4 * N);
  take(r.UW, 6ull * T * N);
  take(r.LB, 4ull * T * N);
  return off;
}

extern "C" he_status he_slot_pcmm_workspace_bytes(const he_slot_pcmm_plan* p, uint64_t* bytes) {
  if (!p || !bytes) return fail(HE_EINVAL, "null argument");
  *bytes = sd_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  return HE_OK;
}

template <int CT, int U, int GW = 2>
static cudaError_t launch_sd_inner_s_cu(const uint32_t* baby, uint64_t baby_cs, const uint32_t* pts, uint32_t b,
                                        uint32_t g, uint32_t N, uint32_t nl, const Mods& M, uint32_t* inner,
                                        uint64_t inner_cs, uint32_t halves, cudaStream_t st) {
  const uint32_t bn = b / halves;
  const int smem = CT * (int)bn * 2 * kSdTile * 4;
  cudaError_t e = cudaFuncSetAttribute(k_sd_inner_s<CT, U, GW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  for (uint32_t h = 0; h < halves; ++h)
    k_sd_inner_s<CT, U, GW><<<dim3(N / kSdTile, nl), kSdSharedThreads, smem, st>>>(baby, baby_cs, pts, b, g, N, nl,
                                                                                   M, inner, inner_cs, h * bn, bn,
                                                                                   h > 0);
  return cudaGetLastError();
}
// U = plaintext terms loaded ahead per group (register budget: 2 U words + 4 CT sums); must divide the range
template <int CT>
static cudaError_t launch_sd_inner_s_ct(const uint32_t* baby, uint64_t baby_cs, const uint32_t* pts, uint32_t b,
                                        uint32_t g, uint32_t N, uint32_t nl, const Mods& M, uint32_t* inner,
                                        uint64_t inner_cs, uint32_t halves, cudaStream_t st) {
  const uint32_t bn = b / halves;
  if (CT <= 2 && bn % 16 == 0)   // 128-register cap at 512 threads: 16 ahead fits two ciphertexts' sums
    return launch_sd_inner_s_cu<CT, (CT <= 2 ? 16 : 8)>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
  // (4 groups per warp: 288 B of spills at 3 cts under the 128-register cap -- not used)
  return launch_sd_inner_s_cu<CT, 8>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
}
static cudaError_t launch_sd_inner_s(uint32_t cc, const uint32_t* baby, uint64_t baby_cs, const uint32_t* pts,
                                     uint32_t b, uint32_t g, uint32_t N, uint32_t nl, const Mods& M, uint32_t* inner,
                                     uint64_t inner_cs, uint32_t halves, cudaStream_t st) {
  switch (cc) {
    case 6: return launch_sd_inner_s_ct<6>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
    case 5: return launch_sd_inner_s_ct<5>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
    case 4: return launch_sd_inner_s_ct<4>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
    case 3: return launch_sd_inner_s_ct<3>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
    case 2: return launch_sd_inner_s_ct<2>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
    default: return launch_sd_inner_s_ct<1>(baby, baby_cs, pts, b, g, N, nl, M, inner, inner_cs, halves, st);
  }
}

// n_ct ciphertexts [n_ct][2][2][N] level 1 -> out [n_ct][2][N] level 0, in chunks of p->chunk sharing each
// plaintext read
static he_status sd_run(const he_slot_pcmm_plan* p, const uint32_t* ct_in, uint32_t n_ct, const uint32_t* keys_baby,
                        const uint32_t* keys_giant, uint32_t* out, void* ws_dev, cudaStream_t st) {
  const he_context* c = p->ctx;
  const uint32_t N = p->N, b = p->b, g = p->g;
  SdWs w;
  sd_ws_words(p, &w, (uint32_t*)ws_dev);
  const dim3 g1 = grid_for(N);
  auto grid3 = [&](uint32_t y, uint32_t z) {
    dim3 gg = g1;
    gg.y = y;
    gg.z = z;
    return gg;
  };
  // digits of cnt sources (a-part of source z at a + z * as) -> D^ [mod][z][t][N] (NTT)
  auto digits = [&](const uint32_t* a, uint64_t as, uint32_t cnt) -> he_status {
    k_sd_digits<<<grid3(1, cnt), 256, 0, st>>>(a, as, 2ull * N, N, cnt, p->M, p->qhinv[0], p->qhinvp[0], p->qhinv[1],
                                               p->qhinvp[1], w.D);
    const uint64_t ms = (uint64_t)cnt * kSdT * N;
    HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1], &c->ntt[2]}, {w.D, w.D + ms, w.D + 2 * ms}, cnt * kSdT, N, st), "NTT(D)");
    return HE_OK;
  };
  // cnt rotations in one pass: rotation z uses perm table t0 + z, key z, digits dz (hoist: all z share D^ 0),
  // source b^ at bh + z * bs; result z at dst + z * 4N (NTT domain)
  // plain digits (dnum-2 keys) of cnt sources -> D^ [mod][z][i < 2][N] (NTT)
  auto digits_plain = [&](const uint32_t* a, uint64_t as, uint32_t cnt) -> he_status {
    k_sd_digits_plain<<<grid3(1, cnt), 256, 0, st>>>(a, as, 2ull * N, N, cnt, p->M, p->qhinv[0], p->qhinvp[0],
                                                     p->qhinv[1], p->qhinvp[1], w.D);
    const uint64_t ms = (uint64_t)cnt * 2 * N;
    HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1], &c->ntt[2]}, {w.D, w.D + ms, w.D + 2 * ms}, cnt * 2, N, st), "NTT(D plain)");
    return HE_OK;
  };
  auto rotate = [&](uint32_t cnt, int hoist, uint32_t dcnt, uint32_t t0, const uint32_t* keys, const uint32_t* bh,
                    uint64_t bs, uint32_t* dst, bool plain = false) -> he_status {
    if (plain)
      k_sd_mac_t<2><<<grid3(3, cnt), 256, 0, st>>>(w.D, dcnt, hoist, p->perms + (size_t)t0 * N, keys, N, cnt, p->M,
                                                   w.UW);
    else
      k_sd_mac_t<kSdT><<<grid3(3, cnt), 256, 0, st>>>(w.D, dcnt, hoist, p->perms + (size_t)t0 * N, keys, N, cnt,
                                                      p->M, w.UW);
    uint32_t* UWP = w.UW + (size_t)2 * cnt * 2 * N;   // [z][part][N] of modulus P
    HE_CUDA(ntt_inverse(c->ntt[2], UWP, 2 * cnt, N, st), "INTT(U_P, W_P)");
    k_moddown_lift<<<grid_for(2ull * cnt * N), 256, 0, st>>>(UWP, (uint64_t)cnt * N, p->M, w.LB);
    HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1]}, {w.LB, w.LB + 2ull * cnt * N}, 2 * cnt, N, st), "NTT(lift)");
    k_sd_combine<<<grid3(2, cnt), 256, 0, st>>>(w.UW, w.LB, bh, bs, 2ull * N, p->perms + (size_t)t0 * N, N, cnt, p->M,
                                               p->pinv[0], p->pinv[1], dst, 4ull * N);
    return HE_OK;
  };
  static const bool inner_simple = getenv("HE_SD_INNER_SIMPLE") != nullptr;
  const uint32_t nl = p->lazy ? 3 : 2;   // moduli the products run over
  const uint64_t baby_cs = 2ull * nl * b * N, inner_cs = 2ull * nl * g * N;
  for (uint32_t c0 = 0; c0 < n_ct; c0 += p->chunk) {
    const uint32_t cc = std::min(p->chunk, n_ct - c0);
    if (p->lazy) {
      // baby steps of all cc ciphertexts together: digits and NTT'd copies of each, P ct, then one key MAC
      // pass per rotation serving every ciphertext (PQ basis, no ModDown): [ct][i][3 moduli][ab][N]
      he_status s = digits(ct_in + (size_t)c0 * 4 * N, 4ull * N, cc);
      if (s) return s;
      HE_CUDA(cudaMemcpyAsync(w.X, ct_in + (size_t)c0 * 4 * N, 4ull * N * cc * sizeof(uint32_t),
                              cudaMemcpyDeviceToDevice, st), "copy");
      for (uint32_t z = 0; z < cc; ++z) {
        HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1]}, {w.X + (size_t)z * 4 * N, w.X + (size_t)z * 4 * N + 2ull * N}, 2,
                         N, st), "NTT(ct)");
        k_sd_lazy_baby0<<<grid3(3, 1), 256, 0, st>>>(w.X + (size_t)z * 4 * N, N, p->M, w.baby + z * baby_cs);
      }
      if (b > 1)
        k_sd_mac_lazy_multi<<<grid3(3, b - 1), 256, 0, st>>>(w.D, cc, p->perms, keys_baby, w.X, N, p->M,
                                                              w.baby + 6ull * N, baby_cs);
    }
    // baby steps per ciphertext: one hoisted digit decomposition, all b - 1 rotations in one pass
    for (uint32_t z = 0; z < cc && !p->lazy; ++z) {
      const uint32_t* ct = ct_in + (size_t)(c0 + z) * 4 * N;
      uint32_t* bz = w.baby + z * baby_cs;
      he_status s = digits(ct, 0, 1);
      if (s) return s;
      HE_CUDA(cudaMemcpyAsync(w.X, ct, 4ull * N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "copy");
      HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1]}, {w.X, w.X + 2ull * N}, 2, N, st), "NTT(ct)");
      HE_CUDA(cudaMemcpyAsync(bz, w.X, 4ull * N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "copy");
      if (b > 1) {
        s = rotate(b - 1, 1, 1, 0, keys_baby, w.X + N, 0, bz + 4ull * N);
        if (s) return s;
      }
    }
    // giant-group products: all groups (and all cc ciphertexts) in one launch
    if (p->shared) {
      cudaError_t e =
          launch_sd_inner_s(cc, w.baby, baby_cs, p->pts, b, g, N, nl, p->M, w.inner, inner_cs, p->halves, st);
      HE_CUDA(e, "slot map products (shared)");
    } else if (g >= 8 && !inner_simple) {
      dim3 gi = grid_for(N / 2);
      gi.y = 2;
      gi.z = (g + 7) / 8;
      k_sd_inner_g<8><<<gi, 256, 0, st>>>(w.baby, p->pts, b, g, N, p->M, w.inner);
    } else {
      k_sd_inner<<<grid3(2, g), 256, 0, st>>>(w.baby, p->pts, b, N, p->M, w.inner);
    }
    // giant rotations per ciphertext (one pass each), sum, one rescale
    for (uint32_t z = 0; z < cc; ++z) {
      uint32_t* iz = w.inner + z * inner_cs;
      if (p->lazy) {
        // one ModDown per group sum: INTT of the P parts, centred lift, NTT, (X - lift) P^-1 -> [j][4N]
        HE_CUDA(ntt_jobs(true, {&c->ntt[2], &c->ntt[2]}, {iz + 4ull * N, iz + 5ull * N}, g, 6ull * N, st),
                "INTT(group sums, P)");
        dim3 gl = grid_for(2ull * g * N / 4);
        k_sd_lazy_lift<<<gl, 256, 0, st>>>(iz, g, N, p->M, w.LB);
        gl.y = 2;
        HE_CUDA(ntt_jobs(false, {&c->ntt[0], &c->ntt[1]}, {w.LB, w.LB + 2ull * g * N}, 2 * g, N, st), "NTT(lift)");
        k_sd_lazy_down<<<gl, 256, 0, st>>>(iz, w.LB, g, N, p->M, p->pinv[0], p->pinv[1], w.innerq);
        iz = w.innerq;
      }
      if (g > 1) {
        uint32_t* in1 = iz + 4ull * N;   // groups 1 .. g-1
        HE_CUDA(ntt_jobs(true, {&c->ntt[0], &c->ntt[1]}, {in1, in1 + 2ull * N}, g - 1, 4ull * N, st), "INTT(inner a)");
        he_status s = p->plain_giant ? digits_plain(in1, 4ull * N, g - 1) : digits(in1, 4ull * N, g - 1);
        if (s) return s;
        s = rotate(g - 1, 0, g - 1, b - 1, keys_giant, in1 + N, 4ull * N, w.rot, p->plain_giant != 0);
        if (s) return s;
      }
      k_sd_accumulate<<<grid3(2, 1), 256, 0, st>>>(iz, w.rot, g - 1, N, p->M, w.acc);
      HE_CUDA(ntt_jobs(true, {&c->ntt[0], &c->ntt[1]}, {w.acc, w.acc + 2ull * N}, 2, N, st), "INTT(acc)");
      k_rh_combine<<<grid_for(2ull * N), 256, 0, st>>>(w.acc, 1, N, p->M.m[0], p->M.m[1], p->q1inv, p->q1invp,
                                                       out + (size_t)(c0 + z) * 2 * N);
    }
  }
  HE_CUDA(cudaGetLastError(), "slot pcmm launch");
  return HE_OK;
}

static he_status sd_run_checked(const he_slot_pcmm_plan* p, const uint32_t* ct_in, uint32_t n_ct, uint32_t level,
                                const uint32_t* keys_baby, const uint32_t* keys_giant, uint32_t* out, void* ws_dev,
                                uint64_t ws_bytes, void* stream, he_ledger* ledger) {
  if (!p) return fail(HE_EINVAL, "null plan");
  if (level < 1) return fail(HE_ENEEDS_BOOTSTRAP, "pcmm needs one level");
  if (level != 1) return fail(HE_EINVAL, "the slot-domain PCMM runs at level 1 (got %u)", level);
  if (!ct_in || !out || !ws_dev || (p->b > 1 && !keys_baby) || (p->g > 1 && !keys_giant))
    return fail(HE_EINVAL, "null argument");
  if (ws_bytes < sd_ws_words(p, nullptr, nullptr) * sizeof(uint32_t)) return fail(HE_EINVAL, "workspace too small");
  he_status s = sd_run(p, ct_in, n_ct, keys_baby, keys_giant, out, ws_dev, (cudaStream_t)stream);
  if (s) return s;
  if (ledger) {
    ledger->ct_rotations += (int64_t)n_ct * ((p->b - 1) + (p->g - 1));
    ledger->pc_mults += (int64_t)n_ct * p->d;
    ledger->rescales += n_ct;
  }
  return HE_OK;
}

extern "C" he_status he_slot_pcmm_run(const he_slot_pcmm_plan* p, const uint32_t* ct_in, uint32_t level,
                                      const uint32_t* keys_baby, const uint32_t* keys_giant, uint32_t* out, void* ws_dev,
                                      uint64_t ws_bytes, void* stream, he_ledger* ledger) {
  return sd_run_checked(p, ct_in, 1, level, keys_baby, keys_giant, out, ws_dev, ws_bytes, stream, ledger);
}

extern "C" he_status he_slot_pcmm_run_batch(const he_slot_pcmm_plan* p, const uint32_t* ct_in, uint32_t n_ct,
                                            uint32_t level, const uint32_t* keys_baby, const uint32_t* keys_giant,
                                            uint32_t* out, void* ws_dev, uint64_t ws_bytes, void* stream,
                                            he_ledger* ledger) {
  if (n_ct == 0) return fail(HE_EINVAL, "empty batch");
  return sd_run_checked(p, ct_in, n_ct, level, keys_baby, keys_giant, out, ws_dev, ws_bytes, stream, ledger);
}
