// he_chain.cu -- the modulus chain above the PCMM's level 1: ciphertexts at any level l of q_0 .. q_l
// (+ the special prime P), encryption there, rotation keys, and BSGS slot linear maps that consume one
// level each -- the machinery of the level-lowered, Cooley-Tukey-factorized SlotToCoeffs the paper
// runs before its PCMv / PCMM inputs ("lower the total level to 4; SlotToCoeffs to level 1",
// PAPER.md:58-60; StC as a homomorphic DFT).  Restated from oracle/he_oracle_chain.c
// (same integer algorithm, bit-exact):
//   key switching: hybrid, dnum = l + 1 one-prime digits d_i = [c_i (Q/q_i)^-1]_{q_i}, lifted to every
//                  modulus, MAC with the key in the NTT domain, ModDown by P with a centred P part;
//   rotation by r: X -> X^(5^r) as an NTT-domain index permutation of the hoisted lifted digits and of b;
//   BSGS map:      out = rescale(sum_j rot_{(j b - T) s}(sum_i pt_{i + j b} * rot_{i s}(ct))), the rescale
//                  dropping q_l with a centred top limb.
// Every step is batched over the rotations of one map (grid z), and the whole map runs on the device.
#include <algorithm>
#include <vector>

#include "he_common.cuh"
#include "he_internal.h"
#include "he_kernels.h"

using namespace he;

namespace {

constexpr int kChMaxQ = 8;  // data primes + P

struct ChMods {  // the moduli of one level: m[0 .. nq) data primes, m[nq] = P
  uint32_t m[kChMaxQ];
  uint64_t mu[kChMaxQ];
  uint32_t nq;
};
HE_D uint32_t ch_barrett(uint64_t x, uint64_t mu, uint32_t q) {
  const uint64_t qh = __umul64hi(x, mu);
  return csub((uint32_t)(x - qh * q), q);
}
HE_D uint32_t ch_mulmod(uint32_t a, uint32_t b, uint64_t mu, uint32_t q) { return ch_barrett((uint64_t)a * b, mu, q); }

inline dim3 ch_grid(uint64_t work, int threads = 256) {
  uint64_t b = (work + threads - 1) / threads;
  if (b > 148ull * 32) b = 148ull * 32;
  if (b == 0) b = 1;
  return dim3((unsigned)b);
}

// ---------------------------------------------------------------- encryption (oracle or_encrypt, any limb count)
__global__ void k_ch_gen_a(RngCtx rc, uint64_t seed, uint32_t r0, uint32_t N, ChMods M, uint32_t* ct) {
  const uint32_t r = blockIdx.y, L = blockIdx.z, nq = M.nq;
  const Rng key = rng_make(rc, seed, stream_a(r0 + r, L));
  uint32_t* a = ct + ((size_t)r * nq + L) * 2 * N;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)(rng_next(key, i) % M.m[L]);
    a[i] = v;
    a[N + i] = v;
  }
}
__global__ void k_ch_reduce_secret(const int32_t* s, uint32_t N, ChMods M, uint32_t cnt, uint32_t* out) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < cnt * N; x += gridDim.x * blockDim.x) {
    const uint32_t j = x / N, i = x % N;
    const int32_t v = s[i];
    out[x] = v < 0 ? M.m[j] + v : (uint32_t)v;
  }
}
// b slot holds NTT(a) on entry; b <- NTT(a) * NTT(s) (in place)
__global__ void k_ch_mul_s(uint32_t* ct, uint32_t n_ct, uint32_t N, ChMods M, const uint32_t* s_ntt) {
  const uint32_t nq = M.nq;
  const uint64_t tot = (uint64_t)n_ct * nq * N;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < tot; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(x % N), L = (uint32_t)((x / N) % nq);
    const uint64_t r = x / ((uint64_t)N * nq);
    uint32_t* b = ct + ((r * nq + L) * 2 + 1) * N;
    b[c] = ch_mulmod(b[c], s_ntt[(size_t)L * N + c], M.mu[L], M.m[L]);
  }
}
// b = pt + e - a s  (b holds a s in coefficient form on entry)
__global__ void k_ch_finish(RngCtx rc, const int64_t* __restrict__ pt, uint64_t seed, uint32_t r0, uint32_t N, ChMods M,
                            uint32_t* ct) {
  const uint32_t r = blockIdx.y, nq = M.nq;
  const Rng ekey = rng_make(rc, seed, stream_e(r0 + r));
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    const long long p = pt[(size_t)r * N + c];
    const long long e = cbd21_d(rng_next(ekey, c));
    for (uint32_t L = 0; L < nq; ++L) {
      const uint32_t q = M.m[L];
      uint32_t* b = ct + ((size_t)r * nq + L) * 2 * N + N;
      const uint64_t v = (uint64_t)from_i64(p, q) + from_i64(e, q) + (q - b[c]);
      b[c] = (uint32_t)(v % q);
    }
  }
}

// ---------------------------------------------------------------- key generation
__global__ void k_ch_secret_auto(const int32_t* s, uint32_t N, uint64_t g, int32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const uint64_t j = ((uint64_t)i * g) % (2ull * N);
    if (j < N) out[j] = s[i];
    else out[j - N] = -s[i];
  }
}
// alpha (uniform) and t = g s_old + e (coefficient form, modulus q)
__global__ void k_ch_ksk_prep(RngCtx rc, uint64_t seed, uint32_t id, uint32_t i, uint32_t j, uint32_t q, uint32_t g,
                              const int32_t* s_old, uint32_t n, uint32_t* alpha, uint32_t* t) {
  const Rng ka = rng_make(rc, seed, 0xC000000000000000ULL | ((uint64_t)id << 16) | ((uint64_t)i << 8) | j);
  const Rng ke = rng_make(rc, seed, 0xCE00000000000000ULL | ((uint64_t)id << 16) | ((uint64_t)i << 8));
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    alpha[c] = (uint32_t)(rng_next(ka, c) % q);
    const int64_t e = cbd21_d(rng_next(ke, c));
    const uint64_t gs = (uint64_t)g * from_i64(s_old[c], q) % q;
    t[c] = (uint32_t)((gs + from_i64(e, q)) % q);
  }
}
__global__ void k_ch_ksk_beta(const uint32_t* alpha, const uint32_t* s_new, uint32_t n, uint32_t q, uint32_t* t) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
    t[c] = sub_mod(t[c], mul_mod(alpha[c], s_new[c], q), q);
}

// ---------------------------------------------------------------- key switching (batched over rotations z)
// A batch of key switches over the ciphertexts of a chunk: rotation z reads the digits of source src(z),
// applies the automorphism of rotation rot(z) and combines with the b part of block blk(z):
//   hoisted baby steps (giant = 0):  src = blk = z / per (the ct), rot = z % per (baby step index)
//   giant groups     (giant = 1):  src = z, blk = (z / per) g + gidx[z % per], rot = gidx[z % per]
struct RotMap {
  uint32_t per, giant, g;
  uint8_t gidx[64];
};
HE_D uint32_t rm_src(const RotMap& m, uint32_t z) { return m.giant ? z : z / m.per; }
HE_D uint32_t rm_rot(const RotMap& m, uint32_t z) { return m.giant ? m.gidx[z % m.per] : z % m.per; }
HE_D uint32_t rm_blk(const RotMap& m, uint32_t z) { return m.giant ? (z / m.per) * m.g + m.gidx[z % m.per] : z / m.per; }

// lifted digits of the a parts of cnt sources (coefficient form; source z = block blk(z) of the a buffer,
// limb L at + L ls):  D [j < nq+1][z][i < nq][N] = d_i mod m_j,  d_i = a_i qhinv_i mod m_i
__global__ void k_ch_digits(const uint32_t* __restrict__ a, uint64_t as, uint64_t ls, uint32_t N, uint32_t cnt, ChMods M,
                            const uint32_t* qhinv, RotMap rm, int mapped, uint32_t* __restrict__ D) {
  const uint32_t z = blockIdx.y, nq = M.nq;
  const uint32_t* src = a + (size_t)(mapped ? rm_blk(rm, z) : z) * as;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < N; x += gridDim.x * blockDim.x) {
    for (uint32_t i = 0; i < nq; ++i) {
      const uint32_t d = ch_mulmod(src[(size_t)i * ls + x], qhinv[i], M.mu[i], M.m[i]);
      for (uint32_t j = 0; j <= nq; ++j)
        D[(((size_t)j * cnt + z) * nq + i) * N + x] = j == i ? d : ch_barrett(d, M.mu[j], M.m[j]);
    }
  }
}
// UW [j][z][part][N] = sum_i D[j][src(z)][i][perm_rot(z) c] K_rot(z)[i][part][j][c] for the C ciphertexts of the
// chunk: grid z = the rotation slot r < per, each thread loads its key words once and loops z = ct per + r
// NQ: the number of data primes (compile time, so the digit loop unrolls and every gather of a ct is in flight
// at once -- the runtime-nq loop sat on long-scoreboard stalls, ~21 per issue)
template <uint32_t NQ>
__global__ void k_ch_mac(const uint32_t* __restrict__ D, uint32_t dcnt, RotMap rm, uint32_t C,
                         const uint32_t* __restrict__ perms, const uint32_t* __restrict__ K, uint64_t kstride,
                         uint32_t N, uint32_t cnt, ChMods M, uint32_t* __restrict__ UW) {
  constexpr uint32_t nq = NQ, nm = NQ + 1;
  const uint32_t j = blockIdx.y, r0 = blockIdx.z, r = rm_rot(rm, r0);
  const uint32_t q = M.m[j];
  const uint64_t mu = M.mu[j];
  const uint32_t* perm = perms + (size_t)r * N;
  const uint32_t* Kz = K + (size_t)r * kstride;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    const uint32_t pc = perm[c];
    uint32_t ku[NQ], kw[NQ];
#pragma unroll
    for (uint32_t i = 0; i < nq; ++i) {
      ku[i] = Kz[((size_t)(i * 2 + 0) * nm + j) * N + c];
      kw[i] = Kz[((size_t)(i * 2 + 1) * nm + j) * N + c];
    }
#pragma unroll 2
    for (uint32_t ct = 0; ct < C; ++ct) {
      const uint32_t z = ct * rm.per + r0;
      const uint32_t* Dz = D + ((size_t)j * dcnt + rm_src(rm, z)) * nq * N + pc;
      uint32_t dv[NQ];
#pragma unroll
      for (uint32_t i = 0; i < nq; ++i) dv[i] = Dz[(size_t)i * N];
      uint64_t u = 0, w = 0;   // nq <= 7 products < 2^60 each: no overflow
#pragma unroll
      for (uint32_t i = 0; i < nq; ++i) {
        u += (uint64_t)dv[i] * ku[i];
        w += (uint64_t)dv[i] * kw[i];
      }
      UW[(((size_t)j * cnt + z) * 2 + 0) * N + c] = ch_barrett(u, mu, q);
      UW[(((size_t)j * cnt + z) * 2 + 1) * N + c] = ch_barrett(w, mu, q);
    }
  }
}
// ModDown, first half: centred lift of the (coefficient-form) P parts [z][part][N] to every data prime:
//   LB [j < nq][z][part][N]
__global__ void k_ch_lift(const uint32_t* __restrict__ UWP, uint64_t cnt2N, ChMods M, uint32_t* __restrict__ LB) {
  const uint32_t nq = M.nq, P = M.m[nq];
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < cnt2N; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = UWP[x];
    const int64_t c = v > P / 2 ? (int64_t)v - P : (int64_t)v;
    for (uint32_t j = 0; j < nq; ++j)
      LB[(size_t)j * cnt2N + x] = ch_barrett((uint64_t)(c + ((int64_t)M.m[j] << 32)), M.mu[j], M.m[j]);
  }
}
// rotated ct z (NTT domain) [j][ab][N] at out + z os:  a = (U - LB_u) P^-1,  b = bh[blk(z)][j][perm_rot(z) c] + (W - LB_w) P^-1
// (4 coefficients per thread, 16-byte accesses except the b gather)
__global__ void k_ch_combine(const uint32_t* __restrict__ UW, const uint32_t* __restrict__ LB,
                             const uint32_t* __restrict__ bh, uint64_t bs, RotMap rm, const uint32_t* __restrict__ perms,
                             uint32_t N, uint32_t cnt, ChMods M, const uint32_t* pinv, uint32_t* __restrict__ out,
                             uint64_t os) {
  const uint32_t j = blockIdx.y, z = blockIdx.z, q = M.m[j];
  const uint64_t mu = M.mu[j];
  const uint4* perm = reinterpret_cast<const uint4*>(perms + (size_t)rm_rot(rm, z) * N);
  const uint4* U = reinterpret_cast<const uint4*>(UW + (((size_t)j * cnt + z) * 2) * N);
  const uint4* lb = reinterpret_cast<const uint4*>(LB + (((size_t)j * cnt + z) * 2) * N);
  const uint32_t* b = bh + (size_t)rm_blk(rm, z) * bs + (size_t)j * 2 * N;
  uint4* o = reinterpret_cast<uint4*>(out + z * os + (size_t)j * 2 * N);
  const uint32_t pi = pinv[j], n4 = N / 4;
  auto md = [&](uint32_t x, uint32_t l) { return ch_mulmod(sub_mod(x, l, q), pi, mu, q); };
  for (uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x; c4 < n4; c4 += gridDim.x * blockDim.x) {
    const uint4 ua = U[c4], la = lb[c4], uw = U[n4 + c4], lw = lb[n4 + c4], pc = perm[c4];
    o[c4] = make_uint4(md(ua.x, la.x), md(ua.y, la.y), md(ua.z, la.z), md(ua.w, la.w));
    o[n4 + c4] = make_uint4(add_mod(b[pc.x], md(uw.x, lw.x), q), add_mod(b[pc.y], md(uw.y, lw.y), q),
                            add_mod(b[pc.z], md(uw.z, lw.z), q), add_mod(b[pc.w], md(uw.w, lw.w), q));
  }
}
// inner [ct][g'][j][ab][N] = sum_{i < b} pt[i + g' b][j] * baby_i   (NTT domain, grid z = ct g + g'),
// baby_0 = X[ct], baby_i = rot[ct (b - 1) + i - 1]  (4 coefficients per thread)
__global__ void k_ch_inner(const uint32_t* __restrict__ X, const uint32_t* __restrict__ rot,
                           const uint32_t* __restrict__ pts, uint32_t b, uint32_t g, uint32_t N, ChMods M,
                           uint32_t* __restrict__ inner) {
  const uint32_t j = blockIdx.y, z = blockIdx.z, ct = z / g, gg = z % g, nq = M.nq, q = M.m[j];
  const uint64_t mu = M.mu[j], cw = (uint64_t)nq * 2 * N;
  const uint32_t n4 = N / 4;
  for (uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x; c4 < n4; c4 += gridDim.x * blockDim.x) {
    uint64_t sa[4] = {0, 0, 0, 0}, sb[4] = {0, 0, 0, 0};
    for (uint32_t i = 0; i < b; ++i) {
      const uint32_t* bb = (i == 0 ? X + ct * cw : rot + ((uint64_t)ct * (b - 1) + i - 1) * cw) + (size_t)j * 2 * N;
      const uint4 p = __ldg(reinterpret_cast<const uint4*>(pts + ((size_t)(i + gg * b) * nq + j) * N) + c4);
      const uint4 xa = reinterpret_cast<const uint4*>(bb)[c4], xb = reinterpret_cast<const uint4*>(bb + N)[c4];
      const uint32_t ps[4] = {p.x, p.y, p.z, p.w}, as[4] = {xa.x, xa.y, xa.z, xa.w}, bs[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sa[e] += (uint64_t)ps[e] * as[e];
        sb[e] += (uint64_t)ps[e] * bs[e];
      }
      if ((i & 7) == 7) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          sa[e] = ch_barrett(sa[e], mu, q);
          sb[e] = ch_barrett(sb[e], mu, q);
        }
      }
    }
    uint4* o = reinterpret_cast<uint4*>(inner + (uint64_t)z * cw + (size_t)j * 2 * N);
    o[c4] = make_uint4(ch_barrett(sa[0], mu, q), ch_barrett(sa[1], mu, q), ch_barrett(sa[2], mu, q),
                       ch_barrett(sa[3], mu, q));
    o[n4 + c4] = make_uint4(ch_barrett(sb[0], mu, q), ch_barrett(sb[1], mu, q), ch_barrett(sb[2], mu, q),
                            ch_barrett(sb[3], mu, q));
  }
}
// acc [ct][j][ab][N] = idn[ct] (the zero-step group, NTT domain, or 0) + sum_{r < per} rot[ct per + r]
__global__ void k_ch_sum(const uint32_t* __restrict__ rot, uint32_t per, const uint32_t* __restrict__ idn, uint64_t is,
                         uint32_t C, uint32_t N, ChMods M, uint32_t* __restrict__ acc) {
  const uint32_t nq = M.nq;
  const uint64_t cw = (uint64_t)nq * 2 * N;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < C * cw; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ct = x / cw, y = x % cw;
    const uint32_t q = M.m[(uint32_t)(y / (2ull * N))];
    uint64_t s = idn ? idn[ct * is + y] : 0;
    for (uint32_t r = 0; r < per; ++r) s += rot[(ct * per + r) * cw + y];   // per <= 64 terms < 2^30
    acc[x] = (uint32_t)(s % q);
  }
}
// rescale (coefficient form): out [j < nq-1][ab][N] = (x_j - [x_top]_centred) q_top^-1 mod q_j
__global__ void k_ch_rescale(const uint32_t* __restrict__ acc_all, uint32_t C, uint32_t N, ChMods M,
                             const uint32_t* topinv, uint32_t* __restrict__ out_all) {
  const uint32_t nq = M.nq, qt = M.m[nq - 1];
  const uint64_t per = (uint64_t)(nq - 1) * 2 * N;
  for (uint64_t xx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; xx < C * per; xx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t ct = xx / per, x = xx % per;
    const uint32_t* acc = acc_all + ct * (uint64_t)nq * 2 * N;
    uint32_t* out = out_all + ct * per;
    const uint32_t j = (uint32_t)(x / (2ull * N));
    const uint64_t k = x % (2ull * N);
    const uint32_t q = M.m[j];
    const uint32_t xt = acc[(size_t)(nq - 1) * 2 * N + k];
    const int64_t c = xt > qt / 2 ? (int64_t)xt - qt : (int64_t)xt;
    const uint32_t v = sub_mod(acc[x], (uint32_t)(((c % (int64_t)q) + q) % q), q);
    out[x] = ch_mulmod(v, topinv[j], M.mu[j], q);
  }
}
__global__ void k_ch_reduce_pts(const int64_t* __restrict__ pt, uint64_t count, uint32_t N, ChMods M,
                                uint32_t* __restrict__ out) {
  const uint32_t nq = M.nq;
  const uint64_t tot = count * N;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < tot; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t t = x / N;
    const uint32_t c = (uint32_t)(x % N);
    for (uint32_t j = 0; j < nq; ++j) out[(t * nq + j) * N + c] = from_i64(pt[x], M.m[j]);
  }
}

// decryption of one limb: a [ct][N] (copied out of the ct) -> a * s (NTT domain, in place)
__global__ void k_ch_dec_mul(uint32_t* a, uint32_t n_ct, uint32_t N, const uint32_t* s_ntt, uint64_t mu, uint32_t q) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < (uint64_t)n_ct * N; x += (uint64_t)gridDim.x * blockDim.x)
    a[x] = ch_mulmod(a[x], s_ntt[x % N], mu, q);
}
// phase [ct][N] = [b + a s]_q centred
__global__ void k_ch_dec_phase(const uint32_t* __restrict__ ct, uint64_t cstride, const uint32_t* __restrict__ as,
                               uint32_t n_ct, uint32_t N, uint32_t q, int64_t* __restrict__ phase) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < (uint64_t)n_ct * N; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = x / N, c = x % N;
    const uint32_t v = add_mod(ct[r * cstride + N + c], as[x], q);
    phase[x] = v > q / 2 ? (int64_t)v - q : (int64_t)v;
  }
}

}  // namespace

// ======================================================================== chain object / C ABI
struct he_chain {
  const he_context* ctx;
  uint32_t N, logN, count;
  uint32_t primes[kChMaxQ - 1];
  uint32_t P;
  NttTable ntt[kChMaxQ];  // [0 .. count) data primes, [kChMaxQ - 1] = P
  uint32_t* consts;       // device scratch for per-level constants (qhinv, pinv, topinv): [level][3][kChMaxQ]
};

static ChMods ch_mods(const he_chain* c, uint32_t level) {
  ChMods M{};
  M.nq = level + 1;
  for (uint32_t j = 0; j < M.nq; ++j) M.m[j] = c->primes[j];
  M.m[M.nq] = c->P;
  for (uint32_t j = 0; j <= M.nq; ++j) M.mu[j] = (uint64_t)(((unsigned __int128)1 << 64) / M.m[j]);
  return M;
}
static const NttTable& ch_tab(const he_chain* c, uint32_t j, uint32_t nq) {
  return j == nq ? c->ntt[kChMaxQ - 1] : c->ntt[j];
}
// the per-limb (and per-component) transforms of a batch as one launch per NTT pass (ntt_*_multi):
// job (j, ab) for j < nj, ab < nab at base + j js + ab abs, table ch_tab(c, j, nq)
static cudaError_t ch_ntt(const he_chain* c, bool inverse, uint32_t nj, uint32_t nab, uint32_t nq, uint32_t* base,
                          uint64_t js, uint64_t abs, uint32_t count, uint64_t stride, cudaStream_t st) {
  const NttTable* t[16];
  uint32_t* d[16];
  int n = 0;
  for (uint32_t j = 0; j < nj; ++j)
    for (uint32_t ab = 0; ab < nab; ++ab) {
      t[n] = &ch_tab(c, j, nq);
      d[n++] = base + (size_t)j * js + (size_t)ab * abs;
    }
  return inverse ? ntt_inverse_multi(t, d, n, count, stride, st) : ntt_forward_multi(t, d, n, count, stride, st);
}
static const uint32_t* ch_qhinv(const he_chain* c, uint32_t level) { return c->consts + (size_t)level * 3 * kChMaxQ; }
static const uint32_t* ch_pinv(const he_chain* c, uint32_t level) { return ch_qhinv(c, level) + kChMaxQ; }
static const uint32_t* ch_topinv(const he_chain* c, uint32_t level) { return ch_qhinv(c, level) + 2 * kChMaxQ; }

extern "C" he_status he_chain_create(const he_context* ctx, const uint32_t* primes, uint32_t count, he_chain** out) {
  if (!ctx || !primes || !out) return fail(HE_EINVAL, "null argument");
  if (count < 2 || count > kChMaxQ - 1) return fail(HE_EINVAL, "a chain holds 2 .. %d primes, got %u", kChMaxQ - 1, count);
  if (primes[0] != ctx->R.q[0] || primes[1] != ctx->R.q[1])
    return fail(HE_EINVAL, "chain primes 0, 1 must be the context's (q0, q1) = (%u, %u)", ctx->R.q[0], ctx->R.q[1]);
  for (uint32_t i = 0; i < count; ++i) {
    if (primes[i] >= (1u << 30) || primes[i] == ctx->R.P) return fail(HE_EINVAL, "prime %u must be < 2^30 and != P", primes[i]);
    for (uint32_t k = 0; k < i; ++k)
      if (primes[k] == primes[i]) return fail(HE_EINVAL, "chain primes must be distinct");
  }
  he_chain* c = new (std::nothrow) he_chain();
  if (!c) return fail(HE_ENOMEM, "out of host memory");
  c->ctx = ctx;
  c->N = ctx->R.N;
  c->logN = (uint32_t)ilog2_h(c->N);
  c->count = count;
  c->P = ctx->R.P;
  for (uint32_t i = 0; i < count; ++i) c->primes[i] = primes[i];
  cudaError_t e = cudaSuccess;
  for (uint32_t i = 0; i < count && e == cudaSuccess; ++i) e = ntt_table_init(c->ntt[i], c->N, primes[i]);
  if (e == cudaSuccess) e = ntt_table_init(c->ntt[kChMaxQ - 1], c->N, c->P);
  std::vector<uint32_t> h((size_t)count * 3 * kChMaxQ, 0);
  for (uint32_t lv = 0; lv < count; ++lv) {
    const uint32_t nq = lv + 1;
    for (uint32_t i = 0; i < nq; ++i) {
      const uint64_t qi = primes[i];
      uint64_t qh = 1;
      for (uint32_t k = 0; k < nq; ++k)
        if (k != i) qh = qh * (primes[k] % qi) % qi;
      h[(size_t)lv * 3 * kChMaxQ + i] = (uint32_t)powmod_h(qh, qi - 2, qi);
      h[(size_t)lv * 3 * kChMaxQ + kChMaxQ + i] = (uint32_t)powmod_h(c->P % qi, qi - 2, qi);
      if (nq >= 2 && i + 1 < nq)
        h[(size_t)lv * 3 * kChMaxQ + 2 * kChMaxQ + i] = (uint32_t)powmod_h(primes[nq - 1] % qi, qi - 2, qi);
    }
  }
  if (e == cudaSuccess) e = cudaMalloc(&c->consts, h.size() * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(c->consts, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    for (auto& t : c->ntt) ntt_table_free(t);
    delete c;
    return cuda_fail(e, "chain tables (primes must be NTT-friendly: 1 mod 2N)");
  }
  *out = c;
  return HE_OK;
}

extern "C" he_status he_chain_destroy(he_chain* c) {
  if (c) {
    for (auto& t : c->ntt) ntt_table_free(t);
    if (c->consts) cudaFree(c->consts);
    delete c;
  }
  return HE_OK;
}

extern "C" he_status he_chain_encrypt(const he_chain* c, const int32_t* s_dev, const int64_t* pt_dev, uint32_t n_ct,
                                      uint32_t level, uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream) {
  if (!c || !s_dev || !pt_dev || !ct_dev) return fail(HE_EINVAL, "null argument");
  if (level >= c->count) return fail(HE_EINVAL, "level %u above the chain's top level %u", level, c->count - 1);
  if (n_ct == 0) return fail(HE_EINVAL, "no plaintexts");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->N, nq = level + 1;
  const ChMods M = ch_mods(c, level);
  uint32_t* s_ntt = nullptr;
  HE_CUDA(cudaMallocAsync(&s_ntt, (size_t)nq * N * sizeof(uint32_t), st), "alloc");
  k_ch_reduce_secret<<<ch_grid((uint64_t)nq * N), 256, 0, st>>>(s_dev, N, M, nq, s_ntt);
  for (uint32_t L = 0; L < nq; ++L) HE_CUDA(ntt_forward(c->ntt[L], s_ntt + (size_t)L * N, 1, N, st), "NTT(s)");
  k_ch_gen_a<<<dim3((N + 1023) / 1024, n_ct, nq), 256, 0, st>>>(c->ctx->R.rng, seed, r0, N, M, ct_dev);
  for (uint32_t L = 0; L < nq; ++L)
    HE_CUDA(ntt_forward(c->ntt[L], ct_dev + ((size_t)L * 2 + 1) * N, n_ct, (uint64_t)nq * 2 * N, st), "NTT(a)");
  k_ch_mul_s<<<ch_grid((uint64_t)n_ct * nq * N), 256, 0, st>>>(ct_dev, n_ct, N, M, s_ntt);
  for (uint32_t L = 0; L < nq; ++L)
    HE_CUDA(ntt_inverse(c->ntt[L], ct_dev + ((size_t)L * 2 + 1) * N, n_ct, (uint64_t)nq * 2 * N, st), "INTT(a s)");
  k_ch_finish<<<dim3((N + 1023) / 1024, n_ct), 256, 0, st>>>(c->ctx->R.rng, pt_dev, seed, r0, N, M, ct_dev);
  cudaFreeAsync(s_ntt, st);
  HE_CUDA(cudaGetLastError(), "chain encrypt");
  return HE_OK;
}

// phase of chain ciphertexts [n_ct][level + 1][2][N] in one limb, centred mod that prime (CRT over the limbs
// gives the integer phase, e.g. m + q0 I(X) after ModRaise)
extern "C" he_status he_chain_decrypt(const he_chain* c, const int32_t* s_dev, const uint32_t* ct_dev, uint32_t n_ct,
                                      uint32_t level, uint32_t limb, int64_t* phase_dev, void* stream) {
  if (!c || !s_dev || !ct_dev || !phase_dev) return fail(HE_EINVAL, "null argument");
  if (level >= c->count || limb > level) return fail(HE_EINVAL, "limb %u / level %u outside the chain", limb, level);
  if (n_ct == 0) return fail(HE_EINVAL, "empty batch");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->N, q = c->primes[limb];
  const uint64_t cstride = (uint64_t)(level + 1) * 2 * N;
  ChMods M{};
  M.nq = 1;
  M.m[0] = q;
  M.mu[0] = (uint64_t)(((unsigned __int128)1 << 64) / q);
  uint32_t *sj = nullptr, *tmp = nullptr;
  HE_CUDA(cudaMallocAsync(&sj, (size_t)N * sizeof(uint32_t), st), "alloc");
  HE_CUDA(cudaMallocAsync(&tmp, (size_t)n_ct * N * sizeof(uint32_t), st), "alloc");
  k_ch_reduce_secret<<<ch_grid(N), 256, 0, st>>>(s_dev, N, M, 1, sj);
  cudaError_t e = ntt_forward(c->ntt[limb], sj, 1, N, st);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(tmp, N * sizeof(uint32_t), ct_dev + (size_t)limb * 2 * N, cstride * sizeof(uint32_t),
                          N * sizeof(uint32_t), n_ct, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = ntt_forward(c->ntt[limb], tmp, n_ct, N, st);
  if (e == cudaSuccess) {
    k_ch_dec_mul<<<ch_grid((uint64_t)n_ct * N), 256, 0, st>>>(tmp, n_ct, N, sj, M.mu[0], q);
    e = ntt_inverse(c->ntt[limb], tmp, n_ct, N, st);
  }
  if (e == cudaSuccess)
    k_ch_dec_phase<<<ch_grid((uint64_t)n_ct * N), 256, 0, st>>>(ct_dev + (size_t)limb * 2 * N, cstride, tmp, n_ct, N, q,
                                                                 phase_dev);
  cudaFreeAsync(sj, st);
  cudaFreeAsync(tmp, st);
  if (e != cudaSuccess) return cuda_fail(e, "chain decrypt");
  HE_CUDA(cudaGetLastError(), "chain decrypt");
  return HE_OK;
}

extern "C" uint32_t he_chain_key_id(uint32_t level, uint32_t step) { return 0x400000u + (level << 16) + (step & 0xFFFFu); }

extern "C" he_status he_chain_rotation_keygen(const he_chain* c, uint64_t seed, const int32_t* s_dev, uint32_t level,
                                              const int32_t* steps, uint32_t count, uint32_t* keys_dev, void* stream) {
  if (!c || !s_dev || (!steps && count) || (!keys_dev && count)) return fail(HE_EINVAL, "null argument");
  if (level >= c->count) return fail(HE_EINVAL, "level %u above the chain's top level %u", level, c->count - 1);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->N, nq = level + 1, nm = nq + 1, half = N / 2;
  const ChMods M = ch_mods(c, level);
  int32_t* ss = nullptr;
  uint32_t* snew = nullptr;
  HE_CUDA(cudaMallocAsync(&ss, N * sizeof(int32_t), st), "alloc");
  HE_CUDA(cudaMallocAsync(&snew, (size_t)nm * N * sizeof(uint32_t), st), "alloc");
  k_ch_reduce_secret<<<ch_grid((uint64_t)nm * N), 256, 0, st>>>(s_dev, N, M, nm, snew);
  for (uint32_t j = 0; j < nm; ++j) HE_CUDA(ntt_forward(ch_tab(c, j, nq), snew + (size_t)j * N, 1, N, st), "NTT(s)");
  for (uint32_t t = 0; t < count; ++t) {
    const uint32_t r = (uint32_t)(((int64_t)steps[t] % half + half) % half);
    const uint64_t g = powmod_h(5, r, 2ull * N);
    k_ch_secret_auto<<<ch_grid(N), 256, 0, st>>>(s_dev, N, g, ss);
    const uint32_t id = he_chain_key_id(level, r);
    uint32_t* K = keys_dev + (size_t)t * nq * 2 * nm * N;
    for (uint32_t i = 0; i < nq; ++i)
      for (uint32_t j = 0; j < nm; ++j) {
        const uint32_t q = M.m[j];
        uint32_t gij = 0;
        if (j == i) {
          uint64_t v = c->P % q;
          for (uint32_t k = 0; k < nq; ++k)
            if (k != i) v = v * (M.m[k] % q) % q;
          gij = (uint32_t)v;
        }
        uint32_t* alpha = K + ((size_t)(i * 2 + 0) * nm + j) * N;
        uint32_t* beta = K + ((size_t)(i * 2 + 1) * nm + j) * N;
        k_ch_ksk_prep<<<ch_grid(N), 256, 0, st>>>(c->ctx->R.rng, seed, id, i, j, q, gij, ss, N, alpha, beta);
        HE_CUDA(ntt_forward(ch_tab(c, j, nq), alpha, 1, N, st), "NTT(alpha)");
        HE_CUDA(ntt_forward(ch_tab(c, j, nq), beta, 1, N, st), "NTT(t)");
        k_ch_ksk_beta<<<ch_grid(N), 256, 0, st>>>(alpha, snew + (size_t)j * N, N, q, beta);
      }
  }
  cudaFreeAsync(ss, st);
  cudaFreeAsync(snew, st);
  HE_CUDA(cudaGetLastError(), "chain keygen");
  return HE_OK;
}

extern "C" he_status he_chain_key_words(const he_chain* c, uint32_t level, uint64_t* words) {
  if (!c || !words) return fail(HE_EINVAL, "null argument");
  if (level >= c->count) return fail(HE_EINVAL, "level %u above the chain's top level %u", level, c->count - 1);
  const uint64_t nq = level + 1;
  *words = nq * 2 * (nq + 1) * c->N;
  return HE_OK;
}

extern "C" he_status he_chain_encode_pts(const he_chain* c, const int64_t* pt_dev, uint32_t count, uint32_t level,
                                         uint32_t* pts_ntt_dev, void* stream) {
  if (!c || !pt_dev || !pts_ntt_dev) return fail(HE_EINVAL, "null argument");
  if (level >= c->count) return fail(HE_EINVAL, "level %u above the chain's top level %u", level, c->count - 1);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->N, nq = level + 1;
  const ChMods M = ch_mods(c, level);
  k_ch_reduce_pts<<<ch_grid((uint64_t)count * N), 256, 0, st>>>(pt_dev, count, N, M, pts_ntt_dev);
  for (uint32_t j = 0; j < nq; ++j)
    HE_CUDA(ntt_forward(c->ntt[j], pts_ntt_dev + (size_t)j * N, count, (uint64_t)nq * N, st), "NTT(pt)");
  return HE_OK;
}

// ---------------------------------------------------------------- BSGS slot linear maps on the chain
struct he_chain_map {
  const he_chain* chain;
  uint32_t level, b, g, stride, T, N;
  uint32_t gskip;               // giant group with step 0 (no rotation), or g if none
  const uint32_t* pts;          // caller-owned NTT-domain plaintexts [b g][nq][N]
  uint32_t* perms;              // owned: baby [b-1][N] then giant [g][N]
};

extern "C" he_status he_chain_map_create(const he_chain* c, const uint32_t* pts_ntt_dev, uint32_t level, uint32_t b,
                                         uint32_t g, uint32_t stride, uint32_t T, he_chain_map** out) {
  if (!c || !pts_ntt_dev || !out) return fail(HE_EINVAL, "null argument");
  if (level < 1 || level >= c->count) return fail(HE_EINVAL, "a map consumes one level: level %u not in [1, %u]", level,
                                                  c->count - 1);
  const uint32_t N = c->N, half = N / 2;
  if (b == 0 || g == 0 || stride == 0 || b > 64 || g > 64 || (uint64_t)b * g * stride > (uint64_t)2 * half)
    return fail(HE_EINVAL, "split %ux%u with stride %u does not fit the %u slots", b, g, stride, half);
  he_chain_map* p = new (std::nothrow) he_chain_map();
  if (!p) return fail(HE_ENOMEM, "out of host memory");
  p->chain = c;
  p->level = level;
  p->b = b;
  p->g = g;
  p->stride = stride;
  p->T = T;
  p->N = N;
  p->pts = pts_ntt_dev;
  p->gskip = g;
  std::vector<uint64_t> steps;
  for (uint32_t i = 1; i < b; ++i) steps.push_back(((uint64_t)i * stride) % half);
  for (uint32_t j = 0; j < g; ++j) {
    const uint64_t s = (uint64_t)((((int64_t)j * b - (int64_t)T) * (int64_t)stride % (int64_t)half + half) % half);
    if (s == 0) p->gskip = j;
    steps.push_back(s);
  }
  const int logN = ilog2_h(N);
  std::vector<uint32_t> h(steps.size() * N);
  for (size_t t = 0; t < steps.size(); ++t) {
    const uint64_t gal = powmod_h(5, steps[t], 2ull * N);
    for (uint32_t cc = 0; cc < N; ++cc) {
      const uint64_t e = 2ull * bitrev_h(cc, logN) + 1;
      h[t * N + cc] = bitrev_h((uint32_t)(((e * gal) % (2ull * N) - 1) / 2), logN);
    }
  }
  if (cudaMalloc(&p->perms, h.size() * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemcpy(p->perms, h.data(), h.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    delete p;
    return fail(HE_ECUDA, "chain map tables");
  }
  *out = p;
  return HE_OK;
}

extern "C" he_status he_chain_map_destroy(he_chain_map* p) {
  if (p) {
    if (p->perms) cudaFree(p->perms);
    delete p;
  }
  return HE_OK;
}

constexpr uint32_t kChChunk = 8;  // ciphertexts per batched pass (bounds the workspace: ~1.3 GB at level 4, N = 2^16)

struct ChWs {
  uint32_t *X, *D, *UW, *LB, *rot, *inner, *rot2, *acc;
};
static uint64_t ch_ws_words(const he_chain_map* p, ChWs* w, uint32_t* base) {
  const uint64_t N = p->N, nq = p->level + 1, nm = nq + 1, b = p->b, g = p->g, C = kChChunk;
  const uint64_t cw = nq * 2 * N;
  const uint64_t zmax = C * std::max<uint64_t>(b > 1 ? b - 1 : 1, g);   // key switches in one batch
  uint64_t off = 0;
  auto take = [&](uint32_t*& ptr, uint64_t words) {
    if (w) ptr = base + off;
    off += (words + 63) & ~63ull;
  };
  ChWs dummy;
  ChWs& r = w ? *w : dummy;
  take(r.X, C * cw);
  take(r.D, nm * C * std::max<uint64_t>(g, 1) * nq * N);
  take(r.UW, nm * zmax * 2 * N);
  take(r.LB, nq * zmax * 2 * N);
  take(r.rot, C * (b > 1 ? b - 1 : 1) * cw);
  take(r.inner, C * g * cw);
  take(r.rot2, C * g * cw);
  take(r.acc, C * cw);
  return off;
}

extern "C" he_status he_chain_map_workspace_bytes(const he_chain_map* p, uint64_t* bytes) {
  if (!p || !bytes) return fail(HE_EINVAL, "null argument");
  *bytes = ch_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  return HE_OK;
}

// cnt key switches (RotMap rm): digits D [j][dcnt][i][N] already NTT'd -> rotated cts out [z] (os words)
static he_status ch_keyswitch(const he_chain_map* p, const ChWs& w, const ChMods& M, uint32_t cnt, uint32_t dcnt,
                              const RotMap& rm, const uint32_t* perms, const uint32_t* keys, const uint32_t* bh,
                              uint64_t bs, uint32_t* out, uint64_t os, cudaStream_t st) {
  const he_chain* c = p->chain;
  const uint32_t N = p->N, nq = M.nq, level = p->level;
  const uint64_t kstride = (uint64_t)nq * 2 * (nq + 1) * N;
  {
    const dim3 grid((N + 511) / 512, nq + 1, rm.per);
    const uint32_t C = cnt / rm.per;
    switch (nq) {
#define HE_CH_MAC(Q) \
      case Q: k_ch_mac<Q><<<grid, 256, 0, st>>>(w.D, dcnt, rm, C, perms, keys, kstride, N, cnt, M, w.UW); break;
      HE_CH_MAC(1) HE_CH_MAC(2) HE_CH_MAC(3) HE_CH_MAC(4) HE_CH_MAC(5) HE_CH_MAC(6) HE_CH_MAC(7)
#undef HE_CH_MAC
      default: return fail(HE_EINVAL, "chain level %u out of range", level);
    }
  }
  // ModDown: P parts to coefficient form, centred lift to every data prime, back to the NTT domain
  uint32_t* UWP = w.UW + (size_t)nq * cnt * 2 * N;
  HE_CUDA(ntt_inverse(ch_tab(c, nq, nq), UWP, 2 * cnt, N, st), "INTT(U_P, W_P)");
  k_ch_lift<<<ch_grid((uint64_t)cnt * 2 * N), 256, 0, st>>>(UWP, (uint64_t)cnt * 2 * N, M, w.LB);
  HE_CUDA(ch_ntt(c, false, nq, 1, nq, w.LB, (uint64_t)cnt * 2 * N, 0, 2 * cnt, N, st), "NTT(lift)");
  k_ch_combine<<<dim3((N + 4095) / 4096, nq, cnt), 256, 0, st>>>(w.UW, w.LB, bh, bs, rm, perms, N, cnt, M,
                                                                   ch_pinv(c, level), out, os);
  return HE_OK;
}

// one chunk of C ciphertexts through the map
static he_status ch_map_chunk(const he_chain_map* p, const uint32_t* ct_in, uint32_t C, const uint32_t* keys_baby,
                              const uint32_t* keys_giant, uint32_t* ct_out, const ChWs& w, cudaStream_t st) {
  const he_chain* c = p->chain;
  const uint32_t N = p->N, level = p->level, nq = level + 1, b = p->b, g = p->g;
  const ChMods M = ch_mods(c, level);
  const uint64_t cw = (uint64_t)nq * 2 * N;
  RotMap baby{};
  baby.per = b > 1 ? b - 1 : 1;
  baby.giant = 0;
  baby.g = g;
  // baby digits from the coefficient-form inputs, then the inputs to the NTT domain (baby 0)
  k_ch_digits<<<dim3((N + 255) / 256, C), 256, 0, st>>>(ct_in, cw, 2ull * N, N, C, M, ch_qhinv(c, level), baby, 0, w.D);
  HE_CUDA(ch_ntt(c, false, nq + 1, 1, nq, w.D, (uint64_t)C * nq * N, 0, C * nq, N, st), "NTT(D)");
  HE_CUDA(cudaMemcpyAsync(w.X, ct_in, C * cw * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st), "copy");
  HE_CUDA(ch_ntt(c, false, nq, 2, nq, w.X, 2ull * N, N, C, cw, st), "NTT(ct)");
  // baby rotations 1 .. b-1 of every ct (hoisted digits): rot [ct][i - 1]
  if (b > 1) {
    he_status s = ch_keyswitch(p, w, M, C * (b - 1), C, baby, p->perms, keys_baby, w.X + N, cw, w.rot, cw, st);
    if (s) return s;
  }
  // giant groups: inner [ct][j] = sum_i pt_{i + j b} baby_i
  k_ch_inner<<<dim3((N + 1023) / 1024, nq, C * g), 256, 0, st>>>(w.X, w.rot, p->pts, b, g, N, M, w.inner);
  const uint32_t nrot = p->gskip < g ? g - 1 : g;
  RotMap giant{};
  giant.per = nrot;
  giant.giant = 1;
  giant.g = g;
  for (uint32_t j = 0, t = 0; j < g; ++j)
    if (j != p->gskip) giant.gidx[t++] = (uint8_t)j;
  // the zero-step group (if any) is summed as it is (NTT domain) -- seed the sum with it before the a parts
  // of the groups go to coefficient form for their digits
  if (p->gskip < g)
    k_ch_sum<<<ch_grid(C * cw), 256, 0, st>>>(w.rot2, 0, w.inner + (size_t)p->gskip * cw, (uint64_t)g * cw, C, N, M, w.acc);
  if (nrot) {
    HE_CUDA(ch_ntt(c, true, nq, 1, nq, w.inner, 2ull * N, 0, C * g, cw, st), "INTT(inner a)");
    k_ch_digits<<<dim3((N + 255) / 256, C * nrot), 256, 0, st>>>(w.inner, cw, 2ull * N, N, C * nrot, M,
                                                                  ch_qhinv(c, level), giant, 1, w.D);
    HE_CUDA(ch_ntt(c, false, nq + 1, 1, nq, w.D, (uint64_t)C * nrot * nq * N, 0, C * nrot * nq, N, st), "NTT(D)");
    he_status s = ch_keyswitch(p, w, M, C * nrot, C * nrot, giant, p->perms + (size_t)(b - 1) * N, keys_giant,
                               w.inner + N, cw, w.rot2, cw, st);
    if (s) return s;
  }
  // acc = the zero-step group + every rotated group
  k_ch_sum<<<ch_grid(C * cw), 256, 0, st>>>(w.rot2, nrot, p->gskip < g ? w.acc : nullptr, cw, C, N, M, w.acc);
  HE_CUDA(ch_ntt(c, true, nq, 2, nq, w.acc, 2ull * N, N, C, cw, st), "INTT(acc)");
  k_ch_rescale<<<ch_grid((uint64_t)C * (nq - 1) * 2 * N), 256, 0, st>>>(w.acc, C, N, M, ch_topinv(c, level), ct_out);
  return HE_OK;
}

extern "C" he_status he_chain_map_run(const he_chain_map* p, const uint32_t* ct_in, uint32_t n_ct, uint32_t level,
                                      const uint32_t* keys_baby, const uint32_t* keys_giant, uint32_t* ct_out,
                                      void* ws_dev, uint64_t ws_bytes, void* stream, he_ledger* ledger) {
  if (!p) return fail(HE_EINVAL, "null plan");
  if (level < 1) return fail(HE_ENEEDS_BOOTSTRAP, "a slot linear map needs one level");
  if (level != p->level) return fail(HE_EINVAL, "map built for level %u, operand at level %u", p->level, level);
  if (!ct_in || !ct_out || !ws_dev || (p->b > 1 && !keys_baby) || !keys_giant) return fail(HE_EINVAL, "null argument");
  if (n_ct == 0) return fail(HE_EINVAL, "empty batch");
  const uint64_t need = ch_ws_words(p, nullptr, nullptr) * sizeof(uint32_t);
  if (ws_bytes < need)
    return fail(HE_EINVAL, "workspace too small (%llu < %llu)", (unsigned long long)ws_bytes, (unsigned long long)need);
  cudaStream_t st = (cudaStream_t)stream;
  ChWs w;
  ch_ws_words(p, &w, (uint32_t*)ws_dev);
  const uint64_t N = p->N, nq = p->level + 1;
  for (uint32_t r = 0; r < n_ct; r += kChChunk) {
    const uint32_t C = std::min<uint32_t>(kChChunk, n_ct - r);
    he_status s = ch_map_chunk(p, ct_in + (size_t)r * nq * 2 * N, C, keys_baby, keys_giant,
                               ct_out + (size_t)r * (nq - 1) * 2 * N, w, st);
    if (s) return s;
  }
  HE_CUDA(cudaGetLastError(), "chain map");
  if (ledger) {
    const uint64_t nrot = (p->b - 1) + (p->gskip < p->g ? p->g - 1 : p->g);
    ledger->ct_rotations += (int64_t)nrot * n_ct;
    ledger->pc_mults += (int64_t)p->b * p->g * n_ct;
    ledger->rescales += n_ct;
  }
  return HE_OK;
}
