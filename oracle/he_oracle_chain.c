/*
 * he_oracle_chain.c -- CPU restatement of the modulus-chain path (TEST INFRASTRUCTURE ONLY; never linked into
 * the product library): slot linear maps at any level l of a chain q_0 .. q_l (+ special prime P), which is
 * what the level-lowered, Cooley-Tukey-factorized SlotToCoeffs runs on.
 *
 * PARITY UNPINNED at the integer level like the rest of the path (the paper ships no code); this restates,
 * in exact modular arithmetic, the algorithm the CUDA path (he_chain.cu) implements:
 *  - hybrid key switching with dnum = l + 1 digits (one prime each) and the special prime P: digits
 *    d_i = [c_i (Q/q_i)^-1]_{q_i}, lifted to every modulus, U_j = sum_i d_i alpha_{i,j}, W_j = sum_i d_i beta_{i,j},
 *    ModDown x_j = (X_j - [X_P]_centred) P^-1 mod q_j  (he_oracle_rhombus.c's two-prime rule for any l);
 *    keys: beta_{i,j} = -alpha_{i,j} s + g_{i,j} s_old + e_i, g_{i,j} = P (Q/q_i) mod q_j for j == i, else 0;
 *  - a left slot rotation by r is X -> X^(5^r): digits first, then the automorphism on the lifted digits
 *    (what the NTT-domain permutation of the hoisted digits computes);
 *  - BSGS: out = rescale( sum_j rot_{(j b - T) s}( sum_i pt_{i + j b} * rot_{i s}(ct) ) ), the rescale dropping
 *    q_l with a centred top limb: (x_k - [x_l]_centred) q_l^-1 mod q_k.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

void or_sample_uniform(uint64_t seed, uint64_t stream, uint32_t q, uint32_t* out, int64_t n);
void or_sample_cbd(uint64_t seed, uint64_t stream, int32_t* out, int64_t n);
int or_negacyclic_mul(const uint32_t* a, const int32_t* s, uint32_t N, uint32_t q, uint32_t* out);
void or_automorphism(const uint32_t* p, uint32_t n, uint32_t k, uint32_t q, uint32_t* out);

#define CH_STREAM_KSK_A(id, i, j) (0xC000000000000000ULL | ((uint64_t)(id) << 16) | ((uint64_t)(i) << 8) | (uint64_t)(j))
#define CH_STREAM_KSK_E(id, i) (0xCE00000000000000ULL | ((uint64_t)(id) << 16) | ((uint64_t)(i) << 8))
#define CH_MAXQ 8

static inline uint64_t mm(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
static uint64_t pw(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mm(r, a, q);
    a = mm(a, a, q);
    e >>= 1;
  }
  return r;
}
static inline uint32_t mq(int64_t v, uint32_t q) {
  int64_t r = v % (int64_t)q;
  return (uint32_t)(r < 0 ? r + q : r);
}
static void pmul(const uint32_t* a, const uint32_t* b, uint32_t n, uint32_t q, uint32_t* out) {
  int32_t* bs = (int32_t*)malloc(sizeof(int32_t) * n);
  for (uint32_t i = 0; i < n; ++i) bs[i] = b[i] > q / 2 ? (int32_t)((int64_t)b[i] - q) : (int32_t)b[i];
  or_negacyclic_mul(a, bs, n, q, out);
  free(bs);
}
/* Q-hat_i = prod_{k != i, k < nq} m_k  mod q */
static uint64_t qhat_mod(const uint32_t* m, uint32_t nq, uint32_t i, uint32_t q) {
  uint64_t v = 1;
  for (uint32_t k = 0; k < nq; ++k)
    if (k != i) v = mm(v, m[k] % q, q);
  return v;
}

uint32_t or_chain_key_id(uint32_t level, uint32_t step) { return 0x400000u + (level << 16) + (step & 0xFFFFu); }

/* hybrid key s_old -> s_new at level nq - 1: m[0..nq) data primes, m[nq] = P;
 * ksk [i < nq][part][j < nq + 1][n] (coefficient form) */
void or_chain_ksk_gen(uint64_t seed, uint32_t id, const int32_t* s_old, const int32_t* s_new, uint32_t n,
                      const uint32_t* m, uint32_t nq, uint32_t* ksk) {
  int32_t* e = (int32_t*)malloc(sizeof(int32_t) * n);
  uint32_t* as = (uint32_t*)malloc(sizeof(uint32_t) * n);
  const uint32_t nm = nq + 1;
  for (uint32_t i = 0; i < nq; ++i) {
    or_sample_cbd(seed, CH_STREAM_KSK_E(id, i), e, n);
    for (uint32_t j = 0; j < nm; ++j) {
      const uint32_t q = m[j];
      uint32_t* alpha = ksk + ((size_t)(i * 2 + 0) * nm + j) * n;
      uint32_t* beta = ksk + ((size_t)(i * 2 + 1) * nm + j) * n;
      or_sample_uniform(seed, CH_STREAM_KSK_A(id, i, j), q, alpha, n);
      or_negacyclic_mul(alpha, s_new, n, q, as);
      const uint64_t g = (j == i) ? mm(m[nq] % q, qhat_mod(m, nq, i, q), q) : 0;
      for (uint32_t c = 0; c < n; ++c) {
        const uint64_t v = (uint64_t)(q - as[c]) + mq(e[c], q) + mm(g, mq(s_old[c], q), q);
        beta[c] = (uint32_t)(v % q);
      }
    }
  }
  free(e);
  free(as);
}

/* rotation key sigma_{5^r}(s) -> s at level nq - 1 */
void or_chain_rotation_ksk(uint64_t seed, uint32_t r, const int32_t* s, uint32_t N, const uint32_t* m, uint32_t nq,
                           uint32_t* ksk) {
  const uint64_t g = pw(5, r % (N / 2), 2ull * N);
  int32_t* ss = (int32_t*)malloc(sizeof(int32_t) * N);
  for (uint32_t i = 0; i < N; ++i) {
    const uint64_t j = ((uint64_t)i * g) % (2ull * N);
    if (j < N) ss[j] = s[i];
    else ss[j - N] = -s[i];
  }
  or_chain_ksk_gen(seed, or_chain_key_id(nq - 1, r % (N / 2)), ss, s, N, m, nq, ksk);
  free(ss);
}

/* lifted digits D [j < nq + 1][i < nq][n] of an a-part c [nq][n] */
static void ch_digits(const uint32_t* c, uint32_t n, const uint32_t* m, uint32_t nq, uint32_t* D) {
  for (uint32_t i = 0; i < nq; ++i) {
    const uint32_t qi = m[i];
    const uint64_t inv = pw(qhat_mod(m, nq, i, qi), qi - 2, qi);
    for (uint32_t k = 0; k < n; ++k) {
      const uint32_t dg = (uint32_t)mm(c[(size_t)i * n + k], inv, qi);
      for (uint32_t j = 0; j <= nq; ++j) D[((size_t)j * nq + i) * n + k] = dg % m[j];
    }
  }
}
/* rotated ct [nq][2][n] = (u, sigma_g(b) + w), (u, w) = ModDown(sum_i sigma_g(D_i) ksk_i) */
static void ch_rotate(const uint32_t* ct, const uint32_t* D, uint32_t n, uint64_t g, const uint32_t* ksk,
                      const uint32_t* m, uint32_t nq, uint32_t* out) {
  const uint32_t nm = nq + 1, P = m[nq];
  uint32_t* U = (uint32_t*)calloc((size_t)nm * n, sizeof(uint32_t));
  uint32_t* W = (uint32_t*)calloc((size_t)nm * n, sizeof(uint32_t));
  uint32_t* sd = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t j = 0; j < nm; ++j)
    for (uint32_t i = 0; i < nq; ++i) {
      or_automorphism(D + ((size_t)j * nq + i) * n, n, (uint32_t)g, m[j], sd);
      pmul(sd, ksk + ((size_t)(i * 2 + 0) * nm + j) * n, n, m[j], t);
      for (uint32_t k = 0; k < n; ++k) U[(size_t)j * n + k] = (uint32_t)(((uint64_t)U[(size_t)j * n + k] + t[k]) % m[j]);
      pmul(sd, ksk + ((size_t)(i * 2 + 1) * nm + j) * n, n, m[j], t);
      for (uint32_t k = 0; k < n; ++k) W[(size_t)j * n + k] = (uint32_t)(((uint64_t)W[(size_t)j * n + k] + t[k]) % m[j]);
    }
  for (uint32_t j = 0; j < nq; ++j) {
    const uint32_t q = m[j];
    const uint64_t pinv = pw(P % q, q - 2, q);
    or_automorphism(ct + ((size_t)j * 2 + 1) * n, n, (uint32_t)g, q, sd);
    for (uint32_t k = 0; k < n; ++k) {
      int64_t up = U[(size_t)nq * n + k], wp = W[(size_t)nq * n + k];
      if (up > P / 2) up -= P;
      if (wp > P / 2) wp -= P;
      out[((size_t)j * 2 + 0) * n + k] = (uint32_t)mm(mq((int64_t)U[(size_t)j * n + k] - up, q), pinv, q);
      const uint32_t w = (uint32_t)mm(mq((int64_t)W[(size_t)j * n + k] - wp, q), pinv, q);
      out[((size_t)j * 2 + 1) * n + k] = (uint32_t)(((uint64_t)sd[k] + w) % q);
    }
  }
  free(U);
  free(W);
  free(sd);
  free(t);
}

/*
 * BSGS slot linear map at level l = nq - 1 (one ciphertext):
 *   ct_in [nq][2][N] coefficient form; pts [b g][nq][N] coefficient form mod q_j (term k = i + j b, already
 *   rotated by -(j b - T) stride); keys_baby [b-1][nq][2][nq+1][N] for steps i stride (i = 1 .. b-1),
 *   keys_giant [g][..] for steps (j b - T) stride mod N/2 (entry j unused when that step is 0);
 *   out [nq - 1][2][N] = the rescaled sum, level l - 1.
 */
int or_chain_bsgs(uint32_t N, const uint32_t* m, uint32_t nq, uint32_t b, uint32_t g, uint32_t stride, uint32_t T,
                  const uint32_t* ct_in, const uint32_t* pts, const uint32_t* keys_baby, const uint32_t* keys_giant,
                  uint32_t* out) {
  if (nq < 2 || nq + 1 > CH_MAXQ) return -1;
  const uint32_t n = N / 2, nm = nq + 1;
  const size_t cw = (size_t)nq * 2 * N, kw = (size_t)nq * 2 * nm * N;
  uint32_t* D = (uint32_t*)malloc(sizeof(uint32_t) * nm * nq * N);
  uint32_t* baby = (uint32_t*)malloc(sizeof(uint32_t) * cw * b);
  uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * nq * N);
  memcpy(baby, ct_in, sizeof(uint32_t) * cw);
  for (uint32_t j = 0; j < nq; ++j) memcpy(a + (size_t)j * N, ct_in + (size_t)j * 2 * N, sizeof(uint32_t) * N);
  ch_digits(a, N, m, nq, D);
#pragma omp parallel for schedule(dynamic)
  for (uint32_t i = 1; i < b; ++i)
    ch_rotate(ct_in, D, N, pw(5, ((uint64_t)i * stride) % n, 2ull * N), keys_baby + (size_t)(i - 1) * kw, m, nq,
              baby + (size_t)i * cw);
  uint32_t* acc = (uint32_t*)calloc(cw, sizeof(uint32_t));
  uint32_t* inner = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* rot = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (uint32_t gj = 0; gj < g; ++gj) {
    memset(inner, 0, sizeof(uint32_t) * cw);
    for (uint32_t i = 0; i < b; ++i)
      for (uint32_t j = 0; j < nq; ++j)
        for (int ab = 0; ab < 2; ++ab) {
          pmul(baby + (size_t)i * cw + ((size_t)j * 2 + ab) * N, pts + ((size_t)(i + gj * b) * nq + j) * N, N, m[j], t);
          uint32_t* dst = inner + ((size_t)j * 2 + ab) * N;
          for (uint32_t k = 0; k < N; ++k) dst[k] = (uint32_t)(((uint64_t)dst[k] + t[k]) % m[j]);
        }
    const uint32_t step = (uint32_t)((((int64_t)gj * b - (int64_t)T) * (int64_t)stride % (int64_t)n + n) % n);
    const uint32_t* src = inner;
    if (step) {
      for (uint32_t j = 0; j < nq; ++j) memcpy(a + (size_t)j * N, inner + (size_t)j * 2 * N, sizeof(uint32_t) * N);
      ch_digits(a, N, m, nq, D);
      ch_rotate(inner, D, N, pw(5, step, 2ull * N), keys_giant + (size_t)gj * kw, m, nq, rot);
      src = rot;
    }
    for (uint32_t j = 0; j < nq; ++j)
      for (size_t k = 0; k < 2 * (size_t)N; ++k) {
        const size_t x = (size_t)j * 2 * N + k;
        acc[x] = (uint32_t)(((uint64_t)acc[x] + src[x]) % m[j]);
      }
  }
  /* rescale: drop q_l with a centred top limb */
  const uint32_t ql = m[nq - 1];
  for (uint32_t j = 0; j + 1 < nq; ++j) {
    const uint32_t q = m[j];
    const uint64_t inv = pw(ql % q, q - 2, q);
    for (size_t k = 0; k < 2 * (size_t)N; ++k) {
      const uint32_t xl = acc[(size_t)(nq - 1) * 2 * N + k];
      const int64_t c = xl > ql / 2 ? (int64_t)xl - ql : (int64_t)xl;
      out[(size_t)j * 2 * N + k] = (uint32_t)mm(mq((int64_t)acc[(size_t)j * 2 * N + k] - c, q), inv, q);
    }
  }
  free(D);
  free(baby);
  free(a);
  free(acc);
  free(inner);
  free(rot);
  free(t);
  return 0;
}
