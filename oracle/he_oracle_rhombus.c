/*
 * he_oracle_rhombus.c -- CPU restatement of the Rhombus PCMv path (TEST INFRASTRUCTURE ONLY).
 *
 * PARITY UNPINNED: hesim does not implement the PCMv; the paper gives only the step
 * list and the weight shuffle h (bitrev.py:48-54).  This file
 * restates, in plain exact modular arithmetic, the algorithm the CUDA path implements:
 *
 *  (D) decompose: one hybrid key switch (dnum = 2 RNS digits, special prime P) of the degree-N
 *      ciphertext from s to the sparse key s'(X^rho), rho = N/N', after which the X^rho index
 *      split is a free map to rho RLWE-N' ciphertexts under s';
 *  (M) MVM: coefficient-encoded inner products -- for output row r and input piece p the
 *      plaintext w_{r,p}(Z) = c_pack * sum_k W~[r][N' p + h(k)] Z^{-k} puts <row r, piece p> in the
 *      constant coefficient of w_{r,p} * piece_p; products are summed over pieces;
 *  (P) output packing: PackLWEs (Chen-Dai-Kim-Song 2021) over the N' row ciphertexts of an output
 *      piece -- log2 N' levels of  E + X^{N'/2^l} O + sigma_{2^l+1}(E - X^{N'/2^l} O), each
 *      automorphism followed by a Galois key switch; c_pack = N'^-1 cancels the 2^l growth;
 *  (R) rescale by q1 (one level), (C) compose: the free X^rho interleave.
 *
 * Vector layout (App. A with h): element e of the input / output vector sits in piece p = e / N',
 * piece coefficient k with h(k) = e mod N', i.e. degree-N coefficient p + rho k.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

uint64_t or_rng_key(uint64_t seed, uint64_t stream);
void or_sample_uniform(uint64_t seed, uint64_t stream, uint32_t q, uint32_t* out, int64_t n);
void or_sample_cbd(uint64_t seed, uint64_t stream, int32_t* out, int64_t n);
void or_sample_ternary(uint64_t seed, uint64_t stream, int32_t* out, int64_t n);
int or_negacyclic_mul(const uint32_t* a, const int32_t* s, uint32_t N, uint32_t q, uint32_t* out);

#define STREAM_SECRET_RH 0x5EC1000000000000ULL
#define STREAM_KSK_A(id, i, j) (0xC000000000000000ULL | ((uint64_t)(id) << 16) | ((uint64_t)(i) << 8) | (uint64_t)(j))
#define STREAM_KSK_E(id, i) (0xCE00000000000000ULL | ((uint64_t)(id) << 16) | ((uint64_t)(i) << 8))

static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static inline uint32_t modq_i64(int64_t v, uint32_t q) {
  int64_t r = v % (int64_t)q;
  return (uint32_t)(r < 0 ? r + q : r);
}
static int ilog2u(uint32_t x) {
  int l = 0;
  while ((1u << l) < x) ++l;
  return l;
}
static uint32_t brev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int t = 0; t < bits; ++t) r |= ((x >> t) & 1u) << (bits - 1 - t);
  return r;
}
/* h of PAPER.md:676-680 generalised to degree n: fix the top bit, reverse the others */
uint32_t or_half_reverse(uint32_t x, uint32_t n) {
  int l = ilog2u(n) - 1;
  return (x & (n >> 1)) | brev(x & ((n >> 1) - 1), l);
}

/* product of a residue poly with a residue poly (both in [0,q)) via the signed NTT helper */
static void polymul(const uint32_t* a, const uint32_t* b, uint32_t n, uint32_t q, uint32_t* out) {
  int32_t* bs = (int32_t*)malloc(sizeof(int32_t) * n);
  /* or_negacyclic_mul takes a signed second operand; centre b (|b| < q/2 < 2^29 fits int32) */
  for (uint32_t i = 0; i < n; ++i) bs[i] = b[i] > q / 2 ? (int32_t)((int64_t)b[i] - q) : (int32_t)b[i];
  or_negacyclic_mul(a, bs, n, q, out);
  free(bs);
}

/* sigma_k(p)(X) = p(X^k) in Z_q[X]/(X^n+1), k odd */
void or_automorphism(const uint32_t* p, uint32_t n, uint32_t k, uint32_t q, uint32_t* out) {
  for (uint32_t i = 0; i < n; ++i) {
    uint64_t j = ((uint64_t)i * k) % (2ull * n);
    if (j < n) out[j] = p[i];
    else out[j - n] = p[i] ? q - p[i] : 0;
  }
}
/* X^e * p (0 <= e < 2n) */
static void monomial_mul(const uint32_t* p, uint32_t n, uint32_t e, uint32_t q, uint32_t* out) {
  for (uint32_t i = 0; i < n; ++i) {
    uint64_t j = (uint64_t)i + e;
    int neg = 0;
    while (j >= n) {
      j -= n;
      neg ^= 1;
    }
    out[j] = (neg && p[i]) ? q - p[i] : p[i];
  }
}

/*
 * Hybrid key-switching key from s_old to s_new (degree n; moduli m[0..2] = q0, q1, P):
 *   ksk[i][0][j] = alpha_{i,j} (uniform),  ksk[i][1][j] = -alpha s_new + g_{i,j} s_old + e_i  (mod m_j)
 *   g_{i,j} = P * Qhat_i (mod m_j): nonzero only for j == i (Qhat_0 = q1, Qhat_1 = q0).
 * Layout: ksk[((i * 2 + part) * 3 + j) * n + c].
 */
void or_ksk_gen(uint64_t seed, uint32_t id, const int32_t* s_old, const int32_t* s_new, uint32_t n, const uint32_t* m,
                uint32_t* ksk) {
  int32_t* e = (int32_t*)malloc(sizeof(int32_t) * n);
  uint32_t* as = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < 2; ++i) {
    or_sample_cbd(seed, STREAM_KSK_E(id, i), e, n);
    for (uint32_t j = 0; j < 3; ++j) {
      const uint32_t q = m[j];
      uint32_t* alpha = ksk + ((size_t)(i * 2 + 0) * 3 + j) * n;
      uint32_t* beta = ksk + ((size_t)(i * 2 + 1) * 3 + j) * n;
      or_sample_uniform(seed, STREAM_KSK_A(id, i, j), q, alpha, n);
      or_negacyclic_mul(alpha, s_new, n, q, as);
      uint64_t g = 0;
      if (j == i) g = mulmod(m[2] % q, m[1 - i] % q, q);
      for (uint32_t c = 0; c < n; ++c) {
        uint64_t v = (uint64_t)(q - as[c]) + modq_i64(e[c], q) + mulmod(g, modq_i64(s_old[c], q), q);
        beta[c] = (uint32_t)(v % q);
      }
    }
  }
  free(e);
  free(as);
}

/*
 * Key switch of c (2 limbs, coefficient form, [limb][n]) with ksk -> (u, w) [limb][n] mod q0, q1:
 *   d_i = c_i * [Qhat_i^-1]_{q_i} mod q_i  (RNS digit, integer in [0, q_i))
 *   U_j = sum_i d_i * alpha_{i,j},  W_j = sum_i d_i * beta_{i,j}   (mod m_j, j = q0, q1, P)
 *   ModDown: x_j = (X_j - [X_P]_centred) * P^-1 mod q_j
 * so that w + u s_new = c s_old + small.
 */
/* ModUp + key product of one term, accumulated into U, W [3][n] (mod m_j) */
static void ks_accumulate(const uint32_t* c, const uint32_t* ksk, uint32_t n, const uint32_t* m, uint32_t* U,
                          uint32_t* W) {
  uint32_t* d[2];
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* dl = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (int i = 0; i < 2; ++i) {
    d[i] = (uint32_t*)malloc(sizeof(uint32_t) * n);
    const uint32_t qi = m[i];
    const uint64_t inv = powmod(m[1 - i] % qi, qi - 2, qi);
    for (uint32_t k = 0; k < n; ++k) d[i][k] = (uint32_t)mulmod(c[(size_t)i * n + k], inv, qi);
  }
  for (int j = 0; j < 3; ++j) {
    const uint32_t q = m[j];
    for (int i = 0; i < 2; ++i) {
      for (uint32_t k = 0; k < n; ++k) dl[k] = d[i][k] % q;
      polymul(dl, ksk + ((size_t)(i * 2 + 0) * 3 + j) * n, n, q, t);
      for (uint32_t k = 0; k < n; ++k) U[(size_t)j * n + k] = (uint32_t)(((uint64_t)U[(size_t)j * n + k] + t[k]) % q);
      polymul(dl, ksk + ((size_t)(i * 2 + 1) * 3 + j) * n, n, q, t);
      for (uint32_t k = 0; k < n; ++k) W[(size_t)j * n + k] = (uint32_t)(((uint64_t)W[(size_t)j * n + k] + t[k]) % q);
    }
  }
  free(d[0]);
  free(d[1]);
  free(t);
  free(dl);
}
/* ModDown: x_j = (X_j - [X_P]_centred) * P^-1 mod q_j */
static void ks_moddown(const uint32_t* U, const uint32_t* W, uint32_t n, const uint32_t* m, uint32_t* u, uint32_t* w) {
  const uint32_t P = m[2];
  for (int j = 0; j < 2; ++j) {
    const uint32_t q = m[j];
    const uint64_t pinv = powmod(P % q, q - 2, q);
    for (uint32_t k = 0; k < n; ++k) {
      int64_t up = U[2 * (size_t)n + k], wp = W[2 * (size_t)n + k];
      if (up > P / 2) up -= P;
      if (wp > P / 2) wp -= P;
      u[(size_t)j * n + k] = (uint32_t)mulmod(modq_i64((int64_t)U[(size_t)j * n + k] - up, q), pinv, q);
      w[(size_t)j * n + k] = (uint32_t)mulmod(modq_i64((int64_t)W[(size_t)j * n + k] - wp, q), pinv, q);
    }
  }
}
void or_keyswitch(const uint32_t* c, const uint32_t* ksk, uint32_t n, const uint32_t* m, uint32_t* u, uint32_t* w) {
  uint32_t* U = (uint32_t*)calloc((size_t)3 * n, sizeof(uint32_t));
  uint32_t* W = (uint32_t*)calloc((size_t)3 * n, sizeof(uint32_t));
  ks_accumulate(c, ksk, n, m, U, W);
  ks_moddown(U, W, n, m, u, w);
  free(U);
  free(W);
}

/* sparse small secret s' (degree n_small) and its embedding s'(X^rho) (degree N) */
void or_rhombus_secret(uint64_t seed, uint32_t n_small, uint32_t N, int32_t* s_small, int32_t* s_up) {
  or_sample_ternary(seed, STREAM_SECRET_RH, s_small, n_small);
  memset(s_up, 0, sizeof(int32_t) * N);
  const uint32_t rho = N / n_small;
  for (uint32_t k = 0; k < n_small; ++k) s_up[(size_t)rho * k] = s_small[k];
}

/* Galois key of sigma_k: from sigma_k(s') to s'  (id = 1 + log2(k - 1)) */
void or_galois_ksk(uint64_t seed, uint32_t level, const int32_t* s_small, uint32_t n, const uint32_t* m, uint32_t* ksk) {
  const uint32_t k = (1u << level) + 1;
  int32_t* ss = (int32_t*)malloc(sizeof(int32_t) * n);
  for (uint32_t i = 0; i < n; ++i) {
    uint64_t j = ((uint64_t)i * k) % (2ull * n);
    if (j < n) ss[j] = s_small[i];
    else ss[j - n] = -s_small[i];
  }
  or_ksk_gen(seed, 1 + level, ss, s_small, n, m, ksk);
  free(ss);
}

/* ciphertext helpers: ct = [limb][2 (a, b)][n] */
static void ct_apply_sigma_ks(const uint32_t* ct, uint32_t n, uint32_t k, const uint32_t* ksk, const uint32_t* m,
                              uint32_t* out) {
  uint32_t* sa = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  uint32_t* sb = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  for (int L = 0; L < 2; ++L) or_automorphism(ct + ((size_t)L * 2 + 0) * n, n, k, m[L], sa + (size_t)L * n);
  or_keyswitch(sa, ksk, n, m, u, w);
  for (int L = 0; L < 2; ++L) {
    or_automorphism(ct + ((size_t)L * 2 + 1) * n, n, k, m[L], sb);
    for (uint32_t i = 0; i < n; ++i) {
      out[((size_t)L * 2 + 0) * n + i] = u[(size_t)L * n + i];
      out[((size_t)L * 2 + 1) * n + i] = (uint32_t)(((uint64_t)sb[i] + w[(size_t)L * n + i]) % m[L]);
    }
  }
  free(sa);
  free(sb);
  free(u);
  free(w);
}

/* PackLWEs, recursive (CDKS21): v = list of 2^l cts (each [2][2][n]).  Level l (count = 2^l) combines
 *   E + X^{sb / 2^l} O + sigma_{1 + gm 2^l}(E - X^{sb / 2^l} O)
 * Rhombus: sb = n, gm = 1 (the full ring); ring packing: sb = k, gm = d (the subring Z[X^k], N = d k). */
static void pack_rec(const uint32_t* const* v, uint32_t count, uint32_t sb, uint32_t gm, uint32_t n,
                     const uint32_t* const* gal, const uint32_t* m, uint32_t* out) {
  const size_t cw = (size_t)4 * n;
  if (count == 1) {
    memcpy(out, v[0], sizeof(uint32_t) * cw);
    return;
  }
  const uint32_t half = count / 2;
  const uint32_t** ev = (const uint32_t**)calloc(half, sizeof(void*));
  const uint32_t** od = (const uint32_t**)calloc(half, sizeof(void*));
  for (uint32_t i = 0; i < half; ++i) {
    ev[i] = v[2 * i];
    od[i] = v[2 * i + 1];
  }
  uint32_t* E = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* O = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  pack_rec(ev, half, sb, gm, n, gal, m, E);
  pack_rec(od, half, sb, gm, n, gal, m, O);
  const int l = ilog2u(count);
  const uint32_t e = sb >> l;  /* X^{sb / 2^l} */
  uint32_t* MO = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* T = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* ST = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  for (int L = 0; L < 2; ++L)
    for (int ab = 0; ab < 2; ++ab)
      monomial_mul(O + ((size_t)L * 2 + ab) * n, n, e, m[L], MO + ((size_t)L * 2 + ab) * n);
  for (int L = 0; L < 2; ++L)
    for (size_t i = 0; i < (size_t)2 * n; ++i) {
      size_t x = (size_t)L * 2 * n + i;
      T[x] = (uint32_t)(((uint64_t)E[x] + m[L] - MO[x]) % m[L]);
    }
  ct_apply_sigma_ks(T, n, (gm << l) + 1, gal[l - 1], m, ST);
  for (int L = 0; L < 2; ++L)
    for (size_t i = 0; i < (size_t)2 * n; ++i) {
      size_t x = (size_t)L * 2 * n + i;
      out[x] = (uint32_t)(((uint64_t)E[x] + MO[x] + ST[x]) % m[L]);
    }
  free(ev);
  free(od);
  free(E);
  free(O);
  free(MO);
  free(T);
  free(ST);
}

/*
 * Full Rhombus PCMv.
 *   ct_in  [2 limbs][2][N]           level-1 input under s
 *   ksk_dec [2][2][3][N]            key from s to s'(X^rho)
 *   gal     [log2 n][2][2][3][n]     Galois keys sigma_{2^l+1}, l = 1..log2 n
 *   Wt      int64 [n_out][n_in]      W~ = round(q1 W) (unshuffled; h is applied here)
 * outputs: pieces_out [p_out][2][n] level-1 packed pieces before rescale (optional, may be NULL),
 *          out [N] x 2 (a, b) level 0 under s'(X^rho)  -> out[0..N) = a, out[N..2N) = b.
 */
int or_rhombus_pcmv(uint32_t N, uint32_t n, const uint32_t* m, const uint32_t* ct_in, const uint32_t* ksk_dec,
                    const uint32_t* gal, const int64_t* Wt, uint32_t n_out, uint32_t n_in, uint32_t* pieces_out,
                    uint32_t* out) {
  const uint32_t rho = N / n, p_in = (n_in + n - 1) / n, p_out = (n_out + n - 1) / n;
  const int lg = ilog2u(n);
  const size_t cw = (size_t)4 * n;
  /* (D) key switch to s'(X^rho), then split */
  uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  uint32_t* a_in = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  for (int L = 0; L < 2; ++L) memcpy(a_in + (size_t)L * N, ct_in + ((size_t)L * 2 + 0) * N, sizeof(uint32_t) * N);
  or_keyswitch(a_in, ksk_dec, N, m, u, w);
  uint32_t* pieces = (uint32_t*)malloc(sizeof(uint32_t) * cw * p_in);
  for (uint32_t p = 0; p < p_in; ++p)
    for (int L = 0; L < 2; ++L)
      for (uint32_t k = 0; k < n; ++k) {
        const size_t c = p + (size_t)rho * k;
        pieces[(size_t)p * cw + ((size_t)L * 2 + 0) * n + k] = u[(size_t)L * N + c];
        pieces[(size_t)p * cw + ((size_t)L * 2 + 1) * n + k] =
            (uint32_t)(((uint64_t)ct_in[((size_t)L * 2 + 1) * N + c] + w[(size_t)L * N + c]) % m[L]);
      }
  free(u);
  free(w);
  free(a_in);
  /* (M) row ciphertexts, in packing leaf order: leaf j of output piece o is row n*o + h(j) */
  const size_t nrows = (size_t)p_out * n;
  uint32_t* rows = (uint32_t*)calloc(nrows * cw, sizeof(uint32_t));
  uint32_t* pt = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (size_t leaf = 0; leaf < nrows; ++leaf) {
    const uint32_t o = (uint32_t)(leaf / n), j = (uint32_t)(leaf % n);
    const uint32_t r = n * o + or_half_reverse(j, n);
    if (r >= n_out) continue;
    for (uint32_t p = 0; p < p_in; ++p)
      for (int L = 0; L < 2; ++L) {
        const uint32_t q = m[L];
        const uint64_t cpack = powmod(n % q, q - 2, q);
        /* w(Z) = cpack * sum_k W~[r][n p + h(k)] Z^{-k} */
        for (uint32_t k = 0; k < n; ++k) {
          const uint32_t col = n * p + or_half_reverse(k, n);
          const int64_t wv = col < n_in ? Wt[(size_t)r * n_in + col] : 0;
          uint32_t v = (uint32_t)mulmod(modq_i64(wv, q), cpack, q);
          if (k == 0) pt[0] = v;
          else pt[n - k] = v ? q - v : 0;
        }
        for (int ab = 0; ab < 2; ++ab) {
          polymul(pieces + (size_t)p * cw + ((size_t)L * 2 + ab) * n, pt, n, q, t);
          uint32_t* dst = rows + leaf * cw + ((size_t)L * 2 + ab) * n;
          for (uint32_t k = 0; k < n; ++k) dst[k] = (uint32_t)(((uint64_t)dst[k] + t[k]) % q);
        }
      }
  }
  free(pt);
  free(t);
  free(pieces);
  /* (P) pack each output piece */
  const uint32_t** gk = (const uint32_t**)malloc(sizeof(void*) * lg);
  for (int l = 0; l < lg; ++l) gk[l] = gal + (size_t)l * 12 * n;
  const uint32_t** leaves = (const uint32_t**)malloc(sizeof(void*) * n);
  uint32_t* packed = (uint32_t*)malloc(sizeof(uint32_t) * cw * p_out);
  for (uint32_t o = 0; o < p_out; ++o) {
    for (uint32_t j = 0; j < n; ++j) leaves[j] = rows + ((size_t)o * n + j) * cw;
    pack_rec(leaves, n, n, 1, n, gk, m, packed + (size_t)o * cw);
  }
  if (pieces_out) memcpy(pieces_out, packed, sizeof(uint32_t) * cw * p_out);
  /* (R) rescale, (C) compose */
  const uint32_t q0 = m[0], q1 = m[1];
  const uint64_t q1inv = powmod(q1 % q0, q0 - 2, q0);
  memset(out, 0, sizeof(uint32_t) * 2 * N);
  for (uint32_t o = 0; o < p_out; ++o)
    for (int ab = 0; ab < 2; ++ab)
      for (uint32_t k = 0; k < n; ++k) {
        const uint32_t x0 = packed[(size_t)o * cw + (size_t)ab * n + k];
        const uint32_t x1 = packed[(size_t)o * cw + ((size_t)2 + ab) * n + k];
        const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - q1 : (int64_t)x1;
        out[(size_t)ab * N + o + (size_t)rho * k] = (uint32_t)mulmod(modq_i64((int64_t)x0 - x1c, q0), q1inv, q0);
      }
  free(gk);
  free(leaves);
  free(packed);
  free(rows);
  return 0;
}

/* encrypt a vector (n_in values) in the PCMv input layout at level 1 under s (degree N):
 * element e -> coefficient (e / n) + rho * k with h(k) = e mod n */
void or_encode_vector(const double* v, uint32_t n_vals, uint32_t N, uint32_t n, double delta, int64_t* pt) {
  const uint32_t rho = N / n;
  memset(pt, 0, sizeof(int64_t) * N);
  for (uint32_t e = 0; e < n_vals; ++e) {
    const uint32_t p = e / n, k = or_half_reverse(e % n, n);
    pt[p + (size_t)rho * k] = llrint(delta * v[e]);
  }
}
void or_decode_vector(const int64_t* phase, uint32_t n_vals, uint32_t N, uint32_t n, double delta, double* v) {
  const uint32_t rho = N / n;
  for (uint32_t e = 0; e < n_vals; ++e) {
    const uint32_t p = e / n, k = or_half_reverse(e % n, n);
    v[e] = (double)phase[p + (size_t)rho * k] / delta;
  }
}

/* ================================================================== MLWE -> RLWE ring packing
 *
 * The PCMM's MLWE output row y (component t' of output block Y, y = k Y + t') is component 0 of the
 * level-1 RLWE product C_y = sum_r w_{y,r}(X) ct_r, w_{y,r} = sum_t W~[y][k r + t] X^-t, whose
 *   a-polynomial  A_y[k m - j] = a'_y[j][m]   (negacyclic: A_y[N + c] = -a'_y[j][0] for c = -j < 0)
 * is fully determined by the un-rescaled a' words, while only component 0 of its b-polynomial,
 * B_y[k m] = b'_y[m], is known -- which is all the trace needs.  PackLWEs over the subring Z[X^k]
 * (pack_rec with sb = k, gm = d: log2 k levels, automorphisms sigma_{1 + 2^l d} fixing X^{k/2^(l-1)}
 * and negating X^{k/2^l}) sums the k leaves of a block into one RLWE ciphertext whose phase is
 * k sum_t' X^t' phase_{kY+t'}(X^k), so the leaves are pre-scaled by k^-1; a final rescale by q1
 * gives level 0.  The packed phase of block Y at coefficient t' + k m is row (Y, t')'s phase at m:
 * the activation layout of or_encode_acts, i.e. the packed output is the next layer's input format.
 */

/* Galois key of sigma_g, g = 1 + 2^l d, at degree N: from sigma_g(s) to s  (key id 0x100 + l) */
void or_ring_galois_ksk(uint64_t seed, uint32_t l, const int32_t* s, uint32_t N, uint32_t d, const uint32_t* m,
                        uint32_t* ksk) {
  const uint64_t g = ((uint64_t)d << l) + 1;
  int32_t* ss = (int32_t*)malloc(sizeof(int32_t) * N);
  for (uint32_t i = 0; i < N; ++i) {
    uint64_t j = ((uint64_t)i * g) % (2ull * N);
    if (j < N) ss[j] = s[i];
    else ss[j - N] = -s[i];
  }
  or_ksk_gen(seed, 0x100 + l, ss, s, N, m, ksk);
  free(ss);
}

/*
 * leaves  [cnt][2 limbs][2 (a, b)][N]  level-1 leaf ciphertexts C_y (already scaled by k^-1), cnt = blocks k
 * gal     [log2 k][2][2][3][N]         keys of or_ring_galois_ksk, l = 1 .. log2 k
 * packed  [blocks][2][2][N]            level-1 packed ciphertexts (optional)
 * out     [blocks][2 (a, b)][N]        rescaled, level 0
 */
int or_ring_pack(uint32_t N, uint32_t d, uint32_t k, const uint32_t* m, const uint32_t* leaves, uint32_t cnt,
                 const uint32_t* gal, uint32_t* packed, uint32_t* out) {
  if (N != d * k || cnt % k) return 1;
  const int lg = ilog2u(k);
  const uint32_t blocks = cnt / k;
  const size_t cw = (size_t)4 * N;
  const uint32_t** gk = (const uint32_t**)malloc(sizeof(void*) * (lg ? lg : 1));
  for (int l = 0; l < lg; ++l) gk[l] = gal + (size_t)l * 12 * N;
  const uint32_t q0 = m[0], q1 = m[1];
  const uint64_t q1inv = powmod(q1 % q0, q0 - 2, q0);
  int rc = 0;
#pragma omp parallel for schedule(dynamic)
  for (uint32_t o = 0; o < blocks; ++o) {
    const uint32_t** lv = (const uint32_t**)malloc(sizeof(void*) * k);
    uint32_t* pk = (uint32_t*)malloc(sizeof(uint32_t) * cw);
    for (uint32_t j = 0; j < k; ++j) lv[j] = leaves + ((size_t)o * k + j) * cw;
    pack_rec(lv, k, k, d, N, gk, m, pk);
    if (packed) memcpy(packed + (size_t)o * cw, pk, sizeof(uint32_t) * cw);
    for (int ab = 0; ab < 2; ++ab)
      for (uint32_t c = 0; c < N; ++c) {
        const uint32_t x0 = pk[(size_t)ab * N + c], x1 = pk[((size_t)2 + ab) * N + c];
        const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - q1 : (int64_t)x1;
        out[((size_t)o * 2 + ab) * N + c] = (uint32_t)mulmod(modq_i64((int64_t)x0 - x1c, q0), q1inv, q0);
      }
    free(lv);
    free(pk);
  }
  free(gk);
  return rc;
}

/* ------------------------------------------------------------------ MLWE -> RLWE key switching
 * The cheaper packing (HERMES / BCHPS-style): block Y's packed phase
 *   Phi = sum_t X^t (b'_t + sum_j a'_{t,j} * s_j)(X^k) = b_Y + sum_j alpha_j(X) s^_j(X)
 * with b_Y the composed b' words (RLWE order), alpha_j[t + k m] = a'_{kY+t}[j][m] and
 * s^_j(X) = s_j(X^k) (s^_j[k m] = s[j + k m]).  One hybrid key switch per component j from s^_j to s,
 * summed BEFORE the single ModDown:  (a, b) = (sum_j u_j, b_Y + sum_j w_j), then rescale by q1.
 * k key switches per block (no automorphisms, no k^-1 pre-scale, noise grows ~sqrt(k)).
 */
/* key from s^_j = s_j(X^k) to s  (key id 0x200 + j) */
void or_mlwe_ksk(uint64_t seed, uint32_t j, const int32_t* s, uint32_t N, uint32_t k, const uint32_t* m, uint32_t* ksk) {
  int32_t* sj = (int32_t*)calloc(N, sizeof(int32_t));
  for (uint32_t c = 0; c < N; c += k) sj[c] = s[j + c];
  or_ksk_gen(seed, 0x200 + j, sj, s, N, m, ksk);
  free(sj);
}
/*
 * raw_b [2 limbs][n_out/k][N]      un-rescaled b' words, RLWE order (he_pcmm_run_level1)
 * raw_a [2 limbs][n_out][k d]      un-rescaled a' words, MLWE layout a'[j][m] at d j + m
 * ksk   [k][2][2][3][N]            or_mlwe_ksk, j = 0 .. k-1
 * out   [n_out/k][2 (a, b)][N]     level 0
 */
int or_mlwe_to_rlwe(uint32_t d, uint32_t k, const uint32_t* m, const uint32_t* raw_b, const uint32_t* raw_a,
                    uint32_t n_out, const uint32_t* ksk, uint32_t* out) {
  const uint32_t N = d * k;
  if (n_out % k) return 1;
  const uint32_t blocks = n_out / k;
  const uint32_t q0 = m[0], q1 = m[1];
  const uint64_t q1inv = powmod(q1 % q0, q0 - 2, q0);
#pragma omp parallel for schedule(dynamic)
  for (uint32_t Y = 0; Y < blocks; ++Y) {
    uint32_t* U = (uint32_t*)calloc((size_t)3 * N, sizeof(uint32_t));
    uint32_t* W = (uint32_t*)calloc((size_t)3 * N, sizeof(uint32_t));
    uint32_t* al = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
    uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
    uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
    for (uint32_t j = 0; j < k; ++j) {
      for (int L = 0; L < 2; ++L)
        for (uint32_t t = 0; t < k; ++t)
          for (uint32_t mm = 0; mm < d; ++mm)
            al[(size_t)L * N + t + (size_t)k * mm] =
                raw_a[((size_t)L * n_out + (size_t)Y * k + t) * N + (size_t)d * j + mm];
      ks_accumulate(al, ksk + (size_t)j * 12 * N, N, m, U, W);
    }
    ks_moddown(U, W, N, m, u, w);
    for (uint32_t c = 0; c < N; ++c) {
      uint32_t x[2][2];
      for (int L = 0; L < 2; ++L) {
        x[L][0] = u[(size_t)L * N + c];
        x[L][1] = (uint32_t)(((uint64_t)raw_b[((size_t)L * blocks + Y) * N + c] + w[(size_t)L * N + c]) % m[L]);
      }
      for (int ab = 0; ab < 2; ++ab) {
        const int64_t x1c = x[1][ab] > q1 / 2 ? (int64_t)x[1][ab] - q1 : (int64_t)x[1][ab];
        out[((size_t)Y * 2 + ab) * N + c] = (uint32_t)mulmod(modq_i64((int64_t)x[0][ab] - x1c, q0), q1inv, q0);
      }
    }
    free(U);
    free(W);
    free(al);
    free(u);
    free(w);
  }
  return 0;
}

/* ------------------------------------------------------------------ one-digit variant (he_ring_pack KEYSWITCH1)
 * The same packed phase, key-switched with ONE digit -- alpha_j itself, centred mod Q = q0 q1 -- and the special
 * modulus P1 P2 (m4 = {q0, q1, P1 = P, P2}): keys (alpha, beta = -alpha s + e + P1 P2 s^_j) mod q0, q1, P1, P2
 * (beta's gadget term vanishes mod P1, P2), U = sum_j [alpha_j]_Q K_j[0], W = sum_j [alpha_j]_Q K_j[1] mod each
 * modulus, ModDown x_q = (X_q - [X]_{P1 P2}) (P1 P2)^-1 mod q with [X]_{P1 P2} centred by CRT.
 */
/* key from s^_j = s_j(X^k) to s (key id 0x300 + j, digit i = 0): ksk [2 (alpha, beta)][4][N], coefficient form */
void or_mlwe_ksk1(uint64_t seed, uint32_t j, const int32_t* s, uint32_t N, uint32_t k, const uint32_t* m4,
                  uint32_t* ksk) {
  int32_t* sj = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* e = (int32_t*)malloc(sizeof(int32_t) * N);
  uint32_t* as = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (uint32_t c = 0; c < N; c += k) sj[c] = s[j + c];
  const uint32_t id = 0x300 + j;
  or_sample_cbd(seed, STREAM_KSK_E(id, 0), e, N);
  for (uint32_t mi = 0; mi < 4; ++mi) {
    const uint32_t q = m4[mi];
    uint32_t* alpha = ksk + ((size_t)0 * 4 + mi) * N;
    uint32_t* beta = ksk + ((size_t)1 * 4 + mi) * N;
    or_sample_uniform(seed, STREAM_KSK_A(id, 0, mi), q, alpha, N);
    or_negacyclic_mul(alpha, s, N, q, as);
    const uint64_t g = mi < 2 ? mulmod(m4[2] % q, m4[3] % q, q) : 0;
    for (uint32_t c = 0; c < N; ++c) {
      uint64_t v = (uint64_t)(q - as[c]) + modq_i64(e[c], q) + mulmod(g, modq_i64(sj[c], q), q);
      beta[c] = (uint32_t)(v % q);
    }
  }
  free(sj);
  free(e);
  free(as);
}
/* raw_b, raw_a as or_mlwe_to_rlwe; ksk [k][2][4][N] (or_mlwe_ksk1) -> out [n_out/k][2 (a, b)][N] level 0 */
int or_mlwe_to_rlwe1(uint32_t d, uint32_t k, const uint32_t* m4, const uint32_t* raw_b, const uint32_t* raw_a,
                     uint32_t n_out, const uint32_t* ksk, uint32_t* out) {
  const uint32_t N = d * k;
  if (n_out % k) return 1;
  const uint32_t blocks = n_out / k;
  const uint32_t q0 = m4[0], q1 = m4[1], P1 = m4[2], P2 = m4[3];
  const uint64_t q1inv = powmod(q1 % q0, q0 - 2, q0);
  const uint64_t q0inv1 = powmod(q0 % q1, q1 - 2, q1), p1inv2 = powmod(P1 % P2, P2 - 2, P2);
  const uint64_t Q = (uint64_t)q0 * q1, PP = (uint64_t)P1 * P2;
  uint32_t* U = (uint32_t*)malloc(sizeof(uint32_t) * 4 * N);
  uint32_t* W = (uint32_t*)malloc(sizeof(uint32_t) * 4 * N);
  for (uint32_t Y = 0; Y < blocks; ++Y) {
    memset(U, 0, sizeof(uint32_t) * 4 * N);
    memset(W, 0, sizeof(uint32_t) * 4 * N);
    /* the k components of one block in parallel (thread-private sums, added mod q at the end: the same
       residues in any order) */
#pragma omp parallel
    {
      uint32_t* Ut = (uint32_t*)calloc((size_t)4 * N, sizeof(uint32_t));
      uint32_t* Wt = (uint32_t*)calloc((size_t)4 * N, sizeof(uint32_t));
      int64_t* al = (int64_t*)malloc(sizeof(int64_t) * N);
      uint32_t* dl = (uint32_t*)malloc(sizeof(uint32_t) * N);
      uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * N);
#pragma omp for schedule(dynamic)
      for (uint32_t j = 0; j < k; ++j) {
        for (uint32_t tt = 0; tt < k; ++tt)
          for (uint32_t mm = 0; mm < d; ++mm) {
            const size_t src = ((size_t)Y * k + tt) * N + (size_t)d * j + mm;
            const uint64_t a0 = raw_a[src], a1 = raw_a[(size_t)n_out * N + src];
            const uint64_t x = a0 + (uint64_t)q0 * mulmod((a1 + q1 - a0 % q1) % q1, q0inv1, q1);   /* CRT, [0, Q) */
            al[tt + (size_t)k * mm] = x > Q / 2 ? (int64_t)x - (int64_t)Q : (int64_t)x;
          }
        const uint32_t* K = ksk + (size_t)j * 8 * N;
        for (uint32_t mi = 0; mi < 4; ++mi) {
          const uint32_t q = m4[mi];
          for (uint32_t c = 0; c < N; ++c) dl[c] = modq_i64(al[c], q);
          polymul(dl, K + ((size_t)0 * 4 + mi) * N, N, q, t);
          for (uint32_t c = 0; c < N; ++c) Ut[(size_t)mi * N + c] = (uint32_t)(((uint64_t)Ut[(size_t)mi * N + c] + t[c]) % q);
          polymul(dl, K + ((size_t)1 * 4 + mi) * N, N, q, t);
          for (uint32_t c = 0; c < N; ++c) Wt[(size_t)mi * N + c] = (uint32_t)(((uint64_t)Wt[(size_t)mi * N + c] + t[c]) % q);
        }
      }
#pragma omp critical
      for (uint32_t mi = 0; mi < 4; ++mi)
        for (uint32_t c = 0; c < N; ++c) {
          const size_t i = (size_t)mi * N + c;
          U[i] = (uint32_t)(((uint64_t)U[i] + Ut[i]) % m4[mi]);
          W[i] = (uint32_t)(((uint64_t)W[i] + Wt[i]) % m4[mi]);
        }
      free(Ut);
      free(Wt);
      free(al);
      free(dl);
      free(t);
    }
    for (uint32_t c = 0; c < N; ++c) {
      uint32_t x[2][2];
      for (int part = 0; part < 2; ++part) {
        const uint32_t* V = part ? W : U;
        const uint64_t v1 = V[2 * (size_t)N + c], v2 = V[3 * (size_t)N + c];
        const uint64_t xp = v1 + (uint64_t)P1 * mulmod((v2 + P2 - v1 % P2) % P2, p1inv2, P2);   /* [0, P1 P2) */
        const int64_t xc = xp > PP / 2 ? (int64_t)xp - (int64_t)PP : (int64_t)xp;   /* |xc| <= P1 P2 / 2 < 2^60 */
        for (int L = 0; L < 2; ++L) {
          const uint32_t q = m4[L];
          const uint64_t ppinv = powmod(mulmod(P1 % q, P2 % q, q), q - 2, q);
          uint32_t v = (uint32_t)mulmod(modq_i64((int64_t)V[(size_t)L * N + c] - xc, q), ppinv, q);
          if (part) v = (uint32_t)(((uint64_t)v + raw_b[((size_t)L * blocks + Y) * N + c]) % q);
          x[L][part] = v;
        }
      }
      for (int ab = 0; ab < 2; ++ab) {
        const int64_t x1c = x[1][ab] > q1 / 2 ? (int64_t)x[1][ab] - q1 : (int64_t)x[1][ab];
        out[((size_t)Y * 2 + ab) * N + c] = (uint32_t)mulmod(modq_i64((int64_t)x[0][ab] - x1c, q0), q1inv, q0);
      }
    }
  }
  free(U);
  free(W);
  return 0;
}
/* all k keys of or_mlwe_ksk1 (components in parallel): ksk [k][2][4][N] */
void or_mlwe_ksk1_all(uint64_t seed, const int32_t* s, uint32_t N, uint32_t k, const uint32_t* m4, uint32_t* ksk) {
#pragma omp parallel for schedule(dynamic)
  for (uint32_t j = 0; j < k; ++j) or_mlwe_ksk1(seed, j, s, N, k, m4, ksk + (size_t)j * 8 * N);
}

/* ================================================================== slot-domain BSGS PCMM
 * hesim pcmm_bsgs (matmul.py:165-176) on real CKKS ciphertexts: the input matrix sits row-major in the
 * slots (tiled), a left slot rotation by r is the automorphism X -> X^(5^r) followed by a hybrid key
 * switch (dnum 2, special prime P) from sigma(s) back to s.  Integer algorithm (the CUDA path is
 * bit-exact with it):
 *   D = digits of ct.a (RNS digits d_i = a_i Qhat_i^-1 mod q_i, lifted to q0, q1, P)      -- once (hoisting)
 *   baby_i = (KS_{5^(i d)}(sigma(D)), sigma(ct.b) + ...)  i = 1 .. b-1;  baby_0 = ct
 *   inner_j = sum_i pt_{i + j b} * baby_i                                        (level 1, scale Delta q1)
 *   partial_j = inner_j (j = 0) or its rotation by j b d (digits of inner_j.a, then the same key switch)
 *   out = rescale_q1(sum_j partial_j)                                            (level 0, scale Delta)
 * where KS_g(sigma(D)) = ModDown(sum_i sigma_g(D_i) * ksk_g[i])  (sigma applied to the lifted digits).
 */
/* Gadget hybrid key (the slot rotations): each RNS digit d_i is further split into SD = 2 sub-digits of
 * SW = 15 bits (d_i = lo + 2^15 hi), so the key-switching noise sum_t d_t e_t / P is ~2^15 smaller than with
 * the plain dnum-2 key -- needed because the baby rotations act on the input at scale Delta = 2^26.
 *   ksk[t = i SD + h][0][j] = alpha,  ksk[t][1][j] = -alpha s_new + g_{t,j} s_old + e_t,
 *   g_{t,j} = P Qhat_i 2^(15 h) mod q_j for j == i, else 0.   Layout [t][part][j][n], t < 4. */
#define SD 2
#define SW 15
void or_ksk_gen_gadget(uint64_t seed, uint32_t id, const int32_t* s_old, const int32_t* s_new, uint32_t n,
                       const uint32_t* m, uint32_t* ksk) {
  int32_t* e = (int32_t*)malloc(sizeof(int32_t) * n);
  uint32_t* as = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t t = 0; t < 2 * SD; ++t) {
    const uint32_t i = t / SD, h = t % SD;
    or_sample_cbd(seed, STREAM_KSK_E(id, t), e, n);
    for (uint32_t j = 0; j < 3; ++j) {
      const uint32_t q = m[j];
      uint32_t* alpha = ksk + ((size_t)(t * 2 + 0) * 3 + j) * n;
      uint32_t* beta = ksk + ((size_t)(t * 2 + 1) * 3 + j) * n;
      or_sample_uniform(seed, STREAM_KSK_A(id, t, j), q, alpha, n);
      or_negacyclic_mul(alpha, s_new, n, q, as);
      uint64_t g = 0;
      if (j == i) g = mulmod(mulmod(m[2] % q, m[1 - i] % q, q), powmod(2, (uint64_t)SW * h, q), q);
      for (uint32_t c = 0; c < n; ++c) {
        uint64_t v = (uint64_t)(q - as[c]) + modq_i64(e[c], q) + mulmod(g, modq_i64(s_old[c], q), q);
        beta[c] = (uint32_t)(v % q);
      }
    }
  }
  free(e);
  free(as);
}
void or_rotation_ksk(uint64_t seed, uint32_t r, const int32_t* s, uint32_t N, const uint32_t* m, uint32_t* ksk) {
  uint64_t g = 1;
  for (uint32_t t = 0; t < r % (N / 2); ++t) g = g * 5 % (2ull * N);
  int32_t* ss = (int32_t*)malloc(sizeof(int32_t) * N);
  for (uint32_t i = 0; i < N; ++i) {
    uint64_t j = ((uint64_t)i * g) % (2ull * N);
    if (j < N) ss[j] = s[i];
    else ss[j - N] = -s[i];
  }
  or_ksk_gen_gadget(seed, 0x10000 + r, ss, s, N, m, ksk);
  free(ss);
}
/* plain (dnum-2 hybrid) rotation key sigma_{5^r}(s) -> s, layout [i < 2][part][mod][N] */
void or_rotation_ksk_plain(uint64_t seed, uint32_t r, const int32_t* s, uint32_t N, const uint32_t* m, uint32_t* ksk) {
  uint64_t g = 1;
  for (uint32_t t = 0; t < r % (N / 2); ++t) g = g * 5 % (2ull * N);
  int32_t* ss = (int32_t*)malloc(sizeof(int32_t) * N);
  for (uint32_t i = 0; i < N; ++i) {
    uint64_t j = ((uint64_t)i * g) % (2ull * N);
    if (j < N) ss[j] = s[i];
    else ss[j - N] = -s[i];
  }
  or_ksk_gen(seed, 0x30000 + r, ss, s, N, m, ksk);
  free(ss);
}
/* gadget digits D [3 mod][t < 4][n] of the a-part c [2 limbs][n]: sub-digits of d_i (< 2^15, so the
 * same value under every modulus) */
static void ks_digits(const uint32_t* c, uint32_t n, const uint32_t* m, uint32_t* D) {
  for (int i = 0; i < 2; ++i) {
    const uint32_t qi = m[i];
    const uint64_t inv = powmod(m[1 - i] % qi, qi - 2, qi);
    for (uint32_t k = 0; k < n; ++k) {
      const uint32_t dg = (uint32_t)mulmod(c[(size_t)i * n + k], inv, qi);
      for (int h = 0; h < SD; ++h) {
        const uint32_t sd = (dg >> (SW * h)) & ((1u << SW) - 1u);
        for (int j = 0; j < 3; ++j) D[((size_t)j * 2 * SD + i * SD + h) * n + k] = sd % m[j];
      }
    }
  }
}
/* (u, w) = ModDown(sum_t sigma_g(D_t) ksk[t])  [2 limbs][n] each */
static void ks_from_digits(const uint32_t* D, uint32_t n, uint64_t g, const uint32_t* ksk, const uint32_t* m,
                           uint32_t* u, uint32_t* w) {
  uint32_t* U = (uint32_t*)calloc((size_t)3 * n, sizeof(uint32_t));
  uint32_t* W = (uint32_t*)calloc((size_t)3 * n, sizeof(uint32_t));
  uint32_t* sd = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 2 * SD; ++i) {
      or_automorphism(D + ((size_t)j * 2 * SD + i) * n, n, (uint32_t)g, m[j], sd);
      polymul(sd, ksk + ((size_t)(i * 2 + 0) * 3 + j) * n, n, m[j], t);
      for (uint32_t k = 0; k < n; ++k) U[(size_t)j * n + k] = (uint32_t)(((uint64_t)U[(size_t)j * n + k] + t[k]) % m[j]);
      polymul(sd, ksk + ((size_t)(i * 2 + 1) * 3 + j) * n, n, m[j], t);
      for (uint32_t k = 0; k < n; ++k) W[(size_t)j * n + k] = (uint32_t)(((uint64_t)W[(size_t)j * n + k] + t[k]) % m[j]);
    }
  ks_moddown(U, W, n, m, u, w);
  free(U);
  free(W);
  free(sd);
  free(t);
}
/* rotate ct [2 limbs][2][n] given the lifted digits of its a-part */
static void rotate_with_digits(const uint32_t* ct, const uint32_t* D, uint32_t n, uint32_t r, const uint32_t* ksk,
                               const uint32_t* m, uint32_t* out) {
  uint64_t g = 1;
  for (uint32_t t = 0; t < r % (n / 2); ++t) g = g * 5 % (2ull * n);
  uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  uint32_t* sb = (uint32_t*)malloc(sizeof(uint32_t) * n);
  ks_from_digits(D, n, g, ksk, m, u, w);
  for (int L = 0; L < 2; ++L) {
    or_automorphism(ct + ((size_t)L * 2 + 1) * n, n, (uint32_t)g, m[L], sb);
    for (uint32_t k = 0; k < n; ++k) {
      out[((size_t)L * 2 + 0) * n + k] = u[(size_t)L * n + k];
      out[((size_t)L * 2 + 1) * n + k] = (uint32_t)(((uint64_t)sb[k] + w[(size_t)L * n + k]) % m[L]);
    }
  }
  free(u);
  free(w);
  free(sb);
}
/*
 * BSGS slot linear map with stride d (d = block dim for the PCMM, 1 for SlotToCoeffs):
 * ct_in [2][2][N] level 1; pts [b g][2 limbs][N] coefficient form mod q_L (term k = i + j b);
 * keys_baby [b-1][4][2][3][N] (gadget keys) for steps i d, keys_giant [g-1][..] for steps j b d; out [2][N].
 */
int or_slot_bsgs(uint32_t N, const uint32_t* m, uint32_t d, uint32_t b, uint32_t g, const uint32_t* ct_in,
                 const uint32_t* pts, const uint32_t* keys_baby, const uint32_t* keys_giant, uint32_t* out) {
  if ((uint64_t)b * g * d > N / 2) return 1;
  const size_t cw = (size_t)4 * N;
  uint32_t* D = (uint32_t*)malloc(sizeof(uint32_t) * 6 * SD * N);
  uint32_t* a_in = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  for (int L = 0; L < 2; ++L) memcpy(a_in + (size_t)L * N, ct_in + ((size_t)L * 2 + 0) * N, sizeof(uint32_t) * N);
  ks_digits(a_in, N, m, D);
  uint32_t* baby = (uint32_t*)malloc(sizeof(uint32_t) * cw * b);
  memcpy(baby, ct_in, sizeof(uint32_t) * cw);
  for (uint32_t i = 1; i < b; ++i) rotate_with_digits(ct_in, D, N, i * d, keys_baby + (size_t)(i - 1) * 24 * N, m, baby + i * cw);
  uint32_t* acc = (uint32_t*)calloc(cw, sizeof(uint32_t));
  uint32_t* inner = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* rot = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (uint32_t j = 0; j < g; ++j) {
    memset(inner, 0, sizeof(uint32_t) * cw);
    for (uint32_t i = 0; i < b; ++i)
      for (int L = 0; L < 2; ++L)
        for (int ab = 0; ab < 2; ++ab) {
          polymul(baby + i * cw + ((size_t)L * 2 + ab) * N, pts + ((size_t)(i + j * b) * 2 + L) * N, N, m[L], t);
          uint32_t* dst = inner + ((size_t)L * 2 + ab) * N;
          for (uint32_t k = 0; k < N; ++k) dst[k] = (uint32_t)(((uint64_t)dst[k] + t[k]) % m[L]);
        }
    const uint32_t* part = inner;
    if (j > 0) {
      for (int L = 0; L < 2; ++L) memcpy(a_in + (size_t)L * N, inner + ((size_t)L * 2 + 0) * N, sizeof(uint32_t) * N);
      ks_digits(a_in, N, m, D);
      rotate_with_digits(inner, D, N, j * b * d, keys_giant + (size_t)(j - 1) * 24 * N, m, rot);
      part = rot;
    }
    for (int L = 0; L < 2; ++L)
      for (size_t k = 0; k < (size_t)2 * N; ++k) {
        const size_t x = (size_t)L * 2 * N + k;
        acc[x] = (uint32_t)(((uint64_t)acc[x] + part[x]) % m[L]);
      }
  }
  const uint32_t q0 = m[0], q1 = m[1];
  const uint64_t q1inv = powmod(q1 % q0, q0 - 2, q0);
  for (int ab = 0; ab < 2; ++ab)
    for (uint32_t k = 0; k < N; ++k) {
      const uint32_t x0 = acc[(size_t)ab * N + k], x1 = acc[((size_t)2 + ab) * N + k];
      const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - q1 : (int64_t)x1;
      out[(size_t)ab * N + k] = (uint32_t)mulmod(modq_i64((int64_t)x0 - x1c, q0), q1inv, q0);
    }
  free(D);
  free(a_in);
  free(baby);
  free(acc);
  free(inner);
  free(rot);
  free(t);
  return 0;
}

/*
 * The same map with lazy ModDown (hoisted BSGS, baby rotations kept in the PQ basis): baby_i = (U, P sigma(b) + W)
 * mod (q0, q1, P) straight from the key MAC (baby_0 = P ct), the products taken mod q0, q1 and P, and one
 * ModDown per giant group sum -- so the baby rotations' rounding noise is never multiplied by the
 * plaintexts.  pts [b g][3 moduli][N] coefficient form.  Then giant rotations, sum, rescale as above.
 */
int or_slot_bsgs_lazy(uint32_t N, const uint32_t* m, uint32_t d, uint32_t b, uint32_t g, const uint32_t* ct_in,
                      const uint32_t* pts, const uint32_t* keys_baby, const uint32_t* keys_giant, int plain_giant,
                      uint32_t* out) {
  if ((uint64_t)b * g * d > N / 2) return 1;
  const size_t cw = (size_t)4 * N, bw = (size_t)6 * N;   /* Q ct [2][2][N]; PQ ct [3][2][N] */
  const uint32_t P = m[2];
  uint32_t* D = (uint32_t*)malloc(sizeof(uint32_t) * 6 * SD * N);
  uint32_t* a_in = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  for (int L = 0; L < 2; ++L) memcpy(a_in + (size_t)L * N, ct_in + ((size_t)L * 2 + 0) * N, sizeof(uint32_t) * N);
  ks_digits(a_in, N, m, D);
  uint32_t* baby = (uint32_t*)calloc(bw * b, sizeof(uint32_t));
  uint32_t* U = (uint32_t*)malloc(sizeof(uint32_t) * 3 * N);
  uint32_t* W = (uint32_t*)malloc(sizeof(uint32_t) * 3 * N);
  uint32_t* sd = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * N);
  for (int L = 0; L < 2; ++L)
    for (int ab = 0; ab < 2; ++ab)
      for (uint32_t k = 0; k < N; ++k)
        baby[((size_t)L * 2 + ab) * N + k] = (uint32_t)mulmod(ct_in[((size_t)L * 2 + ab) * N + k], P % m[L], m[L]);
  for (uint32_t i = 1; i < b; ++i) {
    uint64_t gal = 1;
    for (uint64_t e = 0; e < ((uint64_t)i * d) % (N / 2); ++e) gal = gal * 5 % (2ull * N);
    const uint32_t* ksk = keys_baby + (size_t)(i - 1) * 24 * N;
    memset(U, 0, sizeof(uint32_t) * 3 * N);
    memset(W, 0, sizeof(uint32_t) * 3 * N);
    for (int j = 0; j < 3; ++j)
      for (int x = 0; x < 2 * SD; ++x) {
        or_automorphism(D + ((size_t)j * 2 * SD + x) * N, N, (uint32_t)gal, m[j], sd);
        polymul(sd, ksk + ((size_t)(x * 2 + 0) * 3 + j) * N, N, m[j], t);
        for (uint32_t k = 0; k < N; ++k) U[(size_t)j * N + k] = (uint32_t)(((uint64_t)U[(size_t)j * N + k] + t[k]) % m[j]);
        polymul(sd, ksk + ((size_t)(x * 2 + 1) * 3 + j) * N, N, m[j], t);
        for (uint32_t k = 0; k < N; ++k) W[(size_t)j * N + k] = (uint32_t)(((uint64_t)W[(size_t)j * N + k] + t[k]) % m[j]);
      }
    uint32_t* bi = baby + i * bw;
    for (int j = 0; j < 3; ++j) {
      if (j < 2) or_automorphism(ct_in + ((size_t)j * 2 + 1) * N, N, (uint32_t)gal, m[j], sd);
      for (uint32_t k = 0; k < N; ++k) {
        bi[((size_t)j * 2 + 0) * N + k] = U[(size_t)j * N + k];
        const uint64_t pb = j < 2 ? mulmod(sd[k], P % m[j], m[j]) : 0;
        bi[((size_t)j * 2 + 1) * N + k] = (uint32_t)((pb + W[(size_t)j * N + k]) % m[j]);
      }
    }
  }
  uint32_t* acc = (uint32_t*)calloc(cw, sizeof(uint32_t));
  uint32_t* inner = (uint32_t*)malloc(sizeof(uint32_t) * bw);
  uint32_t* innerq = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* rot = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* XA = (uint32_t*)malloc(sizeof(uint32_t) * 3 * N);
  uint32_t* XB = (uint32_t*)malloc(sizeof(uint32_t) * 3 * N);
  uint32_t* xa = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  uint32_t* xb = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  for (uint32_t j = 0; j < g; ++j) {
    memset(inner, 0, sizeof(uint32_t) * bw);
    for (uint32_t i = 0; i < b; ++i)
      for (int L = 0; L < 3; ++L)
        for (int ab = 0; ab < 2; ++ab) {
          polymul(baby + i * bw + ((size_t)L * 2 + ab) * N, pts + ((size_t)(i + j * b) * 3 + L) * N, N, m[L], t);
          uint32_t* dst = inner + ((size_t)L * 2 + ab) * N;
          for (uint32_t k = 0; k < N; ++k) dst[k] = (uint32_t)(((uint64_t)dst[k] + t[k]) % m[L]);
        }
    for (int L = 0; L < 3; ++L) {   /* [mod][n] views of the a and b parts for ks_moddown */
      memcpy(XA + (size_t)L * N, inner + ((size_t)L * 2 + 0) * N, sizeof(uint32_t) * N);
      memcpy(XB + (size_t)L * N, inner + ((size_t)L * 2 + 1) * N, sizeof(uint32_t) * N);
    }
    ks_moddown(XA, XB, N, m, xa, xb);
    for (int L = 0; L < 2; ++L) {
      memcpy(innerq + ((size_t)L * 2 + 0) * N, xa + (size_t)L * N, sizeof(uint32_t) * N);
      memcpy(innerq + ((size_t)L * 2 + 1) * N, xb + (size_t)L * N, sizeof(uint32_t) * N);
    }
    const uint32_t* part = innerq;
    if (j > 0 && plain_giant) {
      /* plain dnum-2 key (its noise lands at scale Delta q1): digits d_i of a, lifted into every modulus,
       * then sigma on the lifted digits (as the device does in the NTT domain), MAC, ModDown */
      uint64_t gal = 1;
      for (uint64_t e = 0; e < ((uint64_t)j * b * d) % (N / 2); ++e) gal = gal * 5 % (2ull * N);
      const uint32_t* ksk = keys_giant + (size_t)(j - 1) * 12 * N;
      memset(U, 0, sizeof(uint32_t) * 3 * N);
      memset(W, 0, sizeof(uint32_t) * 3 * N);
      for (int i = 0; i < 2; ++i) {
        const uint32_t qi = m[i];
        const uint64_t inv = powmod(m[1 - i] % qi, qi - 2, qi);
        for (int jm = 0; jm < 3; ++jm) {
          for (uint32_t k = 0; k < N; ++k)
            t[k] = (uint32_t)(mulmod(innerq[((size_t)i * 2 + 0) * N + k], inv, qi) % m[jm]);
          or_automorphism(t, N, (uint32_t)gal, m[jm], sd);
          polymul(sd, ksk + ((size_t)(i * 2 + 0) * 3 + jm) * N, N, m[jm], t);
          for (uint32_t k = 0; k < N; ++k) U[(size_t)jm * N + k] = (uint32_t)(((uint64_t)U[(size_t)jm * N + k] + t[k]) % m[jm]);
          for (uint32_t k = 0; k < N; ++k)
            t[k] = (uint32_t)(mulmod(innerq[((size_t)i * 2 + 0) * N + k], inv, qi) % m[jm]);
          or_automorphism(t, N, (uint32_t)gal, m[jm], sd);
          polymul(sd, ksk + ((size_t)(i * 2 + 1) * 3 + jm) * N, N, m[jm], t);
          for (uint32_t k = 0; k < N; ++k) W[(size_t)jm * N + k] = (uint32_t)(((uint64_t)W[(size_t)jm * N + k] + t[k]) % m[jm]);
        }
      }
      ks_moddown(U, W, N, m, xa, xb);
      for (int L = 0; L < 2; ++L) {
        or_automorphism(innerq + ((size_t)L * 2 + 1) * N, N, (uint32_t)gal, m[L], sd);
        for (uint32_t k = 0; k < N; ++k) {
          rot[((size_t)L * 2 + 0) * N + k] = xa[(size_t)L * N + k];
          rot[((size_t)L * 2 + 1) * N + k] = (uint32_t)(((uint64_t)sd[k] + xb[(size_t)L * N + k]) % m[L]);
        }
      }
      part = rot;
    } else if (j > 0) {
      for (int L = 0; L < 2; ++L) memcpy(a_in + (size_t)L * N, innerq + ((size_t)L * 2 + 0) * N, sizeof(uint32_t) * N);
      ks_digits(a_in, N, m, D);
      rotate_with_digits(innerq, D, N, j * b * d, keys_giant + (size_t)(j - 1) * 24 * N, m, rot);
      part = rot;
    }
    for (int L = 0; L < 2; ++L)
      for (size_t k = 0; k < (size_t)2 * N; ++k) {
        const size_t x = (size_t)L * 2 * N + k;
        acc[x] = (uint32_t)(((uint64_t)acc[x] + part[x]) % m[L]);
      }
  }
  const uint32_t q0 = m[0], q1 = m[1];
  const uint64_t q1inv = powmod(q1 % q0, q0 - 2, q0);
  for (int ab = 0; ab < 2; ++ab)
    for (uint32_t k = 0; k < N; ++k) {
      const uint32_t x0 = acc[(size_t)ab * N + k], x1 = acc[((size_t)2 + ab) * N + k];
      const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - q1 : (int64_t)x1;
      out[(size_t)ab * N + k] = (uint32_t)mulmod(modq_i64((int64_t)x0 - x1c, q0), q1inv, q0);
    }
  free(D); free(a_in); free(baby); free(U); free(W); free(sd); free(t); free(acc); free(inner); free(innerq);
  free(rot); free(XA); free(XB); free(xa); free(xb);
  return 0;
}

/* hesim pcmm_bsgs (matmul.py:165-176): the BSGS map with stride d over the d blocks */
int or_slot_pcmm(uint32_t N, const uint32_t* m, uint32_t d, uint32_t b, uint32_t g, const uint32_t* ct_in,
                 const uint32_t* pts, const uint32_t* keys_baby, const uint32_t* keys_giant, uint32_t* out) {
  if (b * g != d) return 1;
  return or_slot_bsgs(N, m, d, b, g, ct_in, pts, keys_baby, keys_giant, out);
}
