/*
 * he_oracle_pcmv.c -- CPU restatement of the Rhombus PCMv with Rhombus's input/output-packing
 * split point (TEST INFRASTRUCTURE ONLY; never linked into the product library).
 *
 * PARITY UNPINNED at the integer level (same status as he_oracle_rhombus.c): the paper names the
 * algorithm ([rhombus]) and its multi-GPU split but ships no code.
 * This file restates, in exact modular arithmetic, the windowed form the CUDA path runs:
 *
 *  Input layout (window w = n / 2^s, s = the split point): element e of the n_in-vector sits in
 *  input piece p = e / w at piece coefficient h_w(e mod w) < w, i.e. degree-N coefficient
 *  p + rho h_w(e mod w) (h_w: fix the top bit, reverse the others -- PAPER.md:676-680's h at w = n).
 *  Because every piece's values live in its low w coefficients, one plaintext x ciphertext product
 *  yields U = n / w inner products without interference (input packing):
 *     pt_{o,j,p}(X) = w^-1 sum_{u<U} X^{u w} sum_{i<w} W~[r(o,j,u)][w p + i] X^{-h_w(i)}
 *  puts <row r(o,j,u), piece p> at coefficient u w of pt * piece_p; r(o,j,u) = n o + h_n(u w + j).
 *  Output packing: PackLWEs (CDKS21) over the w leaves j of output piece o with valid data at the
 *  multiples of w -- log2 w levels  E + X^{n/2^l'} O + sigma_{2^l'+1}(E - X^{n/2^l'} O),
 *  l' = s+1 .. log2 n (the top log2 w Galois keys of the s = 0 packing), garbage at non-multiples
 *  is cancelled level by level.  Leaf j lands at position j, slot u at u w + j, so row r ends at
 *  h_n(r mod n): the same output layout as s = 0.  Key switches per output piece: w - 1 instead of
 *  n - 1; pt x ct products: unchanged (n_out n_in / n).
 *  (D) decompose and (R)(C) rescale / compose are those of he_oracle_rhombus.c.
 *
 * Column shards ("the ciphertext is masked and each GPU is assigned 4096/8 values"):
 * a plan over columns [w piece0, ..) of W runs on input pieces piece0.. and returns its level-1
 * composed output; the shards' outputs are summed mod q_i and rescaled once.
 *
 * Polynomial products use a negacyclic NTT with cached tables and Shoup multiplication (products
 * mod q are unique, so the words equal any other exact method: tests check this file against
 * or_rhombus_pcmv, the schoolbook-checked restatement, at s = 0).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

uint32_t or_half_reverse(uint32_t x, uint32_t n);
void or_automorphism(const uint32_t* p, uint32_t n, uint32_t k, uint32_t q, uint32_t* out);

static inline uint64_t mulmod_p(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
static uint64_t powmod_p(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod_p(r, a, q);
    a = mulmod_p(a, a, q);
    e >>= 1;
  }
  return r;
}
static inline uint32_t modq_s(int64_t v, uint32_t q) {
  int64_t r = v % (int64_t)q;
  return (uint32_t)(r < 0 ? r + q : r);
}
static int lg2(uint32_t x) {
  int l = 0;
  while ((1u << l) < x) ++l;
  return l;
}
static uint32_t rev_bits(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int t = 0; t < bits; ++t) r |= ((x >> t) & 1u) << (bits - 1 - t);
  return r;
}

/* ------------------------------------------------------------------ cached negacyclic NTT */
typedef struct {
  uint32_t n, q;
  uint32_t *fw, *fwp, *iv, *ivp;
  uint32_t ninv, ninvp;
} fntt_t;

static fntt_t g_tabs[32];
static int g_ntabs = 0;

static inline uint32_t shoup_pre32(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
static inline uint32_t shoup_mul32(uint32_t x, uint32_t w, uint32_t wp, uint32_t q) {
  const uint32_t hi = (uint32_t)(((uint64_t)x * wp) >> 32);
  uint32_t r = x * w - hi * q; /* exact mod 2^32, r in [0, 2q) */
  return r >= q ? r - q : r;
}

static const fntt_t* fntt_get(uint32_t n, uint32_t q) {
  const fntt_t* found = NULL;
#pragma omp critical(or_fntt_cache)
  {
    for (int i = 0; i < g_ntabs; ++i)
      if (g_tabs[i].n == n && g_tabs[i].q == q) found = &g_tabs[i];
    if (!found && g_ntabs < 32) {
      fntt_t* t = &g_tabs[g_ntabs];
      uint64_t psi = 0;
      for (uint64_t g = 2; g < q; ++g) {
        const uint64_t c = powmod_p(g, (q - 1) / (2ull * n), q);
        if (powmod_p(c, n, q) == q - 1) {
          psi = c;
          break;
        }
      }
      const uint64_t psii = powmod_p(psi, q - 2, q);
      const int l = lg2(n);
      t->fw = (uint32_t*)malloc(sizeof(uint32_t) * n);
      t->fwp = (uint32_t*)malloc(sizeof(uint32_t) * n);
      t->iv = (uint32_t*)malloc(sizeof(uint32_t) * n);
      t->ivp = (uint32_t*)malloc(sizeof(uint32_t) * n);
      uint64_t p = 1, pi = 1;
      uint32_t* pw = (uint32_t*)malloc(sizeof(uint32_t) * n);
      uint32_t* pwi = (uint32_t*)malloc(sizeof(uint32_t) * n);
      for (uint32_t i = 0; i < n; ++i) {
        pw[i] = (uint32_t)p;
        pwi[i] = (uint32_t)pi;
        p = mulmod_p(p, psi, q);
        pi = mulmod_p(pi, psii, q);
      }
      for (uint32_t i = 0; i < n; ++i) {
        t->fw[i] = pw[rev_bits(i, l)];
        t->iv[i] = pwi[rev_bits(i, l)];
        t->fwp[i] = shoup_pre32(t->fw[i], q);
        t->ivp[i] = shoup_pre32(t->iv[i], q);
      }
      free(pw);
      free(pwi);
      t->ninv = (uint32_t)powmod_p(n, q - 2, q);
      t->ninvp = shoup_pre32(t->ninv, q);
      t->n = n;
      t->q = q;
      ++g_ntabs;
      found = t;
    }
  }
  return found;
}

/* Cooley-Tukey, natural order in, bit-reversed out; values in [0, q) */
static void fntt_fwd(const fntt_t* T, uint32_t* a) {
  const uint32_t n = T->n, q = T->q;
  uint32_t t = n;
  for (uint32_t m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t j1 = 2 * i * t, S = T->fw[m + i], Sp = T->fwp[m + i];
      for (uint32_t j = j1; j < j1 + t; ++j) {
        const uint32_t U = a[j], V = shoup_mul32(a[j + t], S, Sp, q);
        const uint32_t s = U + V;
        a[j] = s >= q ? s - q : s;
        a[j + t] = U >= V ? U - V : U + q - V;
      }
    }
  }
}
/* Gentleman-Sande, bit-reversed in, natural out, scaled by n^-1 */
static void fntt_inv(const fntt_t* T, uint32_t* a) {
  const uint32_t n = T->n, q = T->q;
  uint32_t t = 1;
  for (uint32_t m = n; m > 1; m >>= 1) {
    const uint32_t h = m >> 1;
    uint32_t j1 = 0;
    for (uint32_t i = 0; i < h; ++i) {
      const uint32_t S = T->iv[h + i], Sp = T->ivp[h + i];
      for (uint32_t j = j1; j < j1 + t; ++j) {
        const uint32_t U = a[j], V = a[j + t];
        const uint32_t s = U + V;
        a[j] = s >= q ? s - q : s;
        a[j + t] = shoup_mul32(U >= V ? U - V : U + q - V, S, Sp, q);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (uint32_t j = 0; j < n; ++j) a[j] = shoup_mul32(a[j], T->ninv, T->ninvp, q);
}

/* ------------------------------------------------------------------ hybrid key switching (NTT keys) */
/* NTT of a coefficient-form key [2 digits][2 parts][3 moduli][deg] (he_oracle_rhombus.c or_ksk_gen) */
static uint32_t* ksk_ntt(const uint32_t* ksk, uint32_t deg, const uint32_t* m) {
  uint32_t* K = (uint32_t*)malloc(sizeof(uint32_t) * 12 * deg);
  memcpy(K, ksk, sizeof(uint32_t) * 12 * deg);
  for (int i = 0; i < 2; ++i)
    for (int part = 0; part < 2; ++part)
      for (int j = 0; j < 3; ++j) fntt_fwd(fntt_get(deg, m[j]), K + ((size_t)(i * 2 + part) * 3 + j) * deg);
  return K;
}

/* (u, w) [2 limbs][deg] with w + u s_new = c s_old + small: digits d_i = c_i Qhat_i^-1 mod q_i lifted to
 * q0, q1, P, U_j = sum_i d_i alpha_{i,j}, W_j = sum_i d_i beta_{i,j}, ModDown by P with a centred P part
 * (he_oracle_rhombus.c ks_accumulate / ks_moddown, here with NTT-domain keys) */
static void ks_fast(const uint32_t* c, const uint32_t* KN, uint32_t deg, const uint32_t* m, uint32_t* u, uint32_t* w) {
  uint32_t* d = (uint32_t*)malloc(sizeof(uint32_t) * 2 * deg);
  uint32_t* dl = (uint32_t*)malloc(sizeof(uint32_t) * deg);
  uint32_t* U = (uint32_t*)calloc((size_t)3 * deg, sizeof(uint32_t));
  uint32_t* W = (uint32_t*)calloc((size_t)3 * deg, sizeof(uint32_t));
  for (int i = 0; i < 2; ++i) {
    const uint32_t qi = m[i];
    const uint64_t inv = powmod_p(m[1 - i] % qi, qi - 2, qi);
    for (uint32_t k = 0; k < deg; ++k) d[(size_t)i * deg + k] = (uint32_t)mulmod_p(c[(size_t)i * deg + k], inv, qi);
  }
  for (int j = 0; j < 3; ++j) {
    const uint32_t q = m[j];
    const fntt_t* T = fntt_get(deg, q);
    uint32_t* Uj = U + (size_t)j * deg;
    uint32_t* Wj = W + (size_t)j * deg;
    for (int i = 0; i < 2; ++i) {
      for (uint32_t k = 0; k < deg; ++k) dl[k] = d[(size_t)i * deg + k] % q;
      fntt_fwd(T, dl);
      const uint32_t* ka = KN + ((size_t)(i * 2 + 0) * 3 + j) * deg;
      const uint32_t* kb = KN + ((size_t)(i * 2 + 1) * 3 + j) * deg;
      for (uint32_t k = 0; k < deg; ++k) {
        Uj[k] = (uint32_t)(((uint64_t)Uj[k] + (uint64_t)dl[k] * ka[k] % q) % q);
        Wj[k] = (uint32_t)(((uint64_t)Wj[k] + (uint64_t)dl[k] * kb[k] % q) % q);
      }
    }
    fntt_inv(T, Uj);
    fntt_inv(T, Wj);
  }
  const uint32_t P = m[2];
  for (int j = 0; j < 2; ++j) {
    const uint32_t q = m[j];
    const uint64_t pinv = powmod_p(P % q, q - 2, q);
    for (uint32_t k = 0; k < deg; ++k) {
      int64_t up = U[2 * (size_t)deg + k], wp = W[2 * (size_t)deg + k];
      if (up > P / 2) up -= P;
      if (wp > P / 2) wp -= P;
      u[(size_t)j * deg + k] = (uint32_t)mulmod_p(modq_s((int64_t)U[(size_t)j * deg + k] - up, q), pinv, q);
      w[(size_t)j * deg + k] = (uint32_t)mulmod_p(modq_s((int64_t)W[(size_t)j * deg + k] - wp, q), pinv, q);
    }
  }
  free(d);
  free(dl);
  free(U);
  free(W);
}

/* h_w over log2(w) bits (w >= 1 a power of two) */
uint32_t or_window_reverse(uint32_t x, uint32_t w) { return w < 2 ? 0 : or_half_reverse(x, w); }

/* input layout with window w: element e at p + rho h_w(e mod w), p = e / w */
void or_encode_vector_w(const double* v, uint32_t n_vals, uint32_t N, uint32_t n, uint32_t win, double delta,
                        int64_t* pt) {
  const uint32_t rho = N / n;
  memset(pt, 0, sizeof(int64_t) * N);
  for (uint32_t e = 0; e < n_vals; ++e) {
    const uint32_t p = e / win, k = or_window_reverse(e % win, win);
    pt[p + (size_t)rho * k] = llrint(delta * v[e]);
  }
}

/* X^e * p, 0 <= e < n */
static void mono_mul(const uint32_t* p, uint32_t n, uint32_t e, uint32_t q, uint32_t* out) {
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t j = i + e;
    if (j < n) out[j] = p[i];
    else out[j - n] = p[i] ? q - p[i] : 0;
  }
}

/* one PackLWEs combine at degree n: out = E + X^e O + sigma_k(E - X^e O) (sigma followed by the
 * Galois key switch with NTT-domain key KN);  cts [limb][ab][n] */
static void pack_combine(const uint32_t* E, const uint32_t* O, uint32_t n, uint32_t e, uint32_t k, const uint32_t* KN,
                         const uint32_t* m, uint32_t* out) {
  const size_t cw = (size_t)4 * n;
  uint32_t* MO = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* T = (uint32_t*)malloc(sizeof(uint32_t) * cw);
  uint32_t* sa = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  uint32_t* sb = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * 2 * n);
  for (int L = 0; L < 2; ++L)
    for (int ab = 0; ab < 2; ++ab) {
      const size_t o = ((size_t)L * 2 + ab) * n;
      mono_mul(O + o, n, e, m[L], MO + o);
      for (uint32_t i = 0; i < n; ++i) T[o + i] = (uint32_t)(((uint64_t)E[o + i] + m[L] - MO[o + i]) % m[L]);
    }
  for (int L = 0; L < 2; ++L) or_automorphism(T + (size_t)L * 2 * n, n, k, m[L], sa + (size_t)L * n);
  ks_fast(sa, KN, n, m, u, w);
  for (int L = 0; L < 2; ++L) {
    const uint32_t q = m[L];
    or_automorphism(T + ((size_t)L * 2 + 1) * n, n, k, q, sb);
    for (uint32_t i = 0; i < n; ++i) {
      const size_t oa = (size_t)L * 2 * n + i, ob = oa + n;
      out[oa] = (uint32_t)(((uint64_t)E[oa] + MO[oa] + u[(size_t)L * n + i]) % q);
      out[ob] = (uint32_t)(((uint64_t)E[ob] + MO[ob] + sb[i] + w[(size_t)L * n + i]) % q);
    }
  }
  free(MO);
  free(T);
  free(sa);
  free(sb);
  free(u);
  free(w);
}

/*
 * Windowed Rhombus PCMv.
 *   ct_in   [2 limbs][2][N] level-1 input under s (layout of or_encode_vector_w with the same window)
 *   ksk_dec [2][2][3][N]    key s -> s'(X^rho), coefficient form (or_ksk_gen)
 *   gal     [log2 n][2][2][3][n] Galois keys sigma_{2^l+1}(s') -> s', coefficient form (or_galois_ksk)
 *   Wt      int64 [n_out][n_in]  W~ = round(q1 W) of this plan's columns (input pieces piece0 ..)
 *   level1 = 0: out [2 (a, b)][N] level 0 under s'(X^rho);  level1 = 1: out [2 limbs][2][N], no rescale
 *   (a column shard's partial, summed by or_rhombus_combine).
 */
int or_rhombus_pcmv_w(uint32_t N, uint32_t n, uint32_t win, const uint32_t* m, const uint32_t* ct_in,
                      const uint32_t* ksk_dec, const uint32_t* gal, const int64_t* Wt, uint32_t n_out, uint32_t n_in,
                      uint32_t piece0, int level1, uint32_t* out) {
  const uint32_t rho = N / n, U = n / win;
  const uint32_t p_in = (n_in + win - 1) / win, p_out = (n_out + n - 1) / n;
  const int logn = lg2(n), s = lg2(U);
  const size_t cw = (size_t)4 * n;
  if (win == 0 || n % win || piece0 + p_in > rho || p_out > rho) return -1;
  /* (D) key switch the a part to s'(X^rho) at degree N, then the X^rho split */
  uint32_t* KD = ksk_ntt(ksk_dec, N, m);
  uint32_t* a_in = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  uint32_t* u = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  for (int L = 0; L < 2; ++L) memcpy(a_in + (size_t)L * N, ct_in + ((size_t)L * 2 + 0) * N, sizeof(uint32_t) * N);
  ks_fast(a_in, KD, N, m, u, w);
  free(KD);
  free(a_in);
  uint32_t* pieces = (uint32_t*)malloc(sizeof(uint32_t) * cw * p_in); /* [p][L][ab][n], NTT domain */
  for (uint32_t p = 0; p < p_in; ++p)
    for (int L = 0; L < 2; ++L) {
      uint32_t* pa = pieces + (size_t)p * cw + ((size_t)L * 2 + 0) * n;
      uint32_t* pb = pa + n;
      for (uint32_t k = 0; k < n; ++k) {
        const size_t c = piece0 + p + (size_t)rho * k;
        pa[k] = u[(size_t)L * N + c];
        pb[k] = (uint32_t)(((uint64_t)ct_in[((size_t)L * 2 + 1) * N + c] + w[(size_t)L * N + c]) % m[L]);
      }
      fntt_fwd(fntt_get(n, m[L]), pa);
      fntt_fwd(fntt_get(n, m[L]), pb);
    }
  free(u);
  free(w);
  /* (M) leaves: leaf (o, j) = sum_p pt_{o,j,p} * piece_p */
  const size_t leaves = (size_t)p_out * win;
  uint32_t* A = (uint32_t*)malloc(sizeof(uint32_t) * cw * leaves); /* [leaf][L][ab][n] coefficient form */
  const uint32_t cp[2] = {(uint32_t)powmod_p(win, m[0] - 2, m[0]), (uint32_t)powmod_p(win, m[1] - 2, m[1])};
#pragma omp parallel
  {
    uint32_t* pt = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * 2 * n);
#pragma omp for schedule(dynamic, 4)
    for (size_t leaf = 0; leaf < leaves; ++leaf) {
      const uint32_t o = (uint32_t)(leaf / win), j = (uint32_t)(leaf % win);
      for (int L = 0; L < 2; ++L) {
        const uint32_t q = m[L];
        const fntt_t* T = fntt_get(n, q);
        memset(acc, 0, sizeof(uint64_t) * 2 * n);
        for (uint32_t p = 0; p < p_in; ++p) {
          for (uint32_t pos = 0; pos < n; ++pos) {
            uint32_t uu, hw;
            int neg = 0;
            if (pos == 0) {
              uu = 0;
              hw = 0;
            } else if (pos <= n - win) {
              uu = (pos + win - 1) / win;
              hw = uu * win - pos;
            } else {
              uu = 0;
              hw = n - pos;
              neg = 1;
            }
            const uint32_t r = n * o + or_half_reverse(uu * win + j, n);
            const uint32_t col = win * p + or_window_reverse(hw, win);
            const int64_t wv = (r < n_out && col < n_in) ? Wt[(size_t)r * n_in + col] : 0;
            uint32_t v = (uint32_t)mulmod_p(modq_s(wv, q), cp[L], q);
            pt[pos] = (neg && v) ? q - v : v;
          }
          fntt_fwd(T, pt);
          const uint32_t* pa = pieces + (size_t)p * cw + ((size_t)L * 2 + 0) * n;
          const uint32_t* pb = pa + n;
          for (uint32_t k = 0; k < n; ++k) {
            acc[k] = (acc[k] + (uint64_t)pt[k] * pa[k]) % q;
            acc[n + k] = (acc[n + k] + (uint64_t)pt[k] * pb[k]) % q;
          }
        }
        uint32_t* dst = A + leaf * cw + (size_t)L * 2 * n;
        for (uint32_t k = 0; k < 2 * n; ++k) dst[k] = (uint32_t)acc[k];
        fntt_inv(T, dst);
        fntt_inv(T, dst + n);
      }
    }
    free(pt);
    free(acc);
  }
  free(pieces);
  /* (P) PackLWEs levels l' = s+1 .. log2 n; at level l' leaf e_i pairs with e_i + n/2^l' inside its group */
  size_t cnt = leaves;
  uint32_t* An = (uint32_t*)malloc(sizeof(uint32_t) * cw * (leaves / 2 + 1));
  for (int lv = s + 1; lv <= logn; ++lv) {
    const uint32_t half = n >> lv, k = (1u << lv) + 1;
    const size_t cnt_out = cnt / 2;
    uint32_t* KN = ksk_ntt(gal + (size_t)(lv - 1) * 12 * n, n, m);
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t idx = 0; idx < cnt_out; ++idx) {
      const size_t grp = idx / half, s_ = idx % half;
      const size_t ei = grp * 2 * half + s_, oi = ei + half;
      pack_combine(A + ei * cw, A + oi * cw, n, half, k, KN, m, An + idx * cw);
    }
    free(KN);
    memcpy(A, An, sizeof(uint32_t) * cw * cnt_out);
    cnt = cnt_out;
  }
  free(An);
  /* (R) + (C) */
  const uint32_t q0 = m[0], q1 = m[1];
  if (level1) {
    memset(out, 0, sizeof(uint32_t) * 4 * N);
    for (uint32_t o = 0; o < p_out; ++o)
      for (int L = 0; L < 2; ++L)
        for (int ab = 0; ab < 2; ++ab)
          for (uint32_t k = 0; k < n; ++k)
            out[((size_t)L * 2 + ab) * N + o + (size_t)rho * k] = A[(size_t)o * cw + ((size_t)L * 2 + ab) * n + k];
  } else {
    const uint64_t q1inv = powmod_p(q1 % q0, q0 - 2, q0);
    memset(out, 0, sizeof(uint32_t) * 2 * N);
    for (uint32_t o = 0; o < p_out; ++o)
      for (int ab = 0; ab < 2; ++ab)
        for (uint32_t k = 0; k < n; ++k) {
          const uint32_t x0 = A[(size_t)o * cw + (size_t)ab * n + k];
          const uint32_t x1 = A[(size_t)o * cw + ((size_t)2 + ab) * n + k];
          const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - q1 : (int64_t)x1;
          out[(size_t)ab * N + o + (size_t)rho * k] = (uint32_t)mulmod_p(modq_s((int64_t)x0 - x1c, q0), q1inv, q0);
        }
  }
  free(A);
  return 0;
}

/* column-shard combine: sum `count` level-1 outputs [count][2 limbs][2][N] mod q_i, rescale by q1 -> [2][N] */
void or_rhombus_combine(const uint32_t* parts, uint32_t count, uint32_t N, const uint32_t* m, uint32_t* out) {
  const uint32_t q0 = m[0], q1 = m[1];
  const uint64_t q1inv = powmod_p(q1 % q0, q0 - 2, q0);
  for (int ab = 0; ab < 2; ++ab)
    for (uint32_t k = 0; k < N; ++k) {
      uint64_t x0 = 0, x1 = 0;
      for (uint32_t i = 0; i < count; ++i) {
        x0 += parts[(size_t)i * 4 * N + (size_t)ab * N + k];
        x1 += parts[(size_t)i * 4 * N + ((size_t)2 + ab) * N + k];
      }
      x0 %= q0;
      x1 %= q1;
      const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - q1 : (int64_t)x1;
      out[(size_t)ab * N + k] = (uint32_t)mulmod_p(modq_s((int64_t)x0 - x1c, q0), q1inv, q0);
    }
}
