/*
 * he_oracle_spectral.c -- TEST / BASELINE INFRASTRUCTURE ONLY (never linked into the product library).
 *
 * A CPU restatement of the MLWE PCMM (BCHPS24 Alg. 2, the same integer result as or_pcmm in he_oracle.c)
 * evaluated the way the GPU's K7 path is organised (DESIGN.md §4 "K7"): the a-part columns of an output row are,
 * per input ciphertext r, the length-k correlation of the weight segment g_{y,r}[t] = Wt[y][k r + t] with the
 * negacyclic read A_r(i) of a_r, sampled at c' = k m + (k - 1 - j); blocks of ob = L - k outputs come out of a
 * cyclic length-L convolution (overlap-save), summed over r in the transform domain.  The b-part columns are the
 * plain sum over (r, t).  Exact modular arithmetic throughout, so every word equals or_pcmm's.
 *
 * Written independently of the CUDA code (own NTT, own layouts, row-parallel with OpenMP); its purposes are
 * (1) a CPU baseline that runs the same algorithm as the GPU on the FULL workload (no extrapolation), and
 * (2) a full-output word check of the GPU result at the Llama shapes (or_pcmm is too slow for every row).
 *
 * Follows: the column definition of SURVEY.md App. B.2 / he_oracle.c mlwe_entry (the reference has no
 * implementation of this path: SPEC.md:8), the rescale of PAPER.md:818-824 (he_oracle.c or_rescale).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 sp_u128;

static uint32_t sp_pow(uint64_t a, uint64_t e, uint32_t q) {
    uint64_t r = 1;
    a %= q;
    while (e) {
        if (e & 1) r = r * a % q;
        a = a * a % q;
        e >>= 1;
    }
    return (uint32_t)r;
}
static inline uint32_t sp_pre(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
/* x w mod q for x < 2^32, w < q < 2^31 (Shoup), reduced to [0, q) */
static inline uint32_t sp_mul(uint32_t x, uint32_t w, uint32_t wp, uint32_t q) {
    uint32_t qh = (uint32_t)(((uint64_t)x * wp) >> 32);
    uint32_t r = x * w - qh * q;
    return r >= q ? r - q : r;
}

typedef struct {
    uint32_t L, q, lg;
    uint32_t *w, *wp, *wi, *wip;   /* omega^j, omega^-j and Shoup companions, j < L / 2 */
    uint32_t *rev;
    uint32_t linv, linvp;
} sp_tab;

static int sp_init(sp_tab* t, uint32_t L, uint32_t q) {
    memset(t, 0, sizeof(*t));
    if (L < 2 || (L & (L - 1)) || (q - 1) % L) return -1;
    uint32_t omega = 0;
    for (uint64_t g = 2; g < q && !omega; ++g) {
        uint32_t c = sp_pow(g, (q - 1) / L, q);
        if (sp_pow(c, L / 2, q) != 1) omega = c;   /* order exactly L (L a power of two) */
    }
    if (!omega) return -1;
    t->L = L;
    t->q = q;
    while ((1u << t->lg) < L) ++t->lg;
    t->w = malloc(sizeof(uint32_t) * L / 2);
    t->wp = malloc(sizeof(uint32_t) * L / 2);
    t->wi = malloc(sizeof(uint32_t) * L / 2);
    t->wip = malloc(sizeof(uint32_t) * L / 2);
    t->rev = malloc(sizeof(uint32_t) * L);
    uint32_t oi = sp_pow(omega, q - 2, q);
    uint64_t p = 1, pi = 1;
    for (uint32_t j = 0; j < L / 2; ++j) {
        t->w[j] = (uint32_t)p, t->wp[j] = sp_pre((uint32_t)p, q);
        t->wi[j] = (uint32_t)pi, t->wip[j] = sp_pre((uint32_t)pi, q);
        p = p * omega % q;
        pi = pi * oi % q;
    }
    for (uint32_t i = 0; i < L; ++i) {
        uint32_t r = 0;
        for (uint32_t b = 0; b < t->lg; ++b) r |= ((i >> b) & 1u) << (t->lg - 1 - b);
        t->rev[i] = r;
    }
    t->linv = sp_pow(L, q - 2, q);
    t->linvp = sp_pre(t->linv, q);
    return 0;
}
static void sp_free(sp_tab* t) { free(t->w); free(t->wp); free(t->wi); free(t->wip); free(t->rev); }

/* in-place cyclic DFT over Z_q of length L (inputs and outputs in [0, q)); inverse includes L^-1 */
static void sp_ntt(const sp_tab* t, uint32_t* a, int inverse) {
    const uint32_t L = t->L, q = t->q;
    for (uint32_t i = 0; i < L; ++i) {
        uint32_t r = t->rev[i];
        if (i < r) { uint32_t x = a[i]; a[i] = a[r]; a[r] = x; }
    }
    const uint32_t* W = inverse ? t->wi : t->w;
    const uint32_t* Wp = inverse ? t->wip : t->wp;
    for (uint32_t len = 2; len <= L; len <<= 1) {
        const uint32_t half = len >> 1, step = L / len;
        for (uint32_t i = 0; i < L; i += len)
            for (uint32_t j = 0; j < half; ++j) {
                uint32_t u = a[i + j];
                uint32_t v = sp_mul(a[i + j + half], W[j * step], Wp[j * step], q);
                uint32_t s = u + v, d = u + q - v;
                a[i + j] = s >= q ? s - q : s;
                a[i + j + half] = d >= q ? d - q : d;
            }
    }
    if (inverse)
        for (uint32_t i = 0; i < L; ++i) a[i] = sp_mul(a[i], t->linv, t->linvp, q);
}

/* x mod q for any u64 x (Barrett, mu = floor(2^64 / q): the quotient estimate is short by at most 1) */
static inline uint32_t sp_red(uint64_t x, uint32_t q, uint64_t mu) {
    uint64_t qh = (uint64_t)(((sp_u128)x * mu) >> 64);
    uint64_t r = x - qh * q;
    return (uint32_t)(r >= q ? r - q : r);
}
static inline uint32_t sp_modq_i64(int64_t v, uint32_t q) { int64_t r = v % (int64_t)q; return (uint32_t)(r < 0 ? r + q : r); }

/*
 * Rescaled level-0 output rows [row0, row0 + n_rows) x all d + d k columns (the or_pcmm layout: b' in columns
 * [0, d), a~_{t,j}[m] at column d + d j + m), from level-1 ciphertexts ct [n_in / k][2 limbs][2 (a, b)][N].
 * L: the transform length (a power of two > k with q_i = 1 mod L; 4 k as on the GPU).  Returns 0, or -1 on
 * unsupported parameters.
 */
int or_pcmm_spectral(uint32_t d, uint32_t k, const uint32_t* q, const int64_t* Wt, uint32_t n_out, uint32_t n_in,
                     const uint32_t* ct, uint32_t row0, uint32_t n_rows, uint32_t L, uint32_t* out) {
    const uint32_t N = d * k, n_ct = n_in / k, width = d + d * k;
    if (L <= k || row0 + n_rows > n_out || n_in % k) return -1;
    const uint32_t ob = L - k, nb = (N + ob - 1) / ob;
    sp_tab T[2];
    if (sp_init(&T[0], L, q[0]) || sp_init(&T[1], L, q[1])) return -1;
    /* A^[limb][beta][f][r]: windows win[u] = A_r(ob beta - (k - 1) + u), A_r negacyclic, 0 past N */
    uint32_t* Ah = malloc(sizeof(uint32_t) * 2 * (size_t)nb * L * n_ct);
    #pragma omp parallel
    {
        uint32_t* win = malloc(sizeof(uint32_t) * L);
        #pragma omp for schedule(dynamic, 4)
        for (int64_t it = 0; it < (int64_t)2 * n_ct * nb; ++it) {
            const uint32_t limb = (uint32_t)(it / ((int64_t)n_ct * nb)), r = (uint32_t)((it / nb) % n_ct);
            const uint32_t beta = (uint32_t)(it % nb), qq = q[limb];
            const uint32_t* a = ct + ((size_t)r * 2 + limb) * 2 * N;
            for (uint32_t u = 0; u < L; ++u) {
                int64_t i = (int64_t)ob * beta - (int64_t)(k - 1) + u;
                uint32_t v = 0;
                if (i < 0) { uint32_t x = a[i + N]; v = x ? qq - x : 0; }
                else if (i < (int64_t)N) v = a[i];
                win[u] = v;
            }
            sp_ntt(&T[limb], win, 0);
            for (uint32_t f = 0; f < L; ++f) Ah[(((size_t)limb * nb + beta) * L + f) * n_ct + r] = win[f];
        }
        free(win);
    }
    const uint32_t q0 = q[0], q1 = q[1];
    const uint32_t q1inv = sp_pow(q1 % q0, q0 - 2, q0), q1invp = sp_pre(q1inv, q0);
    /* rows in tasks of SP_ROWS: every A^ slice and b row loaded once per task is used for all of its rows */
    enum { SP_ROWS = 8 };
    #pragma omp parallel
    {
        uint32_t* G = malloc(sizeof(uint32_t) * SP_ROWS * 2 * (size_t)L * n_ct);   /* G^[row][limb][f][r] */
        uint32_t* buf = malloc(sizeof(uint32_t) * SP_ROWS * (size_t)L);
        uint32_t* v = malloc(sizeof(uint32_t) * SP_ROWS * 2 * (size_t)(ob > d ? ob : d));
        uint32_t* wq = malloc(sizeof(uint32_t) * SP_ROWS * (size_t)n_in);
        const size_t vs = 2 * (size_t)(ob > d ? ob : d);
        #pragma omp for schedule(dynamic, 1)
        for (int64_t y0 = 0; y0 < (int64_t)n_rows; y0 += SP_ROWS) {
            const uint32_t R = (uint32_t)((int64_t)n_rows - y0 < SP_ROWS ? (int64_t)n_rows - y0 : SP_ROWS);
            for (uint32_t rr = 0; rr < R; ++rr) {
                const int64_t* w = Wt + (size_t)(row0 + y0 + rr) * n_in;
                for (uint32_t limb = 0; limb < 2; ++limb) {
                    const uint32_t qq = q[limb];
                    for (uint32_t r = 0; r < n_ct; ++r) {   /* filter g'[u] = g[-u mod L] */
                        memset(buf, 0, sizeof(uint32_t) * L);
                        for (uint32_t t = 0; t < k; ++t) buf[(L - t) & (L - 1)] = sp_modq_i64(w[(size_t)k * r + t], qq);
                        sp_ntt(&T[limb], buf, 0);
                        for (uint32_t f = 0; f < L; ++f) G[(((size_t)rr * 2 + limb) * L + f) * n_ct + r] = buf[f];
                    }
                }
            }
            /* a-part, block by block: C^[f] = sum_r G^[f][r] A^[beta][f][r], INTT, outputs u < ob */
            for (uint32_t beta = 0; beta < nb; ++beta) {
                for (uint32_t limb = 0; limb < 2; ++limb) {
                    const uint32_t qq = q[limb];
                    const uint64_t mu = ~0ull / qq;
                    for (uint32_t f = 0; f < L; ++f) {
                        const uint32_t* x = Ah + (((size_t)limb * nb + beta) * L + f) * n_ct;
                        for (uint32_t rr = 0; rr < R; ++rr) {
                            const uint32_t* g = G + (((size_t)rr * 2 + limb) * L + f) * n_ct;
                            uint64_t acc = 0;
                            for (uint32_t r0 = 0; r0 < n_ct; r0 += 16) {   /* 16 products < 2^60: no u64 overflow */
                                const uint32_t r1 = r0 + 16 < n_ct ? r0 + 16 : n_ct;
                                for (uint32_t r = r0; r < r1; ++r) acc += (uint64_t)g[r] * x[r];
                                acc = sp_red(acc, qq, mu);
                            }
                            buf[(size_t)rr * L + f] = (uint32_t)acc;
                        }
                    }
                    for (uint32_t rr = 0; rr < R; ++rr) {
                        sp_ntt(&T[limb], buf + (size_t)rr * L, 1);
                        memcpy(v + rr * vs + (size_t)limb * ob, buf + (size_t)rr * L, sizeof(uint32_t) * ob);
                    }
                }
                for (uint32_t rr = 0; rr < R; ++rr) {
                    uint32_t* o = out + (size_t)(y0 + rr) * width;
                    const uint32_t* vr = v + rr * vs;
                    for (uint32_t u = 0; u < ob; ++u) {
                        const uint32_t cp = ob * beta + u;   /* c' = k m + (k - 1 - j) */
                        if (cp >= N) break;
                        const uint32_t m = cp / k, j = k - 1 - cp % k;
                        const uint32_t x0 = vr[u], x1 = vr[ob + u];
                        const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - (int64_t)q1 : (int64_t)x1;
                        const uint32_t t = sp_modq_i64((int64_t)x0 - x1c, q0);
                        o[d + (size_t)d * j + m] = sp_mul(t, q1inv, q1invp, q0);
                    }
                }
            }
            /* b-part: b'[n] = sum_{r, t} Wt[y][k r + t] b_r[t + k n] */
            for (uint32_t limb = 0; limb < 2; ++limb) {
                const uint32_t qq = q[limb];
                const uint64_t mu = ~0ull / qq;
                for (uint32_t rr = 0; rr < R; ++rr) {
                    const int64_t* w = Wt + (size_t)(row0 + y0 + rr) * n_in;
                    for (uint32_t x = 0; x < n_in; ++x) wq[(size_t)rr * n_in + x] = sp_modq_i64(w[x], qq);
                }
                for (uint32_t n = 0; n < d; ++n) {
                    uint64_t acc[SP_ROWS] = {0};
                    for (uint32_t r = 0; r < n_ct; ++r) {
                        const uint32_t* b = ct + (((size_t)r * 2 + limb) * 2 + 1) * N + (size_t)k * n;
                        for (uint32_t rr = 0; rr < R; ++rr) {
                            const uint32_t* g = wq + (size_t)rr * n_in + (size_t)k * r;
                            uint64_t a = acc[rr];
                            for (uint32_t t0 = 0; t0 < k; t0 += 16) {
                                const uint32_t t1 = t0 + 16 < k ? t0 + 16 : k;
                                for (uint32_t t = t0; t < t1; ++t) a += (uint64_t)g[t] * b[t];
                                a = sp_red(a, qq, mu);
                            }
                            acc[rr] = a;
                        }
                    }
                    for (uint32_t rr = 0; rr < R; ++rr) v[rr * vs + (size_t)limb * d + n] = (uint32_t)acc[rr];
                }
            }
            for (uint32_t rr = 0; rr < R; ++rr) {
                uint32_t* o = out + (size_t)(y0 + rr) * width;
                const uint32_t* vr = v + rr * vs;
                for (uint32_t n = 0; n < d; ++n) {
                    const uint32_t x0 = vr[n], x1 = vr[d + n];
                    const int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - (int64_t)q1 : (int64_t)x1;
                    o[n] = sp_mul(sp_modq_i64((int64_t)x0 - x1c, q0), q1inv, q1invp, q0);
                }
            }
        }
        free(G); free(buf); free(v); free(wq);
    }
    free(Ah);
    sp_free(&T[0]);
    sp_free(&T[1]);
    return 0;
}
