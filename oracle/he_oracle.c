/*
 * he_oracle.c -- CPU restatement of the MLWE-format PCMM path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the integer oracle the CUDA path is checked against.  It is
 * never linked into, called by, or shipped with the product library: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * PARITY UNPINNED at the integer level: the reference package (hesim) does not
 * implement the MLWE PCMM / Rhombus PCMv;
 * the paper's implementation (HEaaN2 + unshipped kernels) is
 * not available.  This restatement follows the prose and algebra instead:
 *   - CKKS Enc/Dec, coefficient encoding, rescale ........ PAPER.md:765-800, 818-824
 *   - MLWE decomposition (degree d, rank k, N = d*k) ..... PAPER.md:54-55, SURVEY.md App. B.2
 *   - App. A block layout ct[i+128j]=A[i][f(j,8)], bit-reversed coefficient order,
 *     g/f permutations ................................... PAPER.md:645-672, bitrev.py:14-54
 *   - per-limb GEMM  W~ . [b | a~]  mod q_i ............... PAPER.md:134, SURVEY.md App. B.3
 * Layout and float semantics ARE pinned: tests check the index maps against the
 * reference's bitrev.py (golden tables in tests/golden/) and decrypted outputs
 * against the float product (hesim.clear_pcmm semantics, matmul.py:179-181).
 *
 * Arithmetic is plain exact modular arithmetic on 64/128-bit integers; the
 * algorithm is the definition (no digit splitting, no tensor-core tricks), so a
 * bit-exact match with the GPU says the GPU's digit/Barrett/Shoup pipeline is
 * exact.  Randomness comes from the counter-based generator below, which the
 * CUDA encryptor restates bit-for-bit (paper_2601_18511_b200/csrc/he_common.cuh).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef __int128 i128;

/* ------------------------------------------------------------------ RNG */
/* splitmix64 finaliser; keyed counter-mode generator (shared definition with CUDA). */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t or_rng_key(uint64_t seed, uint64_t stream) {
    return mix64((seed * 0xD1B54A32D192ED03ULL) ^ mix64(stream + 0x9E3779B97F4A7C15ULL));
}
static inline uint64_t draw(uint64_t key, uint64_t idx) {
    return mix64(key + (idx + 1) * 0x9E3779B97F4A7C15ULL);
}
uint64_t or_rng(uint64_t seed, uint64_t stream, uint64_t idx) { return draw(or_rng_key(seed, stream), idx); }

/* Stream identifiers (same constants in he_common.cuh). */
#define STREAM_SECRET   0x5EC0000000000000ULL
#define STREAM_A(r, i)  (0xA000000000000000ULL | ((uint64_t)(r) << 8) | (uint64_t)(i))
#define STREAM_E(r)     (0xE000000000000000ULL | ((uint64_t)(r) << 8))

void or_sample_uniform(uint64_t seed, uint64_t stream, uint32_t q, uint32_t* out, int64_t n) {
    uint64_t key = or_rng_key(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = (uint32_t)(draw(key, (uint64_t)i) % q);
}
/* centred binomial, eta = 21 (variance 10.5, sigma ~ 3.24) */
void or_sample_cbd(uint64_t seed, uint64_t stream, int32_t* out, int64_t n) {
    uint64_t key = or_rng_key(seed, stream);
    for (int64_t i = 0; i < n; ++i) {
        uint64_t x = draw(key, (uint64_t)i);
        out[i] = __builtin_popcountll(x & 0x1FFFFFULL) - __builtin_popcountll((x >> 21) & 0x1FFFFFULL);
    }
}
/* ternary secret, P(0)=1/2, P(+1)=P(-1)=1/4 */
void or_sample_ternary(uint64_t seed, uint64_t stream, int32_t* out, int64_t n) {
    uint64_t key = or_rng_key(seed, stream);
    for (int64_t i = 0; i < n; ++i) {
        uint32_t b = (uint32_t)(draw(key, (uint64_t)i) & 3u);
        out[i] = b == 1 ? 1 : (b == 2 ? -1 : 0);
    }
}

/* ------------------------------------------------------------------ modular helpers */
static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q; a %= q;
    while (e) { if (e & 1) r = mulmod(r, a, q); a = mulmod(a, a, q); e >>= 1; }
    return r;
}
static inline uint32_t modq_i64(int64_t v, uint32_t q) { int64_t r = v % (int64_t)q; return (uint32_t)(r < 0 ? r + q : r); }
static inline uint32_t modq_i128(i128 v, uint32_t q) { i128 r = v % (i128)q; return (uint32_t)(r < 0 ? r + q : r); }

static uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int t = 0; t < bits; ++t) r |= ((x >> t) & 1u) << (bits - 1 - t);
    return r;
}
static int ilog2(uint32_t x) { int l = 0; while ((1u << l) < x) ++l; return l; }
/* f of PAPER.md:647-652 / bitrev.py:24-29: last bit to the top */
static uint32_t rot_down(uint32_t x, int bits) { return (x >> 1) | ((x & 1u) << (bits - 1)); }
/* sigma(t) = f(bitReverse(t, log k), log k): hidden column carried by MLWE component t
 * (PAPER.md:660-667 with the width-8 reading of bitrev.py:36-37; equals byte_mix(swap(t))). */
uint32_t or_sigma(uint32_t t, uint32_t k) { int l = ilog2(k); return rot_down(bitrev(t, l), l); }

/* ------------------------------------------------------------------ negacyclic NTT */
static int find_psi(uint64_t q, uint32_t N, uint64_t* psi) {
    /* primitive 2N-th root of unity: x^((q-1)/2N) with x^N == -1 */
    if ((q - 1) % (2ull * N)) return -1;
    for (uint64_t g = 2; g < q; ++g) {
        uint64_t c = powmod(g, (q - 1) / (2ull * N), q);
        if (powmod(c, N, q) == q - 1) { *psi = c; return 0; }
    }
    return -1;
}

typedef struct { uint32_t N; uint64_t q; uint64_t* fw; uint64_t* iv; uint64_t ninv; } ntt_tab;

static int ntt_init(ntt_tab* t, uint32_t N, uint64_t q) {
    uint64_t psi;
    if (find_psi(q, N, &psi)) return -1;
    uint64_t psii = powmod(psi, q - 2, q);
    int l = ilog2(N);
    t->N = N; t->q = q;
    t->fw = (uint64_t*)malloc(sizeof(uint64_t) * N);
    t->iv = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t p = 1, pi = 1;
    uint64_t* pw = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t* pwi = (uint64_t*)malloc(sizeof(uint64_t) * N);
    for (uint32_t i = 0; i < N; ++i) { pw[i] = p; pwi[i] = pi; p = mulmod(p, psi, q); pi = mulmod(pi, psii, q); }
    for (uint32_t i = 0; i < N; ++i) { t->fw[i] = pw[bitrev(i, l)]; t->iv[i] = pwi[bitrev(i, l)]; }
    free(pw); free(pwi);
    t->ninv = powmod(N, q - 2, q);
    return 0;
}
static void ntt_free(ntt_tab* t) { free(t->fw); free(t->iv); }

/* Cooley-Tukey, natural order in, bit-reversed order out (negacyclic via psi powers). */
static void ntt_fwd(const ntt_tab* T, uint64_t* a) {
    uint32_t N = T->N, t = N; uint64_t q = T->q;
    for (uint32_t m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (uint32_t i = 0; i < m; ++i) {
            uint32_t j1 = 2 * i * t; uint64_t S = T->fw[m + i];
            for (uint32_t j = j1; j < j1 + t; ++j) {
                uint64_t U = a[j], V = mulmod(a[j + t], S, q);
                a[j] = (U + V) % q; a[j + t] = (U + q - V) % q;
            }
        }
    }
}
/* Gentleman-Sande, bit-reversed in, natural out, scaled by N^-1. */
static void ntt_inv(const ntt_tab* T, uint64_t* a) {
    uint32_t N = T->N, t = 1; uint64_t q = T->q;
    for (uint32_t m = N; m > 1; m >>= 1) {
        uint32_t h = m >> 1, j1 = 0;
        for (uint32_t i = 0; i < h; ++i) {
            uint64_t S = T->iv[h + i];
            for (uint32_t j = j1; j < j1 + t; ++j) {
                uint64_t U = a[j], V = a[j + t];
                a[j] = (U + V) % q; a[j + t] = mulmod((U + q - V) % q, S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (uint32_t j = 0; j < N; ++j) a[j] = mulmod(a[j], T->ninv, q);
}

/* out = a * s mod (X^N + 1, q); a in [0,q), s signed small. Returns 0 on success. */
int or_negacyclic_mul(const uint32_t* a, const int32_t* s, uint32_t N, uint32_t q, uint32_t* out) {
    ntt_tab T;
    if (ntt_init(&T, N, q)) return -1;
    uint64_t* x = (uint64_t*)malloc(sizeof(uint64_t) * N);
    uint64_t* y = (uint64_t*)malloc(sizeof(uint64_t) * N);
    for (uint32_t i = 0; i < N; ++i) { x[i] = a[i] % q; y[i] = modq_i64(s[i], q); }
    ntt_fwd(&T, x); ntt_fwd(&T, y);
    for (uint32_t i = 0; i < N; ++i) x[i] = mulmod(x[i], y[i], q);
    ntt_inv(&T, x);
    for (uint32_t i = 0; i < N; ++i) out[i] = (uint32_t)x[i];
    free(x); free(y); ntt_free(&T);
    return 0;
}

/* schoolbook negacyclic product (independent check of the NTT path; small N only) */
void or_negacyclic_mul_schoolbook(const uint32_t* a, const int32_t* s, uint32_t N, uint32_t q, uint32_t* out) {
    for (uint32_t c = 0; c < N; ++c) {
        i128 acc = 0;
        for (uint32_t i = 0; i < N; ++i) {
            uint32_t j = (c + N - i) % N;           /* a_i * s_j with i + j == c (mod N) */
            i128 p = (i128)a[i] * s[j];
            acc += (i + j >= N) ? -p : p;
        }
        out[c] = modq_i128(acc, q);
    }
}

/* ------------------------------------------------------------------ keys / encoding / encryption */
void or_keygen(uint64_t seed, uint32_t N, int32_t* s) { or_sample_ternary(seed, STREAM_SECRET, s, N); }

/*
 * Coefficient encoding of an activation matrix A (tokens x n_in, tokens = d/2, row-major),
 * App. A layout: RLWE ct r holds columns [k r, k r + k).  Coefficient c = t + k m with
 * m < d/2 carries A[bitReverse(m, log(d/2))][k r + sigma(t)]; c >= N/2 (the Ecd_coeff
 * imaginary half) is zero.  Derivation: ct_c[c] = ct_s[bitReverse(c, log N/2)]
 * and ct_s[i + (d/2) j] = A[i][f(j)], bitReverse(t + k m) =
 * bitReverse(m) + (d/2) bitReverse(t).
 */
void or_encode_acts(const double* A, uint32_t n_in, uint32_t d, uint32_t k, double delta, int64_t* pt) {
    uint32_t N = d * k, half = d / 2, n_ct = n_in / k;
    int lh = ilog2(half);
    memset(pt, 0, sizeof(int64_t) * (size_t)n_ct * N);
    for (uint32_t r = 0; r < n_ct; ++r)
        for (uint32_t m = 0; m < half; ++m)
            for (uint32_t t = 0; t < k; ++t) {
                double v = A[(size_t)bitrev(m, lh) * n_in + (size_t)k * r + or_sigma(t, k)];
                pt[(size_t)r * N + t + (size_t)k * m] = llrint(delta * v);
            }
}

/* inverse of or_encode_acts on a centred phase (n_ct x N) -> tokens x (n_ct k) */
void or_decode_acts(const int64_t* phase, uint32_t n_cols, uint32_t d, uint32_t k, double delta, double* A) {
    uint32_t N = d * k, half = d / 2, n_ct = n_cols / k;
    int lh = ilog2(half);
    for (uint32_t r = 0; r < n_ct; ++r)
        for (uint32_t m = 0; m < half; ++m)
            for (uint32_t t = 0; t < k; ++t)
                A[(size_t)bitrev(m, lh) * n_cols + (size_t)k * r + or_sigma(t, k)] =
                    (double)phase[(size_t)r * N + t + (size_t)k * m] / delta;
}

/*
 * Symmetric RLWE encryption: ct = (a, -a s + pt + e) mod q_i per limb.
 * Output layout [n_ct][limbs][2 = (a, b)][N] u32.  Block index r is offset by r0 so a
 * batch can be encrypted in pieces.
 */
int or_encrypt(uint64_t seed, uint32_t N, uint32_t limbs, const uint32_t* q, const int32_t* s,
               const int64_t* pt, uint32_t n_ct, uint32_t r0, uint32_t* ct) {
    int rc = 0;
    #pragma omp parallel for schedule(dynamic) reduction(|:rc)
    for (uint32_t r = 0; r < n_ct; ++r) {
        int32_t* e = (int32_t*)malloc(sizeof(int32_t) * N);
        uint32_t* as = (uint32_t*)malloc(sizeof(uint32_t) * N);
        or_sample_cbd(seed, STREAM_E(r + r0), e, N);
        for (uint32_t i = 0; i < limbs; ++i) {
            uint32_t* a = ct + ((size_t)r * limbs + i) * 2 * N;
            uint32_t* b = a + N;
            or_sample_uniform(seed, STREAM_A(r + r0, i), q[i], a, N);
            rc |= or_negacyclic_mul(a, s, N, q[i], as);
            for (uint32_t c = 0; c < N; ++c) {
                uint64_t v = (uint64_t)modq_i64(pt[(size_t)r * N + c], q[i]) + modq_i64(e[c], q[i]) + (q[i] - as[c]);
                b[c] = (uint32_t)(v % q[i]);
            }
        }
        free(e); free(as);
    }
    return rc;
}

/* phase = b + a s mod q_i (limb `limb` of an RLWE ct), centred into int64 */
int or_decrypt_rlwe(const uint32_t* a, const uint32_t* b, const int32_t* s, uint32_t N, uint32_t q, int64_t* phase) {
    uint32_t* as = (uint32_t*)malloc(sizeof(uint32_t) * N);
    int rc = or_negacyclic_mul(a, s, N, q, as);
    for (uint32_t c = 0; c < N; ++c) {
        uint64_t v = ((uint64_t)b[c] + as[c]) % q;
        phase[c] = v > q / 2 ? (int64_t)v - (int64_t)q : (int64_t)v;
    }
    free(as);
    return rc;
}

/* ------------------------------------------------------------------ weights */
/*
 * Encoded, block-shuffled weight matrix in GEMM order:
 *   Wt[k r' + t'][k r + t] = round(delta_w * W[k r' + sigma(t')][k r + sigma(t)])
 * i.e. each k x k block conjugated by sigma = g o nibble-swap (bitrev.py:57-70 with the
 * component-order indexing of the MLWE rows).  Rounding: round-half-even of the double product.
 */
void or_encode_weights(const double* W, uint32_t n_out, uint32_t n_in, uint32_t k, double delta_w, int64_t* Wt) {
    #pragma omp parallel for schedule(static)
    for (uint32_t y = 0; y < n_out; ++y) {
        uint32_t src_row = (y / k) * k + or_sigma(y % k, k);
        for (uint32_t x = 0; x < n_in; ++x) {
            uint32_t src_col = (x / k) * k + or_sigma(x % k, k);
            Wt[(size_t)y * n_in + x] = llrint(delta_w * W[(size_t)src_row * n_in + src_col]);
        }
    }
}

/* ------------------------------------------------------------------ MLWE decomposition */
/*
 * Column n of the per-limb GEMM operand [b | a~] for MLWE ciphertext x = (r, t)
 * (component t of RLWE ct r):
 *   n <  d          : b_r[t + k n]
 *   n = d + d j + m : a~_{t,j}[m] = a_r[t - j + k m]  read negacyclically
 *                     (a_r[c] for c < 0 is -a_r[c + N]).
 */
static inline uint32_t mlwe_entry(const uint32_t* a, const uint32_t* b, uint32_t t, uint32_t n,
                                  uint32_t d, uint32_t k, uint32_t N, uint32_t q) {
    if (n < d) return b[t + k * n];
    uint32_t j = (n - d) / d, m = (n - d) % d;
    int64_t c = (int64_t)t - (int64_t)j + (int64_t)k * m;
    if (c >= 0) return a[c];
    uint32_t v = a[c + N];
    return v ? q - v : 0;
}

void or_mlwe_column(const uint32_t* ct, uint32_t n_ct, uint32_t limbs, uint32_t limb, uint32_t d, uint32_t k,
                    uint32_t q, uint32_t n, uint32_t* col /* n_ct*k */) {
    uint32_t N = d * k;
    for (uint32_t r = 0; r < n_ct; ++r) {
        const uint32_t* a = ct + ((size_t)r * limbs + limb) * 2 * N;
        const uint32_t* b = a + N;
        for (uint32_t t = 0; t < k; ++t) col[r * k + t] = mlwe_entry(a, b, t, n, d, k, N, q);
    }
}

/* ------------------------------------------------------------------ PCMM */
/* Rescale dropping q1: ((x0 - [x1]_centred) * q1^-1) mod q0. */
uint32_t or_rescale(uint32_t x0, uint32_t x1, uint32_t q0, uint32_t q1) {
    int64_t x1c = x1 > q1 / 2 ? (int64_t)x1 - (int64_t)q1 : (int64_t)x1;
    uint64_t q1inv = powmod(q1 % q0, q0 - 2, q0);
    uint32_t t = modq_i64((int64_t)x0 - x1c, q0);
    return (uint32_t)mulmod(t, q1inv, q0);
}

/*
 * MLWE PCMM on selected output rows and GEMM columns (BCHPS24 Alg. 2 as used at
 * PAPER.md:54-55,134): for each limb i, v_i[y][n] = sum_x Wt[y][x] * [b|a~]_i[x][n] mod q_i,
 * then out[y][n] = rescale(v_0, v_1).  Input at level 1 (limbs = 2), output at level 0.
 * rows == NULL -> all n_out rows; cols == NULL -> all d + d k columns.
 * out is n_rows x n_cols, row-major.
 */
int or_pcmm(uint32_t d, uint32_t k, const uint32_t* q, const int64_t* Wt, uint32_t n_out, uint32_t n_in,
            const uint32_t* ct, const int32_t* rows, uint32_t n_rows, const int32_t* cols, uint32_t n_cols,
            uint32_t* out) {
    uint32_t N = d * k, n_ct = n_in / k, width = d + d * k;
    if (!rows) n_rows = n_out;
    if (!cols) n_cols = width;
    #pragma omp parallel
    {
        uint32_t* c0 = (uint32_t*)malloc(sizeof(uint32_t) * n_in);
        uint32_t* c1 = (uint32_t*)malloc(sizeof(uint32_t) * n_in);
        #pragma omp for schedule(dynamic, 16)
        for (uint32_t ci = 0; ci < n_cols; ++ci) {
            uint32_t n = cols ? (uint32_t)cols[ci] : ci;
            or_mlwe_column(ct, n_ct, 2, 0, d, k, q[0], n, c0);
            or_mlwe_column(ct, n_ct, 2, 1, d, k, q[1], n, c1);
            for (uint32_t ri = 0; ri < n_rows; ++ri) {
                uint32_t y = rows ? (uint32_t)rows[ri] : ri;
                const int64_t* w = Wt + (size_t)y * n_in;
                i128 a0 = 0, a1 = 0;
                for (uint32_t x = 0; x < n_in; ++x) { a0 += (i128)w[x] * c0[x]; a1 += (i128)w[x] * c1[x]; }
                out[(size_t)ri * n_cols + ci] = or_rescale(modq_i128(a0, q[0]), modq_i128(a1, q[1]), q[0], q[1]);
            }
        }
        free(c0); free(c1);
    }
    (void)N;
    return 0;
}

/* un-rescaled single-limb product (for limb-level checks) */
int or_pcmm_limb(uint32_t d, uint32_t k, uint32_t q, uint32_t limbs, uint32_t limb, const int64_t* Wt,
                 uint32_t n_out, uint32_t n_in, const uint32_t* ct, const int32_t* rows, uint32_t n_rows,
                 const int32_t* cols, uint32_t n_cols, uint32_t* out) {
    uint32_t n_ct = n_in / k, width = d + d * k;
    if (!rows) n_rows = n_out;
    if (!cols) n_cols = width;
    #pragma omp parallel
    {
        uint32_t* c0 = (uint32_t*)malloc(sizeof(uint32_t) * n_in);
        #pragma omp for schedule(dynamic, 16)
        for (uint32_t ci = 0; ci < n_cols; ++ci) {
            uint32_t n = cols ? (uint32_t)cols[ci] : ci;
            or_mlwe_column(ct, n_ct, limbs, limb, d, k, q, n, c0);
            for (uint32_t ri = 0; ri < n_rows; ++ri) {
                uint32_t y = rows ? (uint32_t)rows[ri] : ri;
                const int64_t* w = Wt + (size_t)y * n_in;
                i128 a0 = 0;
                for (uint32_t x = 0; x < n_in; ++x) a0 += (i128)w[x] * c0[x];
                out[(size_t)ri * n_cols + ci] = modq_i128(a0, q);
            }
        }
        free(c0);
    }
    return 0;
}

/*
 * MLWE decryption of output rows (level 0, modulus q0):
 *   phase_y[m] = b'_y[m] + sum_j (a'_y[j] * s_j)[m]   in Z_q0[Y]/(Y^d + 1),  s_j[m] = s[j + k m]
 * rows_out: n_rows x (d + d k) words as produced by or_pcmm (b' in columns [0,d)).
 * phase: n_rows x d, centred.
 */
void or_decrypt_mlwe(uint32_t d, uint32_t k, uint32_t q0, const int32_t* s, const uint32_t* rows_out,
                     uint32_t n_rows, int64_t* phase) {
    uint32_t width = d + d * k;
    #pragma omp parallel for schedule(dynamic)
    for (uint32_t ri = 0; ri < n_rows; ++ri) {
        const uint32_t* row = rows_out + (size_t)ri * width;
        for (uint32_t m = 0; m < d; ++m) {
            i128 acc = row[m];
            for (uint32_t j = 0; j < k; ++j) {
                const uint32_t* aj = row + d + (size_t)j * d;
                for (uint32_t mp = 0; mp < d; ++mp) {
                    /* a_j[mp] * s_j[m - mp] with negacyclic wrap */
                    int64_t idx = (int64_t)m - (int64_t)mp;
                    int32_t sv = idx >= 0 ? s[j + k * (uint32_t)idx] : -s[j + k * (uint32_t)(idx + d)];
                    acc += (i128)aj[mp] * sv;
                }
            }
            uint32_t v = modq_i128(acc, q0);
            phase[(size_t)ri * d + m] = v > q0 / 2 ? (int64_t)v - (int64_t)q0 : (int64_t)v;
        }
    }
}

/* compose the b' rows of output RLWE block r' (PAPER.md:63 / SURVEY.md App. B.4): b_rlwe[t' + k m] = b'_(r',t')[m] */
void or_compose_b(const uint32_t* rows_out /* k rows of block r', width each */, uint32_t d, uint32_t k, uint32_t* b_rlwe) {
    uint32_t width = d + d * k;
    for (uint32_t t = 0; t < k; ++t)
        for (uint32_t m = 0; m < d; ++m) b_rlwe[t + k * m] = rows_out[(size_t)t * width + m];
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
