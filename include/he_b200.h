/*
 * he_b200.h -- C ABI of the B200-native MLWE PCMM / Rhombus PCMv path.
 *
 * Plain pointers and sizes only (no torch types).  Every pointer argument named *_dev
 * is DEVICE memory owned by the caller; `stream` is a cudaStream_t passed as void*.
 * All calls are asynchronous on `stream` unless stated otherwise, validate their
 * arguments before launching anything, and return an he_status.  he_last_error()
 * returns a thread-local message for the last non-OK status.
 *
 * The reference package (hesim) has no FFI: its "operator API" is the Python export
 * list (pkg/src/hesim/__init__.py:8-9,26-27).  Each entry point below cites the
 * reference interface it replaces; the Python mirror lives in
 * paper_2601_18511_b200/pcmm.py and paper_2601_18511_b200/rhombus.py, and
 * INTEGRATION.md shows the ctypes binding a hesim maintainer would add.
 *
 * Status codes map to the reference's exceptions (matmul.py:139-149, slotsim.py:27-28):
 *   HE_EINVAL -> ValueError, HE_ETYPE -> TypeError,
 *   HE_ENEEDS_BOOTSTRAP -> NeedsBootstrapError, HE_ECUDA / HE_ENOMEM -> RuntimeError.
 *
 * Data layouts (u32 words, one residue per word):
 *   RLWE ciphertext batch at level L  : [n_ct][L+1 limbs][2 = (a, b)][N]
 *   plaintext / activations           : f64 [tokens = d/2][n_cols]  (App. A layout)
 *   PCMM output (level 0, limb q0)    : b' composed  [n_out/k][N]   (RLWE order)
 *                                       a' MLWE rows [n_out][k][d]  (row y = block y/k, component y%k)
 *   weight digit planes               : i8 [d_w][n_out][n_in]        (block-shuffled, balanced digits)
 */
#ifndef HE_B200_H
#define HE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HE_OK = 0,
  HE_EINVAL = 1,           /* ValueError          */
  HE_ETYPE = 2,            /* TypeError           */
  HE_ENEEDS_BOOTSTRAP = 3, /* NeedsBootstrapError */
  HE_ECUDA = 4,            /* RuntimeError        */
  HE_ENOMEM = 5            /* RuntimeError        */
} he_status;

/* Scheme parameters; mirrors hesim.SimParams' role (slotsim.py:86-129). */
typedef struct {
  uint32_t mlwe_degree;    /* d  (256)                                  */
  uint32_t mlwe_rank;      /* k  (256);  N = d * k                      */
  uint32_t moduli[2];      /* q0 (base), q1 (PCMM scale prime = Delta_w) */
  uint32_t log_delta;      /* input scale Delta = 2^log_delta           */
  uint32_t rhombus_degree; /* RLWE degree of the PCMv path (4096)       */
  uint32_t special_prime;  /* P of the hybrid key switches (PCMv)       */
} he_params;

typedef struct he_context he_context;     /* NTT tables, device constants       */
typedef struct he_pcmm_plan he_pcmm_plan; /* weight side of the MLWE PCMM       */
typedef struct he_rhombus_plan he_rhombus_plan; /* weight side of the Rhombus PCMv */
typedef struct he_ring_pack_plan he_ring_pack_plan; /* MLWE -> RLWE ring packing tables */
typedef struct he_slot_pcmm_plan he_slot_pcmm_plan; /* slot-domain BSGS PCMM (hesim pcmm_bsgs) */

/* Operation counters, same field names as hesim.CostLedger (slotsim.py:31-83). */
typedef struct {
  int64_t ct_rotations, cc_mults, pc_mults, pt_rotations, pt_mults, rescales, bootstraps;
} he_ledger;

const char* he_last_error(void);
int he_version(void);

/* ---------------------------------------------------------------- context */
/* replaces hesim.SlotContext(SimParams) construction (slotsim.py:171-176) */
he_status he_context_create(const he_params* params, he_context** out);
he_status he_context_destroy(he_context* ctx);
/* Sampling key.  key = 32 secret bytes: secrets, masks a, errors and key-switching keys are drawn from
 * ChaCha20 (RFC 8439) under that key, the per-call `seed` arguments acting as nonces (never reuse one
 * for two encryptions).  key = NULL (the default of he_context_create): the seeded splitmix64 test
 * path -- deterministic, reproduced word for word by the CPU oracle, and NOT secure (a 64-bit seed). */
he_status he_context_set_rng_key(he_context* ctx, const uint8_t* key);
/* one ChaCha20 block (host; the device sampler's block function, for known-answer tests) */
he_status he_chacha20_block(const uint8_t* key, uint32_t counter, const uint8_t* nonce, uint8_t* out);

/* ---------------------------------------------------------------- keys, encryption (test/bench plumbing) */
/* ternary secret s (int32 [N]) and its NTT per limb (u32 [2][N]) */
he_status he_keygen(const he_context* ctx, uint64_t seed, int32_t* s_dev, uint32_t* s_ntt_dev, void* stream);
/* replaces hesim.encrypt_matrix / pack_sheared (packing.py:81-91): coefficient-encode
 * acts (f64 [d/2][n_in], App. A layout) and encrypt at level 1 -> ct [n_in/k][2][2][N].
 * Block r uses RNG streams of global block index r0 + r. */
he_status he_encrypt_acts(const he_context* ctx, const uint32_t* s_ntt_dev, const double* acts_dev, uint32_t n_in,
                          uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream);
/* ModRaise, the hand-off to (Half-)Bootstrapping: level-0 ciphertexts mod q0
 * [n_ct][2][N] -> the centred lift of every coefficient into each of the n_primes (<= 64) target primes
 * (device array): out [n_ct][n_primes][2][N].  The raised phase is phase_q0 + q0 I(X) with a small integer
 * I (the term bootstrapping's EvalMod removes). */
he_status he_mod_raise(const he_context* ctx, const uint32_t* ct_dev, uint32_t n_ct, const uint32_t* primes_dev,
                       uint32_t n_primes, uint32_t* out_dev, void* stream);
/* centred phase of limb `limb` of an RLWE batch: int64 [n_ct][N] */
he_status he_decrypt_rlwe(const he_context* ctx, const uint32_t* s_ntt_dev, const uint32_t* ct_dev, uint32_t n_ct,
                          uint32_t limbs, uint32_t limb, int64_t* phase_dev, void* stream);
/* centred phases of MLWE PCMM output rows [row0, row0+n_rows): int64 [n_rows][d] (level 0, q0) */
he_status he_decrypt_mlwe(const he_context* ctx, const int32_t* s_dev, const uint32_t* out_b_dev,
                          const uint32_t* out_a_dev, uint32_t n_out, uint32_t row0, uint32_t n_rows,
                          int64_t* phase_dev, void* stream);

/* ---------------------------------------------------------------- negacyclic NTT (K2) */
/* in-place forward (natural -> bit-reversed) / inverse (bit-reversed -> natural, scaled)
 * over `count` polys of degree n (n = N or rhombus_degree) spaced `stride` words apart,
 * modulus moduli[limb]. */
he_status he_ntt_forward(const he_context* ctx, uint32_t* data_dev, uint32_t n, uint32_t limb, uint32_t count,
                         uint64_t stride, void* stream);
he_status he_ntt_inverse(const he_context* ctx, uint32_t* data_dev, uint32_t n, uint32_t limb, uint32_t count,
                         uint64_t stride, void* stream);

/* ---------------------------------------------------------------- MLWE PCMM (K1 + K3) */
/* replaces hesim.make_pcmm_plan (matmul.py:77-100).  Step 1: encode + block-shuffle
 * the f64 weights W [n_out][n_in] (row-major, device) into integer W~ = round(q1 * W) in
 * GEMM order and report max|W~| (synchronous). */
he_status he_pcmm_weight_maxabs(const he_context* ctx, const double* w_dev, uint32_t n_out, uint32_t n_in,
                                uint64_t* maxabs_out, void* stream);
/* Step 2: write the d_w balanced digit planes i8 [d_w][n_out][n_in] (caller-allocated). */
he_status he_pcmm_encode_weights(const he_context* ctx, const double* w_dev, uint32_t n_out, uint32_t n_in,
                                 uint32_t d_w, int8_t* digits_dev, void* stream);
/* Step 3: the immutable plan over caller-owned digit planes (kept alive by the caller). */
he_status he_pcmm_plan_create(const he_context* ctx, const int8_t* digits_dev, uint32_t n_out, uint32_t n_in,
                              uint32_t d_w, he_pcmm_plan** out);
he_status he_pcmm_plan_destroy(he_pcmm_plan* plan);
/* bytes of scratch he_pcmm_run needs (ciphertext digit planes) */
he_status he_pcmm_workspace_bytes(const he_pcmm_plan* plan, uint64_t* bytes);
/* replaces hesim.pcmm_depth1 / pcmm_bsgs (matmul.py:152-176): ct_in at level `level`
 * (must be 1; 0 -> HE_ENEEDS_BOOTSTRAP) -> level-0 MLWE output.  Increments `ledger`
 * (may be NULL) like one fused pc_linear per output block: pc_mults += (n_out/k)(n_in/k),
 * rescales += n_out/k, ct_rotations += 0. */
he_status he_pcmm_run(const he_pcmm_plan* plan, const uint32_t* ct_in_dev, uint32_t level, uint32_t* out_b_dev,
                      uint32_t* out_a_dev, void* workspace_dev, uint64_t workspace_bytes, void* stream,
                      he_ledger* ledger);
/* the two stages of he_pcmm_run, exposed for profiling */
he_status he_pcmm_decompose(const he_pcmm_plan* plan, const uint32_t* ct_in_dev, void* workspace_dev,
                            uint64_t workspace_bytes, void* stream);
he_status he_pcmm_gemm(const he_pcmm_plan* plan, const void* workspace_dev, uint32_t* out_b_dev,
                       uint32_t* out_a_dev, void* stream);
/* K1 on output rows [row0, row0 + rows) only (k-aligned), writing the chunk's b' blocks and a'
 * rows to out_b_dev [rows/k][N] / out_a_dev [rows][k*d]: lets a caller stream the output to
 * host memory chunk by chunk while the next chunk computes (pcmm_mlwe_to_host). */
he_status he_pcmm_gemm_rows(const he_pcmm_plan* plan, const void* workspace_dev, uint32_t row0, uint32_t rows,
                            uint32_t* out_b_dev, uint32_t* out_a_dev, void* stream);
/* Fused output all-gather (row-sharded multi-GPU): like he_pcmm_gemm_rows, but the
 * output stage stores every word into each of the n_peers (<= 8) FULL output buffers -- device pointers
 * reachable from this GPU (peer memory over NVLink: CUDA IPC / symmetric memory) -- at destination rows
 * dst_row0 + (y - row0), so the all-gather rides on the kernels' own stores instead of a separate
 * collective.  out_*_peers are HOST arrays of device pointers (b' [n_out/k][N], a' [n_out][k*d] each).
 * Spectral plans need the L = 1024 path (k = 256). */
he_status he_pcmm_gemm_rows_peers(const he_pcmm_plan* plan, const void* workspace_dev, uint32_t row0, uint32_t rows,
                                  uint32_t* const* out_b_peers, uint32_t* const* out_a_peers, uint32_t n_peers,
                                  uint32_t dst_row0, void* stream);
/* Spectral a-part (K7, same output words): the plan's a' columns are computed as blockwise
 * length-2k cyclic NTT correlations instead of the d*k-column GEMM (b' columns stay on K1).
 * Step 1 reports the bytes of the spectral weights G^ (caller-allocated device memory, kept
 * alive by the caller); step 2 fills them from the plan's digit planes and switches the plan's
 * he_pcmm_run / decompose / gemm(_rows) to the spectral path.  Part of plan construction:
 * call it before sharing the plan.  Workspace sizes change accordingly. */
he_status he_pcmm_spectral_weight_bytes(const he_pcmm_plan* plan, uint64_t* bytes);
he_status he_pcmm_spectral_prepare(he_pcmm_plan* plan, int8_t* spec_weights_dev, void* stream);
/* spectral plans: info[0..3] = {transform length L, outputs per block L - k, blocks, blocks padded to 32} */
he_status he_pcmm_spectral_info(const he_pcmm_plan* plan, uint32_t* info);
/* 0 = K1 over all columns (direct), 1 = spectral */
he_status he_pcmm_algo(const he_pcmm_plan* plan, int* algo);
/* Profiling: while enabled, every stage launch of the plan records a CUDA event pair on its
 * stream; he_pcmm_profile_read synchronizes, returns the summed device ms and launch count per
 * stage {0 K3 decompose, 1 K7 data transform S2, 2 K1 GEMM, 3 S3 limb 0, 4 S3 limb 1, 5 S4} and
 * clears them.  Not thread-safe while enabled (mirrors CostLedger's fork/merge rule). */
he_status he_pcmm_profile(const he_pcmm_plan* plan, int enable);
he_status he_pcmm_profile_read(const he_pcmm_plan* plan, double* ms, uint32_t* launches, uint32_t n);

/* ---------------------------------------------------------------- Rhombus PCMv (K6), degree n = rhombus_degree */
/* No hesim entry point exists for the PCMv; the calling convention follows pcmm_depth1
 * (matmul.py:152-162).  Rhombus [rhombus] as the paper uses it:
 *   decompose (key switch s -> s'(X^rho), free X^rho split, rho = N / n)  ->  products  ->  output
 *   packing (PackLWEs with Galois key switches)  ->  rescale  ->  compose.
 * Split point (Rhombus's input/output packing trade-off): window w = n >> split.  Input layout:
 * element e at degree-N coefficient (e / w) + rho h_w(e mod w) (h_w fixes the top bit and reverses
 * the others; w = n is the h layout of PAPER.md:674-680), so every input piece carries w values and
 * one plaintext x ciphertext product yields n / w inner products.  Output packing then needs w - 1
 * Galois key switches per output piece instead of n - 1.  Output layout (any window): element r at
 * (r / n) + rho h_n(r mod n).  Oracle: or_rhombus_pcmv_w (oracle/he_oracle_pcmv.c). */
he_status he_encrypt_vector_w(const he_context* ctx, const uint32_t* s_ntt_dev, const double* v_dev, uint32_t n_vals,
                              uint32_t window, uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream);
/* window = n (split point 0) */
he_status he_encrypt_vector(const he_context* ctx, const uint32_t* s_ntt_dev, const double* v_dev, uint32_t n_vals,
                            uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream);
/* keys: sparse secret s' (int32 [n]), s'(X^rho) (int32 [N]) and its NTT per limb (u32 [2][N]),
 * the decompose key s -> s'(X^rho) (u32 [2][2][3][N], NTT domain, moduli q0 q1 P) and the
 * Galois keys sigma_{2^l+1}(s') -> s' (u32 [log2 n][2][2][3][n], NTT domain; a window-w plan uses
 * the top log2 w of them) */
he_status he_rhombus_keygen(const he_context* ctx, uint64_t seed, const int32_t* s_dev, int32_t* s_small_dev,
                            int32_t* s_up_dev, uint32_t* s_up_ntt_dev, uint32_t* ksk_dec_dev, uint32_t* gal_dev,
                            void* stream);
/* weights: W~ = round(q1 W) as NTT-domain plaintexts u32 [2][leaves][ceil(n_in/w)][n],
 * leaves = ceil(n_out/n) * w / groups.  groups > 1: a leaf-interleaved multi-GPU shard holding the
 * leaves j = group + groups * jl of every output piece (rows r = n o + h_n(u w + j)). */
he_status he_rhombus_weight_bytes_w(const he_context* ctx, uint32_t n_out, uint32_t n_in, uint32_t window,
                                    uint32_t groups, uint64_t* bytes);
he_status he_rhombus_encode_weights_w(const he_context* ctx, const double* w_dev, uint32_t n_out, uint32_t n_in,
                                      uint32_t window, uint32_t groups, uint32_t group, uint32_t* wpt_dev, void* stream);
he_status he_rhombus_plan_create_w(const he_context* ctx, const uint32_t* wpt_dev, uint32_t n_out, uint32_t n_in,
                                   uint32_t window, uint32_t groups, uint32_t group, he_rhombus_plan** out);
/* the split-point-0, one-group forms of the three calls above */
he_status he_rhombus_weight_bytes(const he_context* ctx, uint32_t n_out, uint32_t n_in, uint64_t* bytes);
he_status he_rhombus_encode_weights(const he_context* ctx, const double* w_dev, uint32_t n_out, uint32_t n_in,
                                    uint32_t* wpt_dev, void* stream);
he_status he_rhombus_plan_create(const he_context* ctx, const uint32_t* wpt_dev, uint32_t n_out, uint32_t n_in,
                                 he_rhombus_plan** out);
/* info[0..6] = {window, split, groups, group, input pieces, output pieces, leaves} */
he_status he_rhombus_plan_info(const he_rhombus_plan* plan, uint32_t* info);
he_status he_rhombus_plan_destroy(he_rhombus_plan* plan);
he_status he_rhombus_workspace_bytes(const he_rhombus_plan* plan, uint64_t* bytes);
/* level-1 degree-N ct [2][2][N] under s -> level-0 degree-N ct [2 (a, b)][N] under s'(X^rho)
 * holding W v; ledger: pc_mults += plaintext x ciphertext products (leaves * input pieces),
 * ct_rotations += (w - 1) * ceil(n_out/n) Galois key switches, rescales += 1.  groups must be 1. */
he_status he_rhombus_run(const he_rhombus_plan* plan, const uint32_t* ct_in_dev, uint32_t level,
                         const uint32_t* ksk_dec_dev, const uint32_t* gal_dev, uint32_t* out_dev, void* workspace_dev,
                         uint64_t workspace_bytes, void* stream, he_ledger* ledger);
/* Multi-GPU shards.
 * Column shards ("the ciphertext is masked and each GPU is assigned 4096/8 values"): a plan over the
 * columns [w piece0, ..) of W (groups 1) runs on input pieces piece0.. of the full input ciphertext
 * (and/or on output pieces from opiece0) and writes its LEVEL-1 composed partial output out_l1
 * [2 limbs][2 (a, b)][N] (zeros outside its output pieces; no rescale).  he_rhombus_combine sums `count`
 * such outputs mod q_i (parts [count][2][2][N], e.g. after an all-gather) and rescales once ->
 * level-0 ct [2][N] (the same plaintext as one GPU, different key-switching noise). */
he_status he_rhombus_run_shard(const he_rhombus_plan* plan, const uint32_t* ct_in_dev, uint32_t level,
                               const uint32_t* ksk_dec_dev, const uint32_t* gal_dev, uint32_t piece0, uint32_t opiece0,
                               uint32_t* out_l1_dev, void* workspace_dev, uint64_t workspace_bytes, void* stream,
                               he_ledger* ledger);
he_status he_rhombus_combine(const he_context* ctx, const uint32_t* parts_dev, uint32_t count, uint32_t* out_dev,
                             void* stream, he_ledger* ledger);
/* Row shards ("broadcast the ciphertext ... split the plaintext matrix"): a plan with groups = G
 * ranks (group g) runs the products of its leaves and the packing levels below the top log2 G and
 * writes its subtree roots roots_out [2 limbs][p_out][2][n] (NTT domain, level 1).  After an
 * all-gather of the G roots ([G][2][p_out][2][n], rank order), he_rhombus_finish (any rank's plan)
 * runs the top log2 G levels, the rescale and the compose: the output words equal the one-GPU
 * run's.  ledger: the subtree run counts its products and key switches, the finish (G - 1) p_out key
 * switches and the rescale. */
he_status he_rhombus_run_subtree(const he_rhombus_plan* plan, const uint32_t* ct_in_dev, uint32_t level,
                                 const uint32_t* ksk_dec_dev, const uint32_t* gal_dev, uint32_t* roots_out_dev,
                                 void* workspace_dev, uint64_t workspace_bytes, void* stream, he_ledger* ledger);
he_status he_rhombus_finish(const he_rhombus_plan* plan, const uint32_t* roots_dev, const uint32_t* gal_dev,
                            uint32_t* out_dev, void* workspace_dev, uint64_t workspace_bytes, void* stream,
                            he_ledger* ledger);

/* ---------------------------------------------------------------- MLWE -> RLWE ring packing
 * The step after the PCMM toward Half-Bootstrap: each block of k MLWE output rows
 * becomes ONE RLWE ciphertext under s whose phase at coefficient t + k m is row (block, t)'s phase
 * at m -- the activation layout he_encrypt_acts produces, so the packed output is the next
 * layer's input format.  hesim has no counterpart (its PCMM output stays in slots); the oracle is
 * or_ring_pack in oracle/he_oracle_rhombus.c.
 *
 * Step 1: the PCMM at level 1 WITHOUT the rescale: raw_b [2 limbs][n_out/k][N] (b' in RLWE order,
 * like out_b), raw_a [2 limbs][n_out][k*d] (a' MLWE rows, like out_a), words mod q0 / q1. */
he_status he_pcmm_run_level1(const he_pcmm_plan* plan, const uint32_t* ct_in_dev, uint32_t level, uint32_t* raw_b_dev,
                             uint32_t* raw_a_dev, void* workspace_dev, uint64_t workspace_bytes, void* stream);
/* Packing methods:
 *   HE_RING_PACK_KEYSWITCH (default): MLWE -> RLWE key switching (HERMES / BCHPS style, SURVEY.md
 *     App. B.4): block Y's packed phase is b'_Y + sum_j alpha_j(X) s_j(X^k) with alpha_j the
 *     interleave of the block's a' component j; one hybrid key switch per j from s_j(X^k) to s,
 *     summed before a single ModDown.  Keys: u32 [k][2][2][3][N] (ids 0x200 + j).
 *   HE_RING_PACK_TRACE: PackLWEs over the subring Z[X^k] (CDKS21): log2 k levels of
 *     E + X^{k/2^l} O + sigma_g(E - X^{k/2^l} O), g = 1 + 2^l d, one Galois key switch per combine.
 *     Keys sigma_g(s) -> s: u32 [log2 k][2][2][3][N] (ids 0x100 + l).
 *   HE_RING_PACK_KEYSWITCH1: the same key switching with ONE digit (alpha_j mod Q = q0 q1 itself) and two
 *     special primes P1 = P, P2 = he_ring_pack_special2 (the largest NTT prime < 2^30 that is not q0, q1, P):
 *     4 NTT'd planes per (block, j) instead of 6.  Keys: u32 [k][2 (alpha, beta)][4 (q0, q1, P1, P2)][N]
 *     encrypting P1 P2 s_j(X^k) (ids 0x300 + j); ModDown by P1 P2 with a CRT-centred [x]_{P1 P2}.
 * Keys are NTT domain (moduli q0 q1 P, plus P2 for KEYSWITCH1); all methods give identical plaintexts
 * (different noise). */
#define HE_RING_PACK_KEYSWITCH 0
#define HE_RING_PACK_TRACE 1
#define HE_RING_PACK_KEYSWITCH1 2
he_status he_ring_pack_special2(const he_context* ctx, uint32_t* p2);
he_status he_ring_pack_key_bytes(const he_context* ctx, int method, uint64_t* bytes);
he_status he_ring_pack_keygen(const he_context* ctx, int method, uint64_t seed, const int32_t* s_dev,
                              uint32_t* keys_dev, void* stream);
/* n_out must be a multiple of k */
he_status he_ring_pack_plan_create(const he_context* ctx, uint32_t n_out, int method, he_ring_pack_plan** out);
he_status he_ring_pack_plan_destroy(he_ring_pack_plan* plan);
he_status he_ring_pack_workspace_bytes(const he_ring_pack_plan* plan, uint64_t* bytes);
/* step 2: raw words of step 1 -> level-0 RLWE ciphertexts out [n_out/k][2 (a, b)][N] under s
 * (hybrid key switching with dnum 2 and special prime P, then rescale by q1).  ledger: rescales +=
 * n_out/k; the trace method also ct_rotations += (k - 1) n_out/k. */
he_status he_ring_pack_run(const he_ring_pack_plan* plan, const uint32_t* raw_b_dev, const uint32_t* raw_a_dev,
                           const uint32_t* keys_dev, uint32_t* out_dev, void* workspace_dev, uint64_t workspace_bytes,
                           void* stream, he_ledger* ledger);

/* ---------------------------------------------------------------- slot-domain PCMM
 * hesim's own PCMM, pcmm_bsgs (matmul.py:165-176), on real CKKS ciphertexts: a d x d matrix row-major
 * in the slots (tiled, packing.py:1-17), left slot rotation by r = X -> X^(5^r) + hybrid key switch.
 * baby_i = rot(ct, i d) (hoisted digits), inner_j = sum_i pt_{i + j b} baby_i, out = rescale(sum_j
 * rot(inner_j, j b d)).  Plaintext blocks are CKKS slot encodings (canonical embedding, scale q1)
 * computed by the caller (paper_2601_18511_b200/slots.py) as signed int64 coefficients.
 * Oracle: or_slot_pcmm (oracle/he_oracle_rhombus.c). */
/* encrypt raw integer plaintext polynomials pt [n_ct][N] (int64, signed) at level 1 */
he_status he_encrypt_poly(const he_context* ctx, const uint32_t* s_ntt_dev, const int64_t* pt_dev, uint32_t n_ct,
                          uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream);
/* rotation keys sigma_{5^r}(s) -> s for the host list steps[n]: keys_dev [n][4][2][3][N] (NTT domain; gadget
 * hybrid keys: each of the 2 RNS digits split into 2 sub-digits of 15 bits, ids 0x10000 + r) */
he_status he_slot_rotation_keygen(const he_context* ctx, uint64_t seed, const int32_t* s_dev, const int32_t* steps,
                                  uint32_t n_steps, uint32_t* keys_dev, void* stream);
/* int64 plaintext polys [count][N] -> NTT-domain residues [count][2][N] */
he_status he_slot_pcmm_encode_pts(const he_context* ctx, const int64_t* pt_dev, uint32_t count, uint32_t* pts_ntt_dev,
                                  void* stream);
/* pts_ntt_dev [d][2][N] (block k = i + j b) stays caller-owned; b * g == d, d^2 <= N/2 */
he_status he_slot_pcmm_plan_create(const he_context* ctx, const uint32_t* pts_ntt_dev, uint32_t d, uint32_t b,
                                   uint32_t g, he_slot_pcmm_plan** out);
/* general slot linear map over rotated copies: out = rescale(sum_t pt_t * rot(ct, steps[t])) with steps[0] = 0
 * (hesim pc_linear terms, slotsim.py:330-370; rope_packed, pipeline.py:291-307); runs through
 * he_slot_pcmm_run with keys_baby = rotation keys of steps[1..], keys_giant unused */
he_status he_slot_lt_plan_create(const he_context* ctx, const uint32_t* pts_ntt_dev, uint32_t n_terms,
                                 const int32_t* steps, he_slot_pcmm_plan** out);
/* general BSGS slot linear map over n = b * g diagonals (SlotToCoeffs, PAPER.md:639-643 + App. A bit-reversal;
 * no reference interface -- hesim has no StC): baby steps i * stride, giant steps j * b * stride; pts_ntt_dev
 * [b g][2][N] in order i + j b, diagonal i + j b pre-rotated by -j b stride; runs through he_slot_pcmm_run */
he_status he_slot_bsgs_plan_create(const he_context* ctx, const uint32_t* pts_ntt_dev, uint32_t b, uint32_t g,
                                   uint32_t stride, he_slot_pcmm_plan** out);
/* flags for he_slot_bsgs_plan_create_ext */
#define HE_SLOT_LAZY_MODDOWN 1u /* baby rotations kept mod (q0, q1, P), one ModDown per giant group; pts
                                   [b g][3][N] (he_slot_pcmm_encode_pts_ext with n_mods = 3); b % 8 == 0 */
#define HE_SLOT_PLAIN_GIANT 2u  /* with HE_SLOT_LAZY_MODDOWN: giant rotations use plain dnum-2 keys
                                   (he_slot_rotation_keygen_plain, [g-1][2][2][3][N]) -- their noise lands at
                                   scale Delta q1 -- halving the giant digits' NTTs and key bytes */
/* plain dnum-2 rotation keys sigma_{5^r}(s) -> s, keys_dev [n_steps][2][2][3][N] NTT domain */
he_status he_slot_rotation_keygen_plain(const he_context* ctx, uint64_t seed, const int32_t* s_dev,
                                        const int32_t* steps, uint32_t n_steps, uint32_t* keys_dev, void* stream);
he_status he_slot_bsgs_plan_create_ext(const he_context* ctx, const uint32_t* pts_ntt_dev, uint32_t b, uint32_t g,
                                       uint32_t stride, uint32_t flags, he_slot_pcmm_plan** out);
/* int64 plaintext polys [count][N] -> NTT-domain residues [count][n_mods][N] (n_mods 2: q0, q1; 3: + P) */
he_status he_slot_pcmm_encode_pts_ext(const he_context* ctx, const int64_t* pt_dev, uint32_t count, uint32_t n_mods,
                                      uint32_t* pts_ntt_dev, void* stream);
he_status he_slot_pcmm_plan_destroy(he_slot_pcmm_plan* plan);
he_status he_slot_pcmm_workspace_bytes(const he_slot_pcmm_plan* plan, uint64_t* bytes);
/* ct_in [2][2][N] level 1 -> out [2 (a, b)][N] level 0.  keys_baby: steps i d (i = 1 .. b-1), keys_giant:
 * steps j b d (j = 1 .. g-1).  ledger: ct_rotations += (b-1) + (g-1), pc_mults += d, rescales += 1 */
he_status he_slot_pcmm_run(const he_slot_pcmm_plan* plan, const uint32_t* ct_in_dev, uint32_t level,
                           const uint32_t* keys_baby_dev, const uint32_t* keys_giant_dev, uint32_t* out_dev,
                           void* workspace_dev, uint64_t workspace_bytes, void* stream, he_ledger* ledger);
/* n_ct ciphertexts [n_ct][2][2][N] -> out [n_ct][2][N] under one plan; big maps (b g >= 4096) stream each
 * plaintext once per chunk of up to 3 ciphertexts.  ledger: the per-ct counts times n_ct */
he_status he_slot_pcmm_run_batch(const he_slot_pcmm_plan* plan, const uint32_t* ct_in_dev, uint32_t n_ct,
                                 uint32_t level, const uint32_t* keys_baby_dev, const uint32_t* keys_giant_dev,
                                 uint32_t* out_dev, void* workspace_dev, uint64_t workspace_bytes, void* stream,
                                 he_ledger* ledger);

/* ---------------------------------------------------------------- the modulus chain above level 1
 * ("lower the total level to 4; SlotToCoeffs to level 1").  A chain holds
 * the primes q_0 .. q_L (q_0, q_1 = the context's) and the context's special prime P; a level-l ciphertext
 * is [l + 1 limbs][2 (a, b)][N].  Lowering a level drops top limbs (no kernel: a view).  Slot linear maps
 * consume one level each (BSGS, hybrid key switching with dnum = l + 1); the factorized SlotToCoeffs is three of
 * them.  hesim has no counterpart; oracle: or_chain_* (oracle/he_oracle_chain.c). */
typedef struct he_chain he_chain;
typedef struct he_chain_map he_chain_map;
he_status he_chain_create(const he_context* ctx, const uint32_t* primes, uint32_t count, he_chain** out);
he_status he_chain_destroy(he_chain* chain);
/* pt int64 [n_ct][N] -> ct [n_ct][level + 1][2][N] under s (the context's sampler; oracle or_encrypt) */
he_status he_chain_encrypt(const he_chain* chain, const int32_t* s_dev, const int64_t* pt_dev, uint32_t n_ct,
                           uint32_t level, uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream);
/* phase of ct [n_ct][level + 1][2][N] in limb `limb`, centred int64 [n_ct][N] (CRT over the limbs = the integer
 * phase, e.g. m + q0 I(X) after he_mod_raise into the chain; test/inspection entry point, oracle or_decrypt_rlwe) */
he_status he_chain_decrypt(const he_chain* chain, const int32_t* s_dev, const uint32_t* ct_dev, uint32_t n_ct,
                           uint32_t level, uint32_t limb, int64_t* phase_dev, void* stream);
/* key id of the rotation by `step` at `level` (the sampler's stream); words per rotation key at `level` */
uint32_t he_chain_key_id(uint32_t level, uint32_t step);
he_status he_chain_key_words(const he_chain* chain, uint32_t level, uint64_t* words);
/* rotation keys sigma_{5^r}(s) -> s for `count` steps at `level`: u32 [count][l + 1][2][l + 2][N], NTT domain */
he_status he_chain_rotation_keygen(const he_chain* chain, uint64_t seed, const int32_t* s_dev, uint32_t level,
                                   const int32_t* steps, uint32_t count, uint32_t* keys_dev, void* stream);
/* plaintexts int64 [count][N] -> NTT-domain residues [count][level + 1][N] */
he_status he_chain_encode_pts(const he_chain* chain, const int64_t* pt_dev, uint32_t count, uint32_t level,
                              uint32_t* pts_ntt_dev, void* stream);
/* BSGS map at `level`: out = rescale(sum_j rot_{(j b - T) stride}(sum_i pt_{i + j b} rot_{i stride}(ct))), pts
 * [b g][level + 1][N] (NTT domain, term i + j b pre-rotated by -(j b - T) stride).  Keys: baby [b - 1] for steps
 * i stride, giant [g] for steps (j b - T) stride (the entry of a zero step is not read).  ledger: rotations,
 * b g pc_mults and one rescale per ciphertext. */
he_status he_chain_map_create(const he_chain* chain, const uint32_t* pts_ntt_dev, uint32_t level, uint32_t b,
                              uint32_t g, uint32_t stride, uint32_t T, he_chain_map** out);
he_status he_chain_map_destroy(he_chain_map* map);
he_status he_chain_map_workspace_bytes(const he_chain_map* map, uint64_t* bytes);
he_status he_chain_map_run(const he_chain_map* map, const uint32_t* ct_in_dev, uint32_t n_ct, uint32_t level,
                           const uint32_t* keys_baby_dev, const uint32_t* keys_giant_dev, uint32_t* ct_out_dev,
                           void* workspace_dev, uint64_t workspace_bytes, void* stream, he_ledger* ledger);

#ifdef __cplusplus
}
#endif
#endif /* HE_B200_H */
