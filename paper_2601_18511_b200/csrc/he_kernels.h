// he_kernels.h -- internal launcher declarations shared by the .cu translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace he {

// (weight digits, limb-0 ciphertext digits, limb-1 ciphertext digits) instantiated for K1
#define HE_GEMM_INSTANCES(X) \
  X(1, 4, 3) X(2, 4, 3) X(3, 4, 3) X(4, 4, 3) X(1, 4, 4) X(2, 4, 4) X(3, 4, 4) X(4, 4, 4)

struct GemmEpiConst {
  uint32_t q[2];
  uint32_t offs[2];     // q * ceil(2^31 / q): maps a negative int32 accumulator into [0, 2^32)
  uint32_t pw[2][8];    // 2^(8 s) mod q
  uint32_t pwp[2][8];   // Shoup companions
  uint32_t q1inv, q1invp;
  uint64_t off64[2];    // q * ceil(2^62 / q): maps the signed int64 recombination into [0, 2^64)
  uint64_t mu[2];       // floor(2^64 / q) (Barrett)
};

// fused output all-gather: the output stage stores every word into each rank's full output buffer (peer
// device pointers, e.g. from CUDA IPC / symmetric memory over NVLink) at destination row dst_row0 + local row
constexpr int kMaxPeers = 8;
struct OutPeers {
  uint32_t* a[kMaxPeers];
  uint32_t* b[kMaxPeers];
  int n;                 // 0: plain local output (out_a / out_b)
  uint32_t dst_row0;     // k-aligned
};

struct GemmArgs {
  int n_out, n_in, width, d, k;
  int group_m;          // raster: pair-rows per group (v2)
  int tile_n;           // v2 tile width (48 or 32)
  uint64_t hint_a, hint_b;  // TMA L2 cache-policy hints
  int epi_skip;         // profiling only: drain TMEM without computing/storing
  int fused;            // 1: B tiles come straight from the compact digit planes (K3 fused into K1)
  uint32_t* out_b;
  uint32_t* out_a;
  uint32_t* out1_b = nullptr;  // level-1 mode: no rescale; limb-1 words here, limb-0 words in out_b / out_a
  uint32_t* out1_a = nullptr;
  OutPeers peers;
  GemmEpiConst c;
};

int gemm_smem_bytes(int dw, int d0, int d1);
// variant 1: single-CTA 128x32 tiles; variant 2 (default): CTA pair, 256 x gemm2_tile_n tiles
constexpr int kGemmBoxRows1 = 32;
int gemm2_tile_n(int dw, int d0, int d1);
cudaError_t launch_modgemm(int variant, int dw, int d0, int d1, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmBa, const GemmArgs& args, int grid, cudaStream_t stream);

// NTT tables for one (modulus, degree)
struct NttTable {
  uint32_t n = 0, q = 0;
  uint32_t *fw = nullptr, *fwp = nullptr, *iv = nullptr, *ivp = nullptr;  // device, n entries each
  uint32_t ninv = 0, ninvp = 0;
  uint2 fw16[16] = {};   // host copies of fw / iv pairs 0 .. 15 (the cols-pass twiddles of n = 16 n2, as kernel
  uint2 iv16[16] = {};   // parameters)
};
cudaError_t ntt_table_init(NttTable& t, uint32_t n, uint32_t q);
void ntt_table_free(NttTable& t);
// rows_only: the caller already ran the outer (cols) stages, e.g. fused into the kernel producing the data
cudaError_t ntt_forward(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t s,
                        bool rows_only = false);
cudaError_t ntt_inverse(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t s);
// njobs (<= 16) batches of the same degree, count and stride in one launch per pass (job i: table t[i], data[i]);
// reduce = false leaves the outputs lazy in [0, 4 q) for a consumer that reduces them itself
cudaError_t ntt_forward_multi(const NttTable* const* t, uint32_t* const* data, int njobs, uint32_t count,
                              uint64_t stride, cudaStream_t s, bool rows_only = false, bool reduce = true);
cudaError_t ntt_inverse_multi(const NttTable* const* t, uint32_t* const* data, int njobs, uint32_t count,
                              uint64_t stride, cudaStream_t s);

struct RingDims {
  uint32_t d, k, N, logk, q[2], log_delta;
  uint32_t n_rh, P;  // Rhombus degree and special prime
  RngCtx rng{};      // sampling key (secure == 0: the seeded splitmix test path)
};

cudaError_t launch_decompose(const RingDims& R, const uint32_t* ct, uint32_t n_in, int d0, int d1, int8_t* planes,
                             uint64_t plane_stride, cudaStream_t s, int b_only = 0);

// ---- K7: spectral (overlap-save NTT) form of the a-part GEMM (he_spectral.cu)
struct SpecTable {  // cyclic NTT of length L mod q
  uint32_t L = 0, q = 0;
  uint2* fw = nullptr;   // (w^j, Shoup) j < L/2
  uint2* iv = nullptr;   // (w^-j, Shoup) j < L/2
  uint2* r2 = nullptr;   // L = 512: per-stage lane tables of the fast inverse (he_spectral.cu)
  uint2 r1[26] = {};     // L = 512 / 1024: round-1 twiddles of the fast inverse (host copy, kernel params)
  uint2* f2 = nullptr;   // L = 1024: per-stage lane tables of the fast forward (S2)
  uint2 f1[26] = {};     // L = 1024: lane-uniform twiddles of the fast forward (kernel params)
  uint32_t linv = 0, linvp = 0;
};
cudaError_t spec_table_init(SpecTable& t, uint32_t L, uint32_t q);
void spec_table_free(SpecTable& t);

struct SpecGemmArgs {
  int n_rows, row0, n_out;  // row range [row0, row0 + n_rows) of n_out
  int L, nb, r_pad;         // transform length, blocks (padded to 32), K bytes of A^ (multiple of 64)
  int kg;                   // K bytes of G^ rows (multiple of 16, <= r_pad): the A operand's 16-byte chunks
  uint32_t q;
  uint32_t qninv;           // -q^-1 mod 2^32 (Montgomery)
  uint64_t off64;           // multiple of q above the recombination bound: makes the sum non-negative
  int32_t pw[8];            // 2^(16 i + 32) mod q (paired shifts)
  uint32_t* out;            // C^ [n_out][nb / 8][L][8] (he_spectral.cu cidx)
  uint64_t hint_g = 0x1000000000000000ULL;  // L2 policy of the G^ loads (normal: read by the 3 block tiles of one (y tile, f))
  uint64_t hint_a = 0x14F0000000000000ULL;  // of the A^ loads (evict-last: re-read by every y tile)
  uint64_t hint_c = 0x12F0000000000000ULL;  // of the C^ stores (evict-first: S4 reads them back much later)
};
struct SpecInvConst {
  uint32_t q[2];
  const uint2* iv[2];
  const uint2* r2[2];
  uint2 r1[2][26];          // round-1 twiddles of the fast inverse (spec_table_init)
  uint32_t linv[2], linvp[2];
  uint32_t q1inv, q1invp;
  uint32_t* out1 = nullptr;  // level-1 mode: no rescale; limb-0 words -> out_a, limb-1 words -> out1 (same layout)
  uint32_t q1bar = 0;        // floor(2^32 / q[1]) (set by launch_spec_inverse: the lazy q1 limb's final Barrett step)
};
cudaError_t launch_spec_weights(const int8_t* wdig, uint32_t d_w, uint32_t n_out, uint32_t n_in, uint32_t k,
                                const SpecTable& t, int D, uint32_t r_pad, int8_t* out, cudaStream_t s);
cudaError_t launch_spec_data(const RingDims& Rg, const uint32_t* ct, uint32_t n_ct, uint32_t limb, const SpecTable& t,
                             int D, uint32_t r_pad, uint32_t ob, uint32_t nblk, uint32_t nbp, int8_t* out,
                             cudaStream_t s);
// both limbs of S2 in one launch where the fast L = 1024 kernel applies (else two launch_spec_data calls)
cudaError_t launch_spec_data2(const RingDims& Rg, const uint32_t* ct, uint32_t n_ct, const SpecTable (&t)[2],
                              const int (&D)[2], uint32_t r_pad, uint32_t ob, uint32_t nblk, uint32_t nbp,
                              int8_t* const (&out)[2], cudaStream_t s);
cudaError_t launch_spec_gemm(int D, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                             const SpecGemmArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_spec_gemm_simple(int D, const int8_t* G, const int8_t* A, const SpecGemmArgs& a, cudaStream_t s);
cudaError_t launch_spec_inverse(const RingDims& Rg, const uint32_t* c0, const uint32_t* c1, uint32_t n_out,
                                uint32_t row0, uint32_t rows, uint32_t L, uint32_t nblk, uint32_t nbp,
                                const SpecInvConst& cst, uint32_t* out_a, const OutPeers& peers, cudaStream_t s);
cudaError_t launch_digitize(const RingDims& R, const uint32_t* ct, uint32_t n_ct, int d0, int d1, uint32_t S,
                            int8_t* out_a, int8_t* out_b, cudaStream_t s);
cudaError_t launch_weight_maxabs(const RingDims& R, const double* W, uint32_t n_out, uint32_t n_in,
                                 unsigned long long* maxabs, cudaStream_t s);
cudaError_t launch_encode_weights(const RingDims& R, const double* W, uint32_t n_out, uint32_t n_in, uint32_t dw,
                                  int8_t* planes, cudaStream_t s);
cudaError_t launch_keygen(const RingDims& R, uint64_t seed, int32_t* s_dev, cudaStream_t st);
cudaError_t launch_reduce_secret(const RingDims& R, const int32_t* s_dev, uint32_t limb, uint32_t* out,
                                 cudaStream_t st);
cudaError_t launch_gen_a(const RingDims& R, uint64_t seed, uint32_t r0, uint32_t n_ct, uint32_t* ct, cudaStream_t st);
cudaError_t launch_pointwise_mul(const uint32_t* x, uint64_t x_stride, const uint32_t* y, uint32_t n,
                                 uint32_t count, uint32_t q, uint32_t* out, uint64_t out_stride, cudaStream_t st);
cudaError_t launch_finish_encrypt(const RingDims& R, const double* acts, uint32_t n_in, uint64_t seed, uint32_t r0,
                                  uint32_t n_ct, uint32_t* ct, cudaStream_t st, int layout = 0,
                                  uint32_t win = 0);
cudaError_t launch_phase(const uint32_t* b, uint64_t b_stride, const uint32_t* as, uint64_t as_stride, uint32_t n,
                         uint32_t count, uint32_t q, int64_t* phase, cudaStream_t st);
cudaError_t launch_mlwe_rows_to_poly(const RingDims& R, const uint32_t* out_a, uint32_t row0, uint32_t rows, uint32_t* A,
                                     cudaStream_t st);
cudaError_t launch_mlwe_phase(const RingDims& R, const uint32_t* prod, const uint32_t* out_b, uint32_t row0,
                              uint32_t rows, int64_t* phase, cudaStream_t st);
cudaError_t launch_mod_raise(const RingDims& R, const uint32_t* ct, uint32_t n_ct, const uint32_t* primes_dev,
                             uint32_t n_primes, uint32_t* out, cudaStream_t st);
cudaError_t launch_decrypt_mlwe(const RingDims& R, const int32_t* s, const uint32_t* out_b, const uint32_t* out_a,
                                uint32_t n_out, uint32_t row0, uint32_t n_rows, int64_t* phase, cudaStream_t st);

}  // namespace he
