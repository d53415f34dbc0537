// he_abi.cu -- the extern "C" boundary (include/he_b200.h): argument validation, plan and
// context objects, TMA descriptor construction, and the launch sequence of each op.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "../../include/he_b200.h"
#include "he_common.cuh"
#include "he_kernels.h"

using namespace he;

#include "he_internal.h"

static thread_local std::string g_err;

he_status fail(he_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
he_status cuda_fail(cudaError_t e, const char* what) { return fail(HE_ECUDA, "%s: %s", what, cudaGetErrorString(e)); }

extern "C" const char* he_last_error(void) { return g_err.c_str(); }
extern "C" int he_version(void) { return 1; }

// ---------------------------------------------------------------- TMA descriptors
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled_t)p;
  }
  return fn;
}
// 3-D int8 tensor {inner, rows, planes}, box {128, box_rows, 1}, 128-B swizzle, OOB -> 0
static he_status make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t planes,
                          uint32_t box_rows, uint64_t plane_stride = 0) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return fail(HE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {inner, rows, planes};
  cuuint64_t strides[2] = {inner, plane_stride ? plane_stride : inner * rows};
  cuuint32_t box[3] = {128, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HE_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HE_OK;
}

// 3-D int8 tensor {inner, rows, planes}, box {box_inner, box_rows, 1}, 64-B swizzle (spectral operands)
static he_status make_map_sw64(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t planes,
                               uint32_t box_rows) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return fail(HE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {inner, rows, planes};
  cuuint64_t strides[2] = {inner, inner * rows};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HE_ECUDA, "cuTensorMapEncodeTiled (sw64) failed (%d)", (int)r);
  return HE_OK;
}

// 3-D u32 tensor {inner, rows, planes}, box {box_inner, box_rows, 1}, no swizzle
// extent <= inner: TMA clips stores past `extent` (the padding columns of a row of pitch `inner`)
static he_status make_map_u32(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint64_t planes,
                              uint32_t box_inner, uint32_t box_rows, uint64_t extent = 0) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return fail(HE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {extent ? extent : inner, rows, planes};
  cuuint64_t strides[2] = {inner * 4, inner * rows * 4};
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HE_ECUDA, "cuTensorMapEncodeTiled (u32) failed (%d)", (int)r);
  return HE_OK;
}

// S3's G^ map over the gidx layout: int8 [planes * row tiles][kg / 2 lines][256], box {256, kg / 2, 1}: one
// (digit plane, 128-row tile) = kg / 16 chunks of 128 rows x 16 B (no-swizzle core matrices) copied as is
static he_status make_map_g16(CUtensorMap* m, const void* base, uint64_t kg, uint64_t rows, uint64_t planes) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return fail(HE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const uint64_t tiles = planes * ((rows + 127) / 128);
  cuuint64_t dims[3] = {256, kg / 2, tiles};
  cuuint64_t strides[2] = {256, kg * 128};
  cuuint32_t box[3] = {256, (cuuint32_t)(kg < 64 ? kg / 2 : 32), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HE_ECUDA, "cuTensorMapEncodeTiled (G^) failed (%d)", (int)r);
  return HE_OK;
}

// S3's C^ store map: u32 [n_out][groups][L][8] (he_spectral.cu cidx), box {8, 1 f, 1 group, 32 rows}: one
// epilogue warp's 32 rows x 8 blocks of one frequency; groups past group_ext (all padding) are never stored
static he_status make_map_c4(CUtensorMap* m, const void* base, uint64_t groups, uint64_t L, uint64_t rows,
                             uint64_t group_ext) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return fail(HE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {8, L, group_ext, rows};
  cuuint64_t strides[3] = {8 * 4, L * 8 * 4, groups * L * 8 * 4};
  cuuint32_t box[4] = {8, 1, 1, 32};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HE_ECUDA, "cuTensorMapEncodeTiled (C^) failed (%d)", (int)r);
  return HE_OK;
}

// 4-D int8 tensor with explicit strides (bytes), box {128, box_rows, 1, 1}, 128-B swizzle
static he_status make_map4(CUtensorMap* m, const void* base, const uint64_t dims_in[4], const uint64_t strides_in[3],
                           uint32_t box_rows) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return fail(HE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {dims_in[0], dims_in[1], dims_in[2], dims_in[3]};
  cuuint64_t strides[3] = {strides_in[0], strides_in[1], strides_in[2]};
  cuuint32_t box[4] = {128, box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HE_ECUDA, "cuTensorMapEncodeTiled (4-D) failed (%d)", (int)r);
  return HE_OK;
}

// ---------------------------------------------------------------- context
static int digits_for(uint32_t q) {
  // balanced 8-bit digits for a centred residue |c| <= q/2
  uint64_t bound = q / 2;
  int n = 1;
  while (127ull * (((1ull << (8 * n)) - 1) / 255) < bound) ++n;
  return n;
}

extern "C" he_status he_context_create(const he_params* p, he_context** out) {
  if (!p || !out) return fail(HE_EINVAL, "null argument");
  const uint32_t d = p->mlwe_degree, k = p->mlwe_rank;
  if (d < 32 || d > 256 || (d & (d - 1))) return fail(HE_EINVAL, "mlwe_degree must be a power of two in [32, 256]");
  if (k < 16 || k > 256 || (k & (k - 1))) return fail(HE_EINVAL, "mlwe_rank must be a power of two in [16, 256]");
  const uint32_t N = d * k;
  for (int i = 0; i < 2; ++i) {
    uint32_t q = p->moduli[i];
    if (q < 3 || q >= (1u << 30) || (q - 1) % (2ull * N))
      return fail(HE_EINVAL, "modulus %u must be an NTT-friendly prime below 2^30", q);
  }
  if (p->moduli[1] / 2 >= p->moduli[0]) return fail(HE_EINVAL, "q1/2 must be below q0");
  {
    const uint32_t P = p->special_prime;
    if (P < 3 || P >= (1u << 30) || (P - 1) % (2ull * N) || P == p->moduli[0] || P == p->moduli[1])
      return fail(HE_EINVAL, "special prime %u must be NTT-friendly, below 2^30 and distinct from the moduli", P);
  }
  if (p->log_delta < 1 || p->log_delta > 40) return fail(HE_EINVAL, "log_delta out of range");
  if (p->rhombus_degree < 16 || (p->rhombus_degree & (p->rhombus_degree - 1)) || N % p->rhombus_degree)
    return fail(HE_EINVAL, "rhombus_degree must be a power of two dividing N");
  he_context* c = new (std::nothrow) he_context();
  if (!c) return fail(HE_ENOMEM, "out of host memory");
  c->p = *p;
  c->R.d = d;
  c->R.k = k;
  c->R.N = N;
  c->R.logk = (uint32_t)ilog2_h(k);
  c->R.q[0] = p->moduli[0];
  c->R.q[1] = p->moduli[1];
  c->R.log_delta = p->log_delta;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, dev);
  c->R.n_rh = p->rhombus_degree;
  c->R.P = p->special_prime;
  for (int i = 0; i < 3; ++i) {
    const uint32_t q = i < 2 ? p->moduli[i] : p->special_prime;
    cudaError_t e = ntt_table_init(c->ntt[i], N, q);
    if (e == cudaSuccess) e = ntt_table_init(c->ntt_rh[i], p->rhombus_degree, q);
    if (e != cudaSuccess) {
      he_context_destroy(c);
      return cuda_fail(e, "NTT table init");
    }
  }
  *out = c;
  return HE_OK;
}

extern "C" he_status he_context_set_rng_key(he_context* c, const uint8_t* key) {
  if (!c) return fail(HE_EINVAL, "null argument");
  if (!key) {
    c->R.rng = he::RngCtx{};
    return HE_OK;
  }
  for (int i = 0; i < 8; ++i)
    c->R.rng.key[i] = (uint32_t)key[4 * i] | ((uint32_t)key[4 * i + 1] << 8) | ((uint32_t)key[4 * i + 2] << 16) |
                      ((uint32_t)key[4 * i + 3] << 24);
  c->R.rng.secure = 1;
  return HE_OK;
}

extern "C" he_status he_chacha20_block(const uint8_t* key, uint32_t counter, const uint8_t* nonce, uint8_t* out) {
  if (!key || !nonce || !out) return fail(HE_EINVAL, "null argument");
  uint32_t k[8], n[3], b[16];
  auto le = [](const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
  };
  for (int i = 0; i < 8; ++i) k[i] = le(key + 4 * i);
  for (int i = 0; i < 3; ++i) n[i] = le(nonce + 4 * i);
  he::chacha20_block(k, counter, n[0], n[1], n[2], b);
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 4; ++j) out[4 * i + j] = (uint8_t)(b[i] >> (8 * j));
  return HE_OK;
}

extern "C" he_status he_context_destroy(he_context* c) {
  if (!c) return HE_OK;
  for (int i = 0; i < 3; ++i) {
    ntt_table_free(c->ntt[i]);
    ntt_table_free(c->ntt_rh[i]);
  }
  delete c;
  return HE_OK;
}

// ---------------------------------------------------------------- keys / encryption
extern "C" he_status he_keygen(const he_context* c, uint64_t seed, int32_t* s_dev, uint32_t* s_ntt_dev, void* stream) {
  if (!c || !s_dev || !s_ntt_dev) return fail(HE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  HE_CUDA(launch_keygen(c->R, seed, s_dev, st), "keygen");
  for (uint32_t L = 0; L < 2; ++L) {
    uint32_t* dst = s_ntt_dev + (size_t)L * c->R.N;
    HE_CUDA(launch_reduce_secret(c->R, s_dev, L, dst, st), "reduce secret");
    HE_CUDA(ntt_forward(c->ntt[L], dst, 1, c->R.N, st), "secret NTT");
  }
  return HE_OK;
}

extern "C" he_status he_encrypt_acts(const he_context* c, const uint32_t* s_ntt_dev, const double* acts_dev,
                                     uint32_t n_in, uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream) {
  if (!c || !s_ntt_dev || !acts_dev || !ct_dev) return fail(HE_EINVAL, "null argument");
  if (n_in == 0 || n_in % c->R.k) return fail(HE_EINVAL, "n_in (%u) must be a positive multiple of k = %u", n_in, c->R.k);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N, n_ct = n_in / c->R.k;
  HE_CUDA(launch_gen_a(c->R, seed, r0, n_ct, ct_dev, st), "sample a");
  for (uint32_t L = 0; L < 2; ++L) {
    uint32_t* bslots = ct_dev + (size_t)L * 2 * N + N;  // stride 4N between cts
    HE_CUDA(ntt_forward(c->ntt[L], bslots, n_ct, 4ull * N, st), "NTT(a)");
    HE_CUDA(launch_pointwise_mul(bslots, 4ull * N, s_ntt_dev + (size_t)L * N, N, n_ct, c->R.q[L], bslots, 4ull * N, st),
            "a^ * s^");
    HE_CUDA(ntt_inverse(c->ntt[L], bslots, n_ct, 4ull * N, st), "INTT(a s)");
  }
  HE_CUDA(launch_finish_encrypt(c->R, acts_dev, n_in, seed, r0, n_ct, ct_dev, st), "finish encrypt");
  return HE_OK;
}

extern "C" he_status he_encrypt_vector_w(const he_context* c, const uint32_t* s_ntt_dev, const double* v_dev,
                                         uint32_t n_vals, uint32_t window, uint64_t seed, uint32_t r0, uint32_t* ct_dev,
                                         void* stream) {
  if (!c || !s_ntt_dev || !v_dev || !ct_dev) return fail(HE_EINVAL, "null argument");
  const uint32_t n = c->R.n_rh, rho = c->R.N / n;
  if (window == 0 || window > n || (window & (window - 1)))
    return fail(HE_EINVAL, "window %u must be a power of two in [1, %u]", window, n);
  if (n_vals == 0 || n_vals > (uint64_t)window * rho)
    return fail(HE_EINVAL, "vector length %u outside [1, %u] (window %u x %u pieces)", n_vals, window * rho, window, rho);
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N;
  HE_CUDA(launch_gen_a(c->R, seed, r0, 1, ct_dev, st), "sample a");
  for (uint32_t L = 0; L < 2; ++L) {
    uint32_t* bslot = ct_dev + (size_t)L * 2 * N + N;
    HE_CUDA(ntt_forward(c->ntt[L], bslot, 1, N, st), "NTT(a)");
    HE_CUDA(launch_pointwise_mul(bslot, N, s_ntt_dev + (size_t)L * N, N, 1, c->R.q[L], bslot, N, st), "a^ * s^");
    HE_CUDA(ntt_inverse(c->ntt[L], bslot, 1, N, st), "INTT(a s)");
  }
  HE_CUDA(launch_finish_encrypt(c->R, v_dev, n_vals, seed, r0, 1, ct_dev, st, 1, window), "finish encrypt");
  return HE_OK;
}

extern "C" he_status he_encrypt_vector(const he_context* c, const uint32_t* s_ntt_dev, const double* v_dev,
                                       uint32_t n_vals, uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream) {
  if (!c) return fail(HE_EINVAL, "null argument");
  return he_encrypt_vector_w(c, s_ntt_dev, v_dev, n_vals, c->R.n_rh, seed, r0, ct_dev, stream);
}

extern "C" he_status he_encrypt_poly(const he_context* c, const uint32_t* s_ntt_dev, const int64_t* pt_dev,
                                     uint32_t n_ct, uint64_t seed, uint32_t r0, uint32_t* ct_dev, void* stream) {
  if (!c || !s_ntt_dev || !pt_dev || !ct_dev) return fail(HE_EINVAL, "null argument");
  if (n_ct == 0) return fail(HE_EINVAL, "no plaintexts");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N;
  HE_CUDA(launch_gen_a(c->R, seed, r0, n_ct, ct_dev, st), "sample a");
  for (uint32_t L = 0; L < 2; ++L) {
    uint32_t* bslots = ct_dev + (size_t)L * 2 * N + N;
    HE_CUDA(ntt_forward(c->ntt[L], bslots, n_ct, 4ull * N, st), "NTT(a)");
    HE_CUDA(launch_pointwise_mul(bslots, 4ull * N, s_ntt_dev + (size_t)L * N, N, n_ct, c->R.q[L], bslots, 4ull * N, st),
            "a^ * s^");
    HE_CUDA(ntt_inverse(c->ntt[L], bslots, n_ct, 4ull * N, st), "INTT(a s)");
  }
  HE_CUDA(launch_finish_encrypt(c->R, reinterpret_cast<const double*>(pt_dev), N, seed, r0, n_ct, ct_dev, st, 2),
          "finish encrypt");
  return HE_OK;
}

extern "C" he_status he_mod_raise(const he_context* c, const uint32_t* ct_dev, uint32_t n_ct, const uint32_t* primes_dev,
                                  uint32_t n_primes, uint32_t* out_dev, void* stream) {
  if (!c || !ct_dev || !primes_dev || !out_dev) return fail(HE_EINVAL, "null argument");
  if (n_ct == 0 || n_primes == 0 || n_primes > 64) return fail(HE_EINVAL, "need 1..64 target primes and >= 1 ciphertext");
  HE_CUDA(launch_mod_raise(c->R, ct_dev, n_ct, primes_dev, n_primes, out_dev, (cudaStream_t)stream), "mod raise");
  return HE_OK;
}

extern "C" he_status he_decrypt_rlwe(const he_context* c, const uint32_t* s_ntt_dev, const uint32_t* ct_dev,
                                     uint32_t n_ct, uint32_t limbs, uint32_t limb, int64_t* phase_dev, void* stream) {
  if (!c || !s_ntt_dev || !ct_dev || !phase_dev) return fail(HE_EINVAL, "null argument");
  if (limb >= limbs || limbs > 2 || n_ct == 0) return fail(HE_EINVAL, "bad limb / limbs / n_ct");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t N = c->R.N;
  uint32_t* tmp = nullptr;
  HE_CUDA(cudaMallocAsync(&tmp, (size_t)n_ct * N * sizeof(uint32_t), st), "alloc");
  const uint64_t cstride = (uint64_t)limbs * 2 * N;
  const uint32_t* a = ct_dev + (size_t)limb * 2 * N;
  cudaError_t e = cudaMemcpy2DAsync(tmp, N * sizeof(uint32_t), a, cstride * sizeof(uint32_t), N * sizeof(uint32_t),
                                    n_ct, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = ntt_forward(c->ntt[limb], tmp, n_ct, N, st);
  if (e == cudaSuccess)
    e = launch_pointwise_mul(tmp, N, s_ntt_dev + (size_t)limb * N, N, n_ct, c->R.q[limb], tmp, N, st);
  if (e == cudaSuccess) e = ntt_inverse(c->ntt[limb], tmp, n_ct, N, st);
  if (e == cudaSuccess) e = launch_phase(a + N, cstride, tmp, N, N, n_ct, c->R.q[limb], phase_dev, st);
  cudaFreeAsync(tmp, st);
  if (e != cudaSuccess) return cuda_fail(e, "decrypt");
  return HE_OK;
}

extern "C" he_status he_decrypt_mlwe(const he_context* c, const int32_t* s_dev, const uint32_t* out_b_dev,
                                     const uint32_t* out_a_dev, uint32_t n_out, uint32_t row0, uint32_t n_rows,
                                     int64_t* phase_dev, void* stream) {
  if (!c || !s_dev || !out_b_dev || !out_a_dev || !phase_dev) return fail(HE_EINVAL, "null argument");
  if (row0 + n_rows > n_out || n_out % c->R.k) return fail(HE_EINVAL, "row range outside the output");
  if (n_rows == 0) return HE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  static const bool direct = getenv("HE_DECRYPT_MLWE_DIRECT") != nullptr;   // the O(k d^2) convolution kernel
  if (direct || c->R.k > 256 || c->R.d % 32) {
    HE_CUDA(launch_decrypt_mlwe(c->R, s_dev, out_b_dev, out_a_dev, n_out, row0, n_rows, phase_dev, st), "decrypt mlwe");
    return HE_OK;
  }
  // RLWE view: one degree-N NTT product per row (rows in chunks of 256: 64 MB of scratch)
  const uint32_t N = c->R.N, chunk = n_rows < 256 ? n_rows : 256;
  uint32_t* buf = nullptr;
  HE_CUDA(cudaMallocAsync(&buf, ((size_t)chunk + 1) * N * sizeof(uint32_t), st), "alloc");
  uint32_t* sh = buf + (size_t)chunk * N;
  HE_CUDA(launch_reduce_secret(c->R, s_dev, 0, sh, st), "s mod q0");
  HE_CUDA(ntt_forward(c->ntt[0], sh, 1, N, st), "NTT(s)");
  for (uint32_t r0 = 0; r0 < n_rows; r0 += chunk) {
    const uint32_t rows = n_rows - r0 < chunk ? n_rows - r0 : chunk;
    HE_CUDA(launch_mlwe_rows_to_poly(c->R, out_a_dev, row0 + r0, rows, buf, st), "a' -> A");
    HE_CUDA(ntt_forward(c->ntt[0], buf, rows, N, st), "NTT(A)");
    HE_CUDA(launch_pointwise_mul(buf, N, sh, N, rows, c->R.q[0], buf, N, st), "A^ s^");
    HE_CUDA(ntt_inverse(c->ntt[0], buf, rows, N, st), "INTT(A s)");
    HE_CUDA(launch_mlwe_phase(c->R, buf, out_b_dev, row0 + r0, rows, phase_dev + (size_t)r0 * c->R.d, st), "phase");
  }
  cudaFreeAsync(buf, st);
  return HE_OK;
}

// ---------------------------------------------------------------- NTT
static const NttTable* pick(const he_context* c, uint32_t n, uint32_t limb) {
  if (limb > 2) return nullptr;  // 2 = the special prime P
  if (n == c->R.N) return &c->ntt[limb];
  if (n == c->p.rhombus_degree) return &c->ntt_rh[limb];
  return nullptr;
}
extern "C" he_status he_ntt_forward(const he_context* c, uint32_t* data, uint32_t n, uint32_t limb, uint32_t count,
                                    uint64_t stride, void* stream) {
  if (!c || !data) return fail(HE_EINVAL, "null argument");
  const NttTable* t = pick(c, n, limb);
  if (!t) return fail(HE_EINVAL, "no NTT table for degree %u limb %u", n, limb);
  if (stride < n || stride % 4) return fail(HE_EINVAL, "stride must be >= n and a multiple of 4");
  HE_CUDA(ntt_forward(*t, data, count, stride, (cudaStream_t)stream), "ntt forward");
  return HE_OK;
}
extern "C" he_status he_ntt_inverse(const he_context* c, uint32_t* data, uint32_t n, uint32_t limb, uint32_t count,
                                    uint64_t stride, void* stream) {
  if (!c || !data) return fail(HE_EINVAL, "null argument");
  const NttTable* t = pick(c, n, limb);
  if (!t) return fail(HE_EINVAL, "no NTT table for degree %u limb %u", n, limb);
  if (stride < n || stride % 4) return fail(HE_EINVAL, "stride must be >= n and a multiple of 4");
  HE_CUDA(ntt_inverse(*t, data, count, stride, (cudaStream_t)stream), "ntt inverse");
  return HE_OK;
}

// ---------------------------------------------------------------- PCMM
static he_status check_shape(const he_context* c, uint32_t n_out, uint32_t n_in) {
  if (n_out == 0 || n_in == 0) return fail(HE_EINVAL, "empty weight matrix");
  if (n_out % c->R.k || n_in % c->R.k)
    return fail(HE_EINVAL, "dim mismatch: n_out (%u) and n_in (%u) must be multiples of k = %u", n_out, n_in, c->R.k);
  return HE_OK;
}

extern "C" he_status he_pcmm_weight_maxabs(const he_context* c, const double* w_dev, uint32_t n_out, uint32_t n_in,
                                           uint64_t* maxabs_out, void* stream) {
  if (!c || !w_dev || !maxabs_out) return fail(HE_EINVAL, "null argument");
  he_status s = check_shape(c, n_out, n_in);
  if (s) return s;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* dmax = nullptr;
  HE_CUDA(cudaMallocAsync(&dmax, sizeof(unsigned long long), st), "alloc");
  cudaError_t e = cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = launch_weight_maxabs(c->R, w_dev, n_out, n_in, dmax, st);
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, dmax, sizeof h, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(dmax, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "weight max");
  *maxabs_out = h;
  return HE_OK;
}

extern "C" he_status he_pcmm_encode_weights(const he_context* c, const double* w_dev, uint32_t n_out, uint32_t n_in,
                                            uint32_t d_w, int8_t* digits_dev, void* stream) {
  if (!c || !w_dev || !digits_dev) return fail(HE_EINVAL, "null argument");
  he_status s = check_shape(c, n_out, n_in);
  if (s) return s;
  if (d_w < 1 || d_w > 4) return fail(HE_EINVAL, "d_w must be in [1, 4]");
  HE_CUDA(launch_encode_weights(c->R, w_dev, n_out, n_in, d_w, digits_dev, (cudaStream_t)stream), "encode weights");
  return HE_OK;
}

extern "C" he_status he_pcmm_plan_create(const he_context* c, const int8_t* digits_dev, uint32_t n_out, uint32_t n_in,
                                         uint32_t d_w, he_pcmm_plan** out) {
  if (!c || !digits_dev || !out) return fail(HE_EINVAL, "null argument");
  he_status s = check_shape(c, n_out, n_in);
  if (s) return s;
  if (d_w < 1 || d_w > 4) return fail(HE_EINVAL, "d_w must be in [1, 4]");
  const int d0 = digits_for(c->R.q[0]), d1 = digits_for(c->R.q[1]);
  if (gemm_smem_bytes((int)d_w, d0, d1) < 0)
    return fail(HE_EINVAL, "no GEMM instance for digits (%u, %d, %d)", d_w, d0, d1);
  // exactness bounds of K1 (|digit product| <= 2^14):
  //   int32 shift accumulator:    n_in * 2^14 * max_s pairs(s) < 2^31
  //   int64 recombination (S<=5): n_in * 2^14 * sum_s pairs(s) 2^(8s) < 2^62
  for (int L = 0; L < 2; ++L) {
    const int dl = L ? d1 : d0, S = (int)d_w + dl - 1;
    unsigned __int128 sum = 0;
    int maxp = 0;
    for (int sft = 0; sft < S; ++sft) {
      int pairs = 0;
      for (int a = 0; a < (int)d_w; ++a)
        if (sft - a >= 0 && sft - a < dl) ++pairs;
      maxp = pairs > maxp ? pairs : maxp;
      sum += (unsigned __int128)pairs << (8 * sft);
    }
    if ((uint64_t)n_in * 16384ull * (uint64_t)maxp >= (1ull << 31))
      return fail(HE_EINVAL, "n_in (%u) overflows the int32 digit accumulators at d_w = %u", n_in, d_w);
    if (S <= 5 && (unsigned __int128)n_in * 16384u * sum >= ((unsigned __int128)1 << 62))
      return fail(HE_EINVAL, "n_in (%u) overflows the int64 recombination at d_w = %u", n_in, d_w);
  }
  he_pcmm_plan* p = new (std::nothrow) he_pcmm_plan();
  if (!p) return fail(HE_ENOMEM, "out of host memory");
  p->ctx = c;
  p->n_out = n_out;
  p->n_in = n_in;
  p->d_w = d_w;
  p->d0 = (uint32_t)d0;
  p->d1 = (uint32_t)d1;
  p->width = c->R.d * (1 + c->R.k);
  p->digits = digits_dev;
  s = make_map(&p->tmA, digits_dev, n_in, n_out, d_w, 128);
  if (s) {
    delete p;
    return s;
  }
  GemmEpiConst& e = p->epi;
  for (int L = 0; L < 2; ++L) {
    const uint32_t q = c->R.q[L];
    e.q[L] = q;
    e.offs[L] = (uint32_t)((uint64_t)q * (((1ull << 31) + q - 1) / q));
    for (int sft = 0; sft < 8; ++sft) {
      uint32_t w = (uint32_t)powmod_h(2, 8ull * sft, q);
      e.pw[L][sft] = w;
      e.pwp[L][sft] = shoup_pre(w, q);
    }
  }
  for (int L = 0; L < 2; ++L) {
    const uint64_t q = c->R.q[L];
    e.off64[L] = q * (((1ull << 62) + q - 1) / q);
    e.mu[L] = (uint64_t)(((unsigned __int128)1 << 64) / q);
  }
  e.q1inv = (uint32_t)powmod_h(c->R.q[1] % c->R.q[0], c->R.q[0] - 2, c->R.q[0]);
  e.q1invp = shoup_pre(e.q1inv, c->R.q[0]);
  *out = p;
  return HE_OK;
}

extern "C" he_status he_pcmm_plan_destroy(he_pcmm_plan* p) {
  delete p;
  return HE_OK;
}

// K3 fused into K1 (compact digit planes + 16-byte shifted copies) -- opt-in (HE_GEMM_FUSED=1).
// Measured (profiles/r01/ncu_full_modgemm_fused.json): DRAM reads 56 -> 2.2 GB per launch, but the
// 16-B-aligned window rows split every 128-B TMA row over two L2 lines, doubling L2 requests; K1 is
// L2-request-rate bound at ~6e10 requests/s, so the fused GEMM takes 54 ms vs 25 ms materialised.
// Valid when the K-blocks of 128 stay inside one RLWE ct and the 32-column tiles inside one key
// component: k % 128 == 0, d % 32 == 0.
static int gemm_variant() {
  static int variant = [] {
    const char* v = getenv("HE_GEMM_VARIANT");  // profiling switch: 1 = single-CTA kernel
    return (v && v[0] == '1') ? 1 : 2;
  }();
  return variant;
}
static bool fused_path(const he_pcmm_plan* p) {
  static const bool on = getenv("HE_GEMM_FUSED") != nullptr;  // profiling switch
  const uint32_t k = p->ctx->R.k, d = p->ctx->R.d;
  return on && gemm_variant() == 2 && k % 128 == 0 && d % 32 == 0;
}
static uint64_t fused_stride(const he_pcmm_plan* p) { return (uint64_t)p->ctx->R.N + 2ull * p->ctx->R.k; }
static uint64_t fused_a_bytes(const he_pcmm_plan* p) {
  return 16ull * (p->d0 + p->d1) * (p->n_in / p->ctx->R.k) * fused_stride(p);
}
// spectral workspace: [K3 b-column digit planes][A^ limb 0][A^ limb 1][C^ limb 0][C^ limb 1], 256-B aligned
struct SpecWs {
  uint64_t bdig, a0, a1, c0, c1, total;
};
static uint64_t al256(uint64_t x) { return (x + 255) & ~255ull; }
static SpecWs spec_ws(const he_pcmm_plan* p) {
  const uint64_t d = p->ctx->R.d;
  SpecWs w;
  w.bdig = 0;
  w.a0 = al256((uint64_t)(p->d0 + p->d1) * d * p->n_in);
  const uint64_t nb = p->nbp;
  w.a1 = w.a0 + al256((uint64_t)p->L * p->dsp[0] * nb * p->r_pad);
  w.c0 = w.a1 + al256((uint64_t)p->L * p->dsp[1] * nb * p->r_pad);
  w.c1 = w.c0 + al256((uint64_t)p->L * p->n_out * nb * 4);
  w.total = w.c1 + al256((uint64_t)p->L * p->n_out * nb * 4);
  return w;
}
static uint64_t ws_bytes(const he_pcmm_plan* p) {
  if (p->algo == 1) return spec_ws(p).total;
  if (fused_path(p))
    return fused_a_bytes(p) + (uint64_t)(p->d0 + p->d1) * (p->n_in / p->ctx->R.k) * p->ctx->R.N;
  return (uint64_t)(p->d0 + p->d1) * p->width * p->n_in;
}

extern "C" he_status he_pcmm_workspace_bytes(const he_pcmm_plan* p, uint64_t* bytes) {
  if (!p || !bytes) return fail(HE_EINVAL, "null argument");
  *bytes = ws_bytes(p);
  return HE_OK;
}

extern "C" he_status he_pcmm_decompose(const he_pcmm_plan* p, const uint32_t* ct_in, void* ws, uint64_t ws_size,
                                       void* stream) {
  if (!p || !ct_in || !ws) return fail(HE_EINVAL, "null argument");
  if (ws_size < ws_bytes(p)) return fail(HE_EINVAL, "workspace too small (%llu < %llu)", (unsigned long long)ws_size,
                                         (unsigned long long)ws_bytes(p));
  if (p->algo == 1) {
    const SpecWs w = spec_ws(p);
    cudaStream_t st = (cudaStream_t)stream;
    int8_t* base = (int8_t*)ws;
    p->prof_begin(0, st);
    HE_CUDA(launch_decompose(p->ctx->R, ct_in, p->n_in, (int)p->d0, (int)p->d1, base + w.bdig,
                             (uint64_t)p->ctx->R.d * p->n_in, st, 1),
            "decompose (b columns)");
    p->prof_end(0, st);
    p->prof_begin(1, st);
    HE_CUDA(cudaMemsetAsync(base + w.a0, 0, w.c0 - w.a0, st), "memset");
    const uint32_t n_ct = p->n_in / p->ctx->R.k;
    const int D[2] = {(int)p->dsp[0], (int)p->dsp[1]};
    int8_t* const outs[2] = {base + w.a0, base + w.a1};
    HE_CUDA(launch_spec_data2(p->ctx->R, ct_in, n_ct, p->st, D, p->r_pad, p->ob, p->nblk, p->nbp, outs, st),
            "spectral data transform");
    p->prof_end(1, st);
    return HE_OK;
  }
  if (fused_path(p)) {
    HE_CUDA(launch_digitize(p->ctx->R, ct_in, p->n_in / p->ctx->R.k, (int)p->d0, (int)p->d1, (uint32_t)fused_stride(p),
                            (int8_t*)ws, (int8_t*)ws + fused_a_bytes(p), (cudaStream_t)stream),
            "digitize");
    return HE_OK;
  }
  p->prof_begin(0, (cudaStream_t)stream);
  HE_CUDA(launch_decompose(p->ctx->R, ct_in, p->n_in, (int)p->d0, (int)p->d1, (int8_t*)ws,
                           (uint64_t)p->width * p->n_in, (cudaStream_t)stream),
          "decompose");
  p->prof_end(0, (cudaStream_t)stream);
  return HE_OK;
}

// K7 S3 (per-frequency tcgen05 GEMM, both limbs) + S4 (inverse, rescale, a' store) on rows [row0, row0 + rows)
static he_status spec_rows(const he_pcmm_plan* p, const void* ws, uint32_t row0, uint32_t rows, uint32_t* out_a,
                           uint32_t* out1_a, const OutPeers& peers, cudaStream_t st) {
  const SpecWs w = spec_ws(p);
  const int8_t* base = (const int8_t*)ws;
  static const bool simple = getenv("HE_SPEC_SIMPLE") != nullptr;  // debug: S3 on CUDA cores
  uint32_t* C[2] = {(uint32_t*)(base + w.c0), (uint32_t*)(base + w.c1)};
  for (int L = 0; L < 2; ++L) {
    SpecGemmArgs a;
    a.n_rows = (int)rows;
    a.row0 = (int)row0;
    a.n_out = (int)p->n_out;
    a.L = (int)p->L;
    a.nb = (int)p->nbp;
    a.r_pad = (int)p->r_pad;
    a.kg = (int)p->kg;
    const uint32_t q = p->epi.q[L];
    a.q = q;
    uint32_t inv = 1;  // q^-1 mod 2^32 by Newton iteration
    for (int it = 0; it < 5; ++it) inv *= 2u - q * inv;
    a.qninv = 0u - inv;
    a.off64 = p->spec_off[L];
    for (int i = 0; i < 8; ++i) a.pw[i] = (int32_t)powmod_h(2, 16ull * i + 32, q);
    a.out = C[L];
    // S3 L2 policy (tiles run y-tile-major, SpecGemmArgs): G^ normal, A^ evict-last, C^ stores evict-first (measured
    // 1.02 ms for both limbs at 4096x11008 vs 1.10 with G^ evict-last, 1.39 with G^ evict-first);
    // HE_S3_HINTS=<g><a><c> (digits 0 first / 1 normal / 2 last) overrides for measurements
    if (const char* h = getenv("HE_S3_HINTS")) {
      static const uint64_t pol[3] = {0x12F0000000000000ULL, 0x1000000000000000ULL, 0x14F0000000000000ULL};
      if (strlen(h) == 3) {
        a.hint_g = pol[(h[0] - '0') % 3];
        a.hint_a = pol[(h[1] - '0') % 3];
        a.hint_c = pol[(h[2] - '0') % 3];
      }
    }
    const int8_t* A = base + (L ? w.a1 : w.a0);
    if (simple) {
      const int8_t* G = p->spec_w + (L ? (uint64_t)p->L * p->dsp[0] * ((p->n_out + 127) / 128 * 128) * p->kg : 0);
      HE_CUDA(launch_spec_gemm_simple((int)p->dsp[L], G, A, a, st), "spectral gemm (simple)");
      continue;
    }
    CUtensorMap tmB;
    he_status s = make_map_sw64(&tmB, A, p->r_pad, p->nbp, (uint64_t)p->L * p->dsp[L], 16);
    if (s) return s;
    CUtensorMap tmC;  // C^ limb L: u32 [n_out][nbp / 8][L][8] (cidx), box {8 blocks, 1 f, 1 group, 32 rows}
    s = make_map_c4(&tmC, C[L], p->nbp / 8, p->L, p->n_out, (p->nblk + 7) / 8);  // all-padding groups never stored
    if (s) return s;
    p->prof_begin(3 + L, st);
    HE_CUDA(launch_spec_gemm((int)p->dsp[L], p->tmSA[L], tmB, tmC, a, p->ctx->sm_count, st), "spectral gemm");
    p->prof_end(3 + L, st);
  }
  SpecInvConst c;
  for (int L = 0; L < 2; ++L) {
    c.q[L] = p->epi.q[L];
    c.iv[L] = p->st[L].iv;
    c.r2[L] = p->st[L].r2;
    for (int i = 0; i < 26; ++i) c.r1[L][i] = p->st[L].r1[i];
    c.linv[L] = p->st[L].linv;
    c.linvp[L] = p->st[L].linvp;
  }
  c.q1inv = p->epi.q1inv;
  c.q1invp = p->epi.q1invp;
  c.out1 = out1_a;
  p->prof_begin(5, st);
  HE_CUDA(launch_spec_inverse(p->ctx->R, C[0], C[1], p->n_out, row0, rows, p->L, p->nblk, p->nbp, c, out_a, peers, st),
          "spectral inverse");
  p->prof_end(5, st);
  return HE_OK;
}

static he_status gemm_rows_impl(const he_pcmm_plan* p, const void* ws, uint32_t row0, uint32_t rows, uint32_t* out_b,
                                uint32_t* out_a, const OutPeers& peers, void* stream, uint32_t* out1_b = nullptr,
                                uint32_t* out1_a = nullptr) {
  if (!p || !ws || (peers.n == 0 && (!out_b || !out_a))) return fail(HE_EINVAL, "null argument");
  if (rows == 0 || row0 % p->ctx->R.k || rows % p->ctx->R.k || row0 + rows > p->n_out)
    return fail(HE_EINVAL, "row range [%u, %u) must be k-aligned and inside [0, %u)", row0, row0 + rows, p->n_out);
  const int variant = (p->algo == 1 || out1_b) ? 2 : gemm_variant();
  const bool fused = p->algo != 1 && fused_path(p);
  const bool spec = p->algo == 1;
  const uint32_t gemm_width = spec ? p->ctx->R.d : p->width;  // spectral: K1 on the b' columns only
  // profiling knobs (defaults are the tuned choice): HE_GEMM_BN, HE_GEMM_GROUP_M, HE_GEMM_HINT_A/B
  static const int env_bn = getenv("HE_GEMM_BN") ? atoi(getenv("HE_GEMM_BN")) : 0;
  static const int env_gm = getenv("HE_GEMM_GROUP_M") ? atoi(getenv("HE_GEMM_GROUP_M")) : 0;
  auto hint = [](const char* name, uint64_t dflt) -> uint64_t {
    const char* v = getenv(name);
    if (!v) return dflt;
    if (v[0] == 'f') return 0x12F0000000000000ULL;  // evict_first
    if (v[0] == 'l') return 0x14F0000000000000ULL;  // evict_last
    return 0x1000000000000000ULL;                   // evict_normal
  };
  int bn2 = gemm2_tile_n((int)p->d_w, (int)p->d0, (int)p->d1);
  if (env_bn == 32 || (env_bn == 48 && bn2 == 48)) bn2 = env_bn;
  if (fused) bn2 = 32;  // tiles must not straddle a key component j
  // the spectral path's K1 only forms the d b' columns: 32-column tiles give 128 instead of 96 pair tiles at
  // d = 256 (no ragged last tile; 0.147 -> 0.107 ms at 4096x11008)
  if (spec && env_bn == 0) bn2 = 32;
  CUtensorMap tmB, tmBa;
  he_status s;
  if (fused) {
    const uint64_t n_ct = p->n_in / p->ctx->R.k, k = p->ctx->R.k, N = p->ctx->R.N, S = fused_stride(p);
    const uint64_t planes = p->d0 + p->d1;
    const uint64_t bd[4] = {k, p->ctx->R.d, n_ct, planes}, bs[3] = {k, N, N * n_ct};
    s = make_map4(&tmB, (const int8_t*)ws + fused_a_bytes(p), bd, bs, bn2 / 2);
    if (s) return s;
    // overlapping rows: extent k + 128 bytes, stride k bytes (every window starts 16-B aligned)
    const uint64_t ad[4] = {k + 128, N / k + 2, n_ct, 16 * planes}, as[3] = {k, S, S * n_ct};
    s = make_map4(&tmBa, ws, ad, as, bn2 / 2);
    if (s) return s;
  } else {
    s = make_map(&tmB, ws, p->n_in, gemm_width, p->d0 + p->d1, variant == 1 ? kGemmBoxRows1 : bn2 / 2);
    if (s) return s;
    tmBa = tmB;
  }
  CUtensorMap tmA = p->tmA;
  if (row0 != 0 || rows != p->n_out) {
    s = make_map(&tmA, p->digits + (size_t)row0 * p->n_in, p->n_in, rows, p->d_w, 128, (uint64_t)p->n_out * p->n_in);
    if (s) return s;
  }
  GemmArgs a;
  a.n_out = (int)rows;
  a.n_in = (int)p->n_in;
  a.width = (int)gemm_width;
  a.d = (int)p->ctx->R.d;
  a.k = (int)p->ctx->R.k;
  a.out_b = out_b;
  a.out_a = out_a;
  a.out1_b = out1_b;
  a.out1_a = out1_a;
  a.peers = peers;
  a.c = p->epi;
  a.group_m = env_gm > 0 ? env_gm : 8;
  a.tile_n = bn2;
  a.fused = fused ? 1 : 0;
  static const int env_skip = getenv("HE_GEMM_EPI_SKIP") ? 1 : 0;
  a.epi_skip = env_skip;
  a.hint_a = hint("HE_GEMM_HINT_A", 0x14F0000000000000ULL);
  a.hint_b = hint("HE_GEMM_HINT_B", 0x1000000000000000ULL);  // evict_normal: measured 46 vs 64 GB DRAM reads
  int grid;
  if (variant == 1) {
    const int tiles = (int)((rows + 127) / 128) * (int)(p->width / 32);
    grid = tiles < p->ctx->sm_count ? tiles : p->ctx->sm_count;
  } else {
    const int tiles = (int)((rows + 255) / 256) * (int)((gemm_width + bn2 - 1) / bn2);
    static const int env_pairs = getenv("HE_GEMM_PAIRS") ? atoi(getenv("HE_GEMM_PAIRS")) : 0;  // profiling knob
    int pairs = p->ctx->sm_count / 2;
    if (env_pairs > 0 && env_pairs < pairs) pairs = env_pairs;
    grid = 2 * (tiles < pairs ? tiles : pairs);
  }
  p->prof_begin(2, (cudaStream_t)stream);
  HE_CUDA(launch_modgemm(variant, (int)p->d_w, (int)p->d0, (int)p->d1, tmA, tmB, tmBa, a, grid, (cudaStream_t)stream),
          "modgemm");
  p->prof_end(2, (cudaStream_t)stream);
  if (spec) return spec_rows(p, ws, row0, rows, out_a, out1_a, peers, (cudaStream_t)stream);
  return HE_OK;
}

extern "C" he_status he_pcmm_gemm_rows(const he_pcmm_plan* p, const void* ws, uint32_t row0, uint32_t rows,
                                       uint32_t* out_b, uint32_t* out_a, void* stream) {
  OutPeers none{};
  none.n = 0;
  return gemm_rows_impl(p, ws, row0, rows, out_b, out_a, none, stream);
}

extern "C" he_status he_pcmm_gemm_rows_peers(const he_pcmm_plan* p, const void* ws, uint32_t row0, uint32_t rows,
                                             uint32_t* const* out_b_peers, uint32_t* const* out_a_peers,
                                             uint32_t n_peers, uint32_t dst_row0, void* stream) {
  if (!p || !out_b_peers || !out_a_peers) return fail(HE_EINVAL, "null argument");
  if (n_peers < 1 || n_peers > (uint32_t)kMaxPeers) return fail(HE_EINVAL, "n_peers must be in [1, %d]", kMaxPeers);
  if (dst_row0 % p->ctx->R.k) return fail(HE_EINVAL, "dst_row0 (%u) must be a multiple of k", dst_row0);
  if (p->algo == 1 && p->L != 1024)
    return fail(HE_EINVAL, "fused peer output needs the L = 1024 spectral path or the direct path");
  OutPeers pe{};
  pe.n = (int)n_peers;
  pe.dst_row0 = dst_row0;
  for (uint32_t i = 0; i < n_peers; ++i) {
    if (!out_b_peers[i] || !out_a_peers[i]) return fail(HE_EINVAL, "null peer pointer %u", i);
    pe.a[i] = out_a_peers[i];
    pe.b[i] = out_b_peers[i];
  }
  return gemm_rows_impl(p, ws, row0, rows, nullptr, nullptr, pe, stream);
}

extern "C" he_status he_pcmm_gemm(const he_pcmm_plan* p, const void* ws, uint32_t* out_b, uint32_t* out_a,
                                  void* stream) {
  if (!p) return fail(HE_EINVAL, "null plan");
  return he_pcmm_gemm_rows(p, ws, 0, p->n_out, out_b, out_a, stream);
}

extern "C" he_status he_pcmm_run(const he_pcmm_plan* p, const uint32_t* ct_in, uint32_t level, uint32_t* out_b,
                                 uint32_t* out_a, void* ws, uint64_t ws_size, void* stream, he_ledger* ledger) {
  if (!p) return fail(HE_EINVAL, "null plan");
  if (level < 1) return fail(HE_ENEEDS_BOOTSTRAP, "pcmm needs one level");
  if (level != 1) return fail(HE_EINVAL, "the MLWE PCMM runs at level 1 (got %u); switch levels first", level);
  he_status s = he_pcmm_decompose(p, ct_in, ws, ws_size, stream);
  if (s) return s;
  s = he_pcmm_gemm(p, ws, out_b, out_a, stream);
  if (s) return s;
  if (ledger) {
    const int64_t bo = p->n_out / p->ctx->R.k, bi = p->n_in / p->ctx->R.k;
    ledger->pc_mults += bo * bi;
    ledger->rescales += bo;
  }
  return HE_OK;
}

// level-1 words of both limbs (no rescale): the ring-packing input (he_ring_pack_run)
extern "C" he_status he_pcmm_run_level1(const he_pcmm_plan* p, const uint32_t* ct_in, uint32_t level, uint32_t* raw_b,
                                        uint32_t* raw_a, void* ws, uint64_t ws_size, void* stream) {
  if (!p) return fail(HE_EINVAL, "null plan");
  if (level < 1) return fail(HE_ENEEDS_BOOTSTRAP, "pcmm needs one level");
  if (level != 1) return fail(HE_EINVAL, "the MLWE PCMM runs at level 1 (got %u); switch levels first", level);
  if (!raw_b || !raw_a) return fail(HE_EINVAL, "null argument");
  he_status s = he_pcmm_decompose(p, ct_in, ws, ws_size, stream);
  if (s) return s;
  const uint64_t N = p->ctx->R.N;
  OutPeers none{};
  none.n = 0;
  return gemm_rows_impl(p, ws, 0, p->n_out, raw_b, raw_a, none, stream, raw_b + (uint64_t)(p->n_out / p->ctx->R.k) * N,
                        raw_a + (uint64_t)p->n_out * N);
}

// ---------------------------------------------------------------- K7 spectral a-part
// transform length: 4k (blocks of 3k outputs: 25% less spectral work than 2k) where the fast inverse
// exists (k = 256), else 2k; HE_SPEC_L = 512 / 1024 overrides for measurements
static uint32_t spec_len(const he_context* c) {
  static const int env = getenv("HE_SPEC_L") ? atoi(getenv("HE_SPEC_L")) : 0;
  if (c->R.k == 256 && env != 512) return 1024;
  return 2 * c->R.k;
}
static void spec_dims(const he_pcmm_plan* p, uint32_t& L, uint32_t& r_pad, uint32_t dsp[2], uint32_t* kg = nullptr) {
  L = spec_len(p->ctx);
  r_pad = ((p->n_in / p->ctx->R.k) + 63) / 64 * 64;
  // G^ rows are stored at 16-byte granularity (S3 stages them as no-swizzle core matrices; the MMA's reads past
  // kg meet A^'s zero padding), A^ rows stay padded to the 64-byte swizzle atom
  // (R > 64: whole 64-byte K blocks, so every S3 TMA box is full)
  const uint32_t R = p->n_in / p->ctx->R.k;
  if (kg) *kg = (getenv("HE_SPEC_G64") || R > 64) ? r_pad : (R + 15) / 16 * 16;
  dsp[0] = (uint32_t)digits_for(p->ctx->R.q[0]);
  dsp[1] = (uint32_t)digits_for(p->ctx->R.q[1]);
}

extern "C" he_status he_pcmm_spectral_weight_bytes(const he_pcmm_plan* p, uint64_t* bytes) {
  if (!p || !bytes) return fail(HE_EINVAL, "null argument");
  uint32_t L, r_pad, dsp[2], kg;
  spec_dims(p, L, r_pad, dsp, &kg);
  *bytes = (uint64_t)L * (dsp[0] + dsp[1]) * ((p->n_out + 127) / 128 * 128) * kg;
  return HE_OK;
}

extern "C" he_status he_pcmm_spectral_prepare(he_pcmm_plan* p, int8_t* wspec, void* stream) {
  if (!p || !wspec) return fail(HE_EINVAL, "null argument");
  const he_context* c = p->ctx;
  if (c->R.d % 32) return fail(HE_EINVAL, "spectral path needs mlwe_degree %% 32 == 0");
  uint32_t L, r_pad, dsp[2], kg;
  spec_dims(p, L, r_pad, dsp, &kg);
  // exactness of S3 (|digit product| <= 2^14, K = R = n_in / k terms):
  //   int32 shift accumulators      R * D * 2^14 < 2^31
  //   int32 paired shifts           |t_j| = |acc_2j + 256 acc_2j+1| <= R 2^14 (pairs(2j) + 256 pairs(2j+1)) < 2^31
  //   Montgomery input              off + |sum_j t_j pw_j| < 2 B, B = q sum_j max|t_j| < q 2^32
  const uint64_t R = p->n_in / c->R.k;
  for (int i = 0; i < 2; ++i) {
    const int D = (int)dsp[i], S = 2 * D - 1;
    auto pairs = [&](int sft) { return sft < 0 || sft >= S ? 0 : (sft < D ? sft + 1 : S - sft); };
    uint64_t tsum = 0, tmax = 0;
    for (int j = 0; j < D; ++j) {
      const uint64_t tj = R * 16384ull * (uint64_t)(pairs(2 * j) + 256 * pairs(2 * j + 1));
      tsum += tj;
      tmax = tj > tmax ? tj : tmax;
    }
    const unsigned __int128 B = (unsigned __int128)tsum * c->R.q[i];
    if (R * D * 16384ull >= (1ull << 31) || tmax >= (1ull << 31) || B >= ((unsigned __int128)c->R.q[i] << 32))
      return fail(HE_EINVAL, "n_in (%u) too large for the spectral recombination; use algo=direct", p->n_in);
    p->spec_off[i] = (uint64_t)(B / c->R.q[i] + 1) * c->R.q[i];
  }
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < 2; ++i) {
    spec_table_free(p->st[i]);
    HE_CUDA(spec_table_init(p->st[i], L, c->R.q[i]), "spectral table");
  }
  const uint64_t rows128 = (p->n_out + 127) / 128 * 128;   // G^ is stored in 128-row tiles (gidx)
  const uint64_t sz0 = (uint64_t)L * dsp[0] * rows128 * kg;
  const uint64_t total = sz0 + (uint64_t)L * dsp[1] * rows128 * kg;
  HE_CUDA(cudaMemsetAsync(wspec, 0, total, st), "memset");
  for (int i = 0; i < 2; ++i)
    HE_CUDA(launch_spec_weights(p->digits, p->d_w, p->n_out, p->n_in, c->R.k, p->st[i], (int)dsp[i], kg,
                                wspec + (i ? sz0 : 0), st),
            "spectral weights");
  for (int i = 0; i < 2; ++i) {
    he_status s = make_map_g16(&p->tmSA[i], wspec + (i ? sz0 : 0), kg, p->n_out, (uint64_t)L * dsp[i]);
    if (s) return s;
  }
  p->L = L;
  p->ob = L - c->R.k;
  p->nblk = (c->R.N + p->ob - 1) / p->ob;
  p->nbp = (p->nblk + 31) / 32 * 32;
  p->r_pad = r_pad;
  p->kg = kg;
  p->dsp[0] = dsp[0];
  p->dsp[1] = dsp[1];
  p->spec_w = wspec;
  p->algo = 1;
  return HE_OK;
}

extern "C" he_status he_pcmm_spectral_info(const he_pcmm_plan* p, uint32_t* info) {
  if (!p || !info) return fail(HE_EINVAL, "null argument");
  if (p->algo != 1) return fail(HE_EINVAL, "plan is not spectral");
  info[0] = p->L;
  info[1] = p->ob;
  info[2] = p->nblk;
  info[3] = p->nbp;
  return HE_OK;
}

extern "C" he_status he_pcmm_algo(const he_pcmm_plan* p, int* algo) {
  if (!p || !algo) return fail(HE_EINVAL, "null argument");
  *algo = p->algo;
  return HE_OK;
}

// ---------------------------------------------------------------- per-stage device times (profiling)
extern "C" he_status he_pcmm_profile(const he_pcmm_plan* p, int enable) {
  if (!p) return fail(HE_EINVAL, "null plan");
  p->prof_clear();
  p->prof_on = enable != 0;
  return HE_OK;
}

extern "C" he_status he_pcmm_profile_read(const he_pcmm_plan* p, double* ms, uint32_t* launches, uint32_t n) {
  if (!p || !ms || !launches) return fail(HE_EINVAL, "null argument");
  for (uint32_t i = 0; i < n; ++i) {
    ms[i] = 0;
    launches[i] = 0;
  }
  for (int st = 0; st < he_pcmm_plan::kStages && st < (int)n; ++st) {
    for (auto& pr : p->prof_ev[st]) {
      if (!pr.first || !pr.second) continue;
      HE_CUDA(cudaEventSynchronize(pr.second), "profile sync");
      float t = 0;
      HE_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second), "profile elapsed");
      ms[st] += t;
      launches[st] += 1;
    }
  }
  p->prof_clear();
  return HE_OK;
}
