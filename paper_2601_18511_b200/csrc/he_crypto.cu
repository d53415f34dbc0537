// he_crypto.cu -- K3 (RLWE -> MLWE digit decomposition), weight encoding, and the
// key/encrypt/decrypt plumbing used to make and check ciphertexts on the device.
#include "he_common.cuh"
#include "he_kernels.h"

namespace he {

// ================================================================ K3: decomposition
// For RLWE ct r and limb i, the per-limb GEMM operand has rows x = r*k + t (MLWE component t)
// and columns n:
//   n <  d          : b_r[t + k n]
//   n = d + d j + m : a~_{t,j}[m] = a_r[t - j + k m], negacyclic (a_r[c < 0] = -a_r[c + N])
// stored K-major as balanced signed 8-bit digit planes: plane p holds digit e of limb i
// (p = e for limb 0, D0 + e for limb 1) as planes[p][n][x].  One CTA per (r, m): it stages
// the 2k-word window of a_r around k*m in shared memory and writes the k+1 rows
// {n = m} U {n = d + d j + m : j < k}, 4 components per thread, one 32-bit store per digit.
__global__ void __launch_bounds__(256) decompose_kernel(const uint32_t* __restrict__ ct, uint32_t n_in, uint32_t d,
                                                        uint32_t k, uint32_t N, uint32_t q0, uint32_t q1, int d0,
                                                        int d1, int8_t* __restrict__ planes, uint64_t plane_stride,
                                                        uint32_t n_rho) {
  extern __shared__ uint32_t win[];  // [2 limbs][2k] a-window, then [2 limbs][k] b-row
  const uint32_t r = blockIdx.x, m = blockIdx.y;
  const uint32_t qs[2] = {q0, q1};
  uint32_t* bw = win + 4 * k;
  for (uint32_t i = threadIdx.x; i < 2 * k; i += blockDim.x) {
    const int64_t c = (int64_t)k * m - (int64_t)k + i;
#pragma unroll
    for (int L = 0; L < 2; ++L) {
      const uint32_t* a = ct + ((size_t)r * 2 + L) * 2 * N;
      uint32_t v;
      if (c >= 0) {
        v = a[c];
      } else {
        uint32_t w = a[c + N];
        v = w ? qs[L] - w : 0u;
      }
      win[L * 2 * k + i] = v;
    }
  }
  for (uint32_t t = threadIdx.x; t < k; t += blockDim.x) {
#pragma unroll
    for (int L = 0; L < 2; ++L) bw[L * k + t] = ct[((size_t)r * 2 + L) * 2 * N + N + t + (size_t)k * m];
  }
  __syncthreads();

  const uint32_t tpr = k / 4;                 // threads per output row
  const uint32_t rows_per_pass = blockDim.x / tpr;
  const uint32_t sub = threadIdx.x % tpr, rsel = threadIdx.x / tpr;
  const uint32_t t0 = sub * 4;
  for (uint32_t rho = rsel; rho < n_rho; rho += rows_per_pass) {
    // rho = 0: b-row n = m; rho = 1 + j: a-row n = d + d j + m
    const uint32_t n = rho == 0 ? m : d + d * (rho - 1) + m;
#pragma unroll
    for (int L = 0; L < 2; ++L) {
      const uint32_t q = qs[L];
      // balanced base-256 digits of the centred residue c: the bytes of (c + 0x80808080) ^ 0x80808080
      // (adding 128 at every byte position turns balanced digits into plain bytes)
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t t = t0 + e;
        const uint32_t v = rho == 0 ? bw[L * k + t] : win[L * 2 * k + (t + k - (rho - 1))];
        const uint32_t c = v > (q >> 1) ? v - q : v;          // two's complement of the centred value
        w[e] = (c + 0x80808080u) ^ 0x80808080u;
      }
      // 4x4 byte transpose: packed[p] byte e = digit p of value e
      const uint32_t lo01 = __byte_perm(w[0], w[1], 0x5140), hi01 = __byte_perm(w[0], w[1], 0x7362);
      const uint32_t lo23 = __byte_perm(w[2], w[3], 0x5140), hi23 = __byte_perm(w[2], w[3], 0x7362);
      uint32_t packed[4];
      packed[0] = __byte_perm(lo01, lo23, 0x5410);
      packed[1] = __byte_perm(lo01, lo23, 0x7632);
      packed[2] = __byte_perm(hi01, hi23, 0x5410);
      packed[3] = __byte_perm(hi01, hi23, 0x7632);
      const int nd = L == 0 ? d0 : d1;
      const int pbase = L == 0 ? 0 : d0;
      for (int p = 0; p < nd; ++p) {
        int8_t* dst = planes + (size_t)(pbase + p) * plane_stride + (size_t)n * n_in + (size_t)r * k + t0;
        *reinterpret_cast<uint32_t*>(dst) = packed[p];
      }
    }
  }
}

cudaError_t launch_decompose(const RingDims& R, const uint32_t* ct, uint32_t n_in, int d0, int d1, int8_t* planes,
                             uint64_t plane_stride, cudaStream_t s, int b_only) {
  dim3 grid(n_in / R.k, R.d);
  size_t smem = (size_t)6 * R.k * sizeof(uint32_t);
  decompose_kernel<<<grid, 256, smem, s>>>(ct, n_in, R.d, R.k, R.N, R.q[0], R.q[1], d0, d1, planes, plane_stride,
                                          b_only ? 1u : R.k + 1);
  return cudaGetLastError();
}

// ================================================================ K3 (fused-path form): compact digit planes
// For K1's on-the-fly producer (he_modgemm.cu, fused): instead of materialising every GEMM column,
// write per RLWE ct r and digit plane p
//   b planes  [p][r][N]            digit_p(b_r[i])
//   a copies  [p][s][r][S]         digit_p(X[i + s]),  X[i'] = a_r[i' - k] read negacyclically,
//                                  s = 0..15 (16-byte shifted copies: every ã window a_r[t - j + k m]
//                                  then starts 16-byte aligned in copy s = -j mod 16)
// ~340 MB at 4096x11008 instead of the 5 GB materialised operand.
HE_D void digits16(const uint32_t* v, uint32_t q, uint4* out /* [4 planes] */) {
  uint32_t w[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const uint32_t c = v[e] > (q >> 1) ? v[e] - q : v[e];
    w[e] = (c + 0x80808080u) ^ 0x80808080u;
  }
  uint32_t pk[4][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const uint32_t lo01 = __byte_perm(w[4 * g], w[4 * g + 1], 0x5140), hi01 = __byte_perm(w[4 * g], w[4 * g + 1], 0x7362);
    const uint32_t lo23 = __byte_perm(w[4 * g + 2], w[4 * g + 3], 0x5140),
                   hi23 = __byte_perm(w[4 * g + 2], w[4 * g + 3], 0x7362);
    pk[0][g] = __byte_perm(lo01, lo23, 0x5410);
    pk[1][g] = __byte_perm(lo01, lo23, 0x7632);
    pk[2][g] = __byte_perm(hi01, hi23, 0x5410);
    pk[3][g] = __byte_perm(hi01, hi23, 0x7632);
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) out[p] = make_uint4(pk[p][0], pk[p][1], pk[p][2], pk[p][3]);
}

__global__ void __launch_bounds__(256) digitize_kernel(const uint32_t* __restrict__ ct, uint32_t n_ct, uint32_t k,
                                                       uint32_t N, uint32_t q0, uint32_t q1, int d0, int d1, uint32_t S,
                                                       int8_t* __restrict__ out_a, int8_t* __restrict__ out_b) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;  // 16-byte group
  const uint32_t r = blockIdx.y, z = blockIdx.z;              // z < 16: shift copy; z == 16: b planes
  const uint32_t i0 = 16 * g;
  if (z == 16 ? i0 >= N : i0 >= S) return;
  const uint32_t qs[2] = {q0, q1};
#pragma unroll
  for (int L = 0; L < 2; ++L) {
    const uint32_t q = qs[L];
    const uint32_t* a = ct + ((size_t)r * 2 + L) * 2 * N;
    uint32_t v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      if (z == 16) {
        v[e] = a[N + i0 + e];
      } else {
        const int64_t xi = (int64_t)i0 + e + z - (int64_t)k;  // index into a_r, negacyclic below 0
        uint32_t val = 0;
        if (xi >= 0 && xi < (int64_t)N) val = a[xi];
        else if (xi < 0) {
          const uint32_t w = a[xi + N];
          val = w ? q - w : 0u;
        }
        v[e] = val;
      }
    }
    uint4 dg[4];
    digits16(v, q, dg);
    const int nd = L == 0 ? d0 : d1, pbase = L == 0 ? 0 : d0;
    for (int p = 0; p < nd; ++p) {
      const uint32_t P = pbase + p;
      int8_t* dst = z == 16 ? out_b + ((size_t)P * n_ct + r) * N + i0
                            : out_a + (((size_t)P * 16 + z) * n_ct + r) * S + i0;
      *reinterpret_cast<uint4*>(dst) = dg[p];
    }
  }
}

cudaError_t launch_digitize(const RingDims& R, const uint32_t* ct, uint32_t n_ct, int d0, int d1, uint32_t S,
                            int8_t* out_a, int8_t* out_b, cudaStream_t s) {
  dim3 grid((S / 16 + 255) / 256, n_ct, 17);
  digitize_kernel<<<grid, 256, 0, s>>>(ct, n_ct, R.k, R.N, R.q[0], R.q[1], d0, d1, S, out_a, out_b);
  return cudaGetLastError();
}

// ================================================================ weight encoding
// W~[y][x] = round_half_even(q1 * W[k(y/k) + sigma(y%k)][k(x/k) + sigma(x%k)])
// (block conjugation by sigma = g o nibble swap, PAPER.md:672 / bitrev.py:57-70).
__device__ __forceinline__ long long encoded_weight(const double* W, uint32_t n_in, uint32_t k, int logk, double dw,
                                                    uint32_t y, uint32_t x) {
  const uint32_t sr = (y / k) * k + sigma_h(y % k, logk);
  const uint32_t sc = (x / k) * k + sigma_h(x % k, logk);
  return __double2ll_rn(__dmul_rn(dw, W[(size_t)sr * n_in + sc]));
}

__global__ void weight_maxabs_kernel(const double* __restrict__ W, uint32_t n_out, uint32_t n_in, uint32_t k, int logk,
                                     double dw, unsigned long long* maxabs) {
  unsigned long long m = 0;
  const size_t total = (size_t)n_out * n_in;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    long long v = encoded_weight(W, n_in, k, logk, dw, (uint32_t)(i / n_in), (uint32_t)(i % n_in));
    unsigned long long a = (unsigned long long)(v < 0 ? -v : v);
    m = a > m ? a : m;
  }
  for (int o = 16; o; o >>= 1) {
    unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(maxabs, m);
}

__global__ void encode_weights_kernel(const double* __restrict__ W, uint32_t n_out, uint32_t n_in, uint32_t k,
                                      int logk, double dw, uint32_t ndig, int8_t* __restrict__ planes) {
  const size_t total = (size_t)n_out * n_in;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    long long v = encoded_weight(W, n_in, k, logk, dw, (uint32_t)(i / n_in), (uint32_t)(i % n_in));
    int8_t dg[4];
    balanced_digits4((int32_t)v, dg, 4);
    for (uint32_t p = 0; p < ndig; ++p) planes[(size_t)p * total + i] = dg[p];
  }
}

cudaError_t launch_weight_maxabs(const RingDims& R, const double* W, uint32_t n_out, uint32_t n_in,
                                 unsigned long long* maxabs, cudaStream_t s) {
  weight_maxabs_kernel<<<1184, 256, 0, s>>>(W, n_out, n_in, R.k, (int)R.logk, (double)R.q[1], maxabs);
  return cudaGetLastError();
}

cudaError_t launch_encode_weights(const RingDims& R, const double* W, uint32_t n_out, uint32_t n_in, uint32_t dw,
                                  int8_t* planes, cudaStream_t s) {
  encode_weights_kernel<<<1184, 256, 0, s>>>(W, n_out, n_in, R.k, (int)R.logk, (double)R.q[1], dw, planes);
  return cudaGetLastError();
}

// ================================================================ keys / encryption / decryption
__global__ void keygen_kernel(RngCtx rc, uint64_t seed, uint32_t N, int32_t* s) {
  const Rng key = rng_make(rc, seed, kStreamSecret);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
    s[i] = ternary(rng_next(key, i));
}
cudaError_t launch_keygen(const RingDims& R, uint64_t seed, int32_t* s_dev, cudaStream_t st) {
  keygen_kernel<<<(R.N + 255) / 256, 256, 0, st>>>(R.rng, seed, R.N, s_dev);
  return cudaGetLastError();
}

__global__ void reduce_secret_kernel(const int32_t* s, uint32_t N, uint32_t q, uint32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    int32_t v = s[i];
    out[i] = v < 0 ? q + v : (uint32_t)v;
  }
}
cudaError_t launch_reduce_secret(const RingDims& R, const int32_t* s_dev, uint32_t limb, uint32_t* out,
                                 cudaStream_t st) {
  reduce_secret_kernel<<<(R.N + 255) / 256, 256, 0, st>>>(s_dev, R.N, R.q[limb], out);
  return cudaGetLastError();
}

// a-part of every (ct, limb) and a copy in the b slot (NTT'd in place to form a*s)
__global__ void gen_a_kernel(RngCtx rc, uint64_t seed, uint32_t r0, uint32_t N, uint32_t q0, uint32_t q1,
                             uint32_t* ct) {
  const uint32_t r = blockIdx.y, L = blockIdx.z;
  const uint32_t q = L ? q1 : q0;
  const Rng key = rng_make(rc, seed, stream_a(r0 + r, L));
  uint32_t* a = ct + ((size_t)r * 2 + L) * 2 * N;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    uint32_t v = (uint32_t)(rng_next(key, i) % q);
    a[i] = v;
    a[N + i] = v;
  }
}
cudaError_t launch_gen_a(const RingDims& R, uint64_t seed, uint32_t r0, uint32_t n_ct, uint32_t* ct, cudaStream_t st) {
  dim3 g((R.N + 1023) / 1024, n_ct, 2);
  gen_a_kernel<<<g, 256, 0, st>>>(R.rng, seed, r0, R.N, R.q[0], R.q[1], ct);
  return cudaGetLastError();
}

__global__ void pointwise_kernel(const uint32_t* x, uint64_t xs, const uint32_t* y, uint32_t n, uint32_t q,
                                 uint32_t* out, uint64_t os) {
  const uint32_t p = blockIdx.y;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[p * os + i] = mul_mod(x[p * xs + i], y[i], q);
}
cudaError_t launch_pointwise_mul(const uint32_t* x, uint64_t x_stride, const uint32_t* y, uint32_t n,
                                 uint32_t count, uint32_t q, uint32_t* out, uint64_t out_stride, cudaStream_t st) {
  dim3 g((n + 1023) / 1024, count);
  pointwise_kernel<<<g, 256, 0, st>>>(x, x_stride, y, n, q, out, out_stride);
  return cudaGetLastError();
}

// b = -(a s) + Ecd_coeff(acts) + e; the b slot holds a*s on entry.
// layout 0: App. A activation block (tokens x n_in); layout 1: Rhombus vector of n_in values with
// window w (split point, oracle or_encode_vector_w): element e at coefficient (e / w) + rho h_w(e mod w),
// rho = N / n_rh (w = n_rh: the plain h layout of PAPER.md:674-680)
__global__ void finish_encrypt_kernel(const double* __restrict__ acts, uint32_t n_in, uint32_t d, uint32_t k,
                                      int logk, uint32_t N, double delta, uint64_t seed, uint32_t r0, uint32_t q0,
                                      uint32_t q1, uint32_t* ct, int layout, uint32_t n_rh, uint32_t win, RngCtx rc) {
  const uint32_t r = blockIdx.y;
  const Rng ekey = rng_make(rc, seed, stream_e(r0 + r));
  const uint32_t half = d / 2;
  const int lh = ilog2_h(half);
  const int lw = ilog2_h(win);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    long long pt = 0;
    if (layout == 0) {
      const uint32_t t = c % k, m = c / k;
      if (m < half) {
        const double v = acts[(size_t)bitrev_h(m, lh) * n_in + (size_t)k * r + sigma_h(t, logk)];
        pt = __double2ll_rn(__dmul_rn(delta, v));
      }
    } else if (layout == 2) {  // raw integer plaintext polynomials int64 [n_ct][N] (slot encodings)
      pt = reinterpret_cast<const long long*>(acts)[(size_t)r * N + c];
    } else {
      const uint32_t rho = N / n_rh, p = c % rho, kk = c / rho;
      if (kk < win) {
        const uint32_t hk = win < 2 ? 0u : (kk & (win >> 1)) | bitrev_h(kk & ((win >> 1) - 1), lw - 1);
        const uint32_t e = win * p + hk;
        if (e < n_in) pt = __double2ll_rn(__dmul_rn(delta, acts[e]));
      }
    }
    const long long e = cbd21_d(rng_next(ekey, c));
#pragma unroll
    for (int L = 0; L < 2; ++L) {
      const uint32_t q = L ? q1 : q0;
      uint32_t* b = ct + ((size_t)r * 2 + L) * 2 * N + N;
      const uint32_t as = b[c];
      uint64_t v = (uint64_t)from_i64(pt, q) + from_i64(e, q) + (q - as);
      b[c] = (uint32_t)(v % q);
    }
  }
}
cudaError_t launch_finish_encrypt(const RingDims& R, const double* acts, uint32_t n_in, uint64_t seed, uint32_t r0,
                                  uint32_t n_ct, uint32_t* ct, cudaStream_t st, int layout, uint32_t win) {
  dim3 g((R.N + 1023) / 1024, n_ct);
  finish_encrypt_kernel<<<g, 256, 0, st>>>(acts, n_in, R.d, R.k, (int)R.logk, R.N, (double)(1ull << R.log_delta),
                                           seed, r0, R.q[0], R.q[1], ct, layout, R.n_rh, win ? win : R.n_rh, R.rng);
  return cudaGetLastError();
}

__global__ void phase_kernel(const uint32_t* b, uint64_t bs, const uint32_t* as, uint64_t ass, uint32_t n, uint32_t q,
                             int64_t* phase) {
  const uint32_t p = blockIdx.y;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t v = add_mod(b[p * bs + i], as[p * ass + i], q);
    phase[(size_t)p * n + i] = v > q / 2 ? (int64_t)v - q : (int64_t)v;
  }
}
cudaError_t launch_phase(const uint32_t* b, uint64_t b_stride, const uint32_t* as, uint64_t as_stride, uint32_t n,
                         uint32_t count, uint32_t q, int64_t* phase, cudaStream_t st) {
  dim3 g((n + 1023) / 1024, count);
  phase_kernel<<<g, 256, 0, st>>>(b, b_stride, as, as_stride, n, q, phase);
  return cudaGetLastError();
}

// MLWE decryption of PCMM output rows (level 0, q0):
//   phase_y[m] = b'_y[m] + sum_j sum_m' a'_y[j][m'] * s_j[m - m']  (negacyclic in Y^d = -1),
//   s_j[m] = s[j + k m].   One CTA per row, one thread per m, j streamed through smem.
__global__ void __launch_bounds__(256) decrypt_mlwe_kernel(const int32_t* __restrict__ s,
                                                           const uint32_t* __restrict__ out_b,
                                                           const uint32_t* __restrict__ out_a, uint32_t d, uint32_t k,
                                                           uint32_t N, uint32_t q0, uint32_t row0, int64_t* phase) {
  extern __shared__ uint32_t sh[];  // a_j [d], s_j [2d] (s_j[m - m'] with wrap sign folded)
  int32_t* sj = reinterpret_cast<int32_t*>(sh + d);
  const uint32_t y = row0 + blockIdx.x;
  const uint32_t* arow = out_a + (size_t)y * N;
  int64_t acc = 0;
  for (uint32_t j = 0; j < k; ++j) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
      sh[i] = arow[(size_t)j * d + i];
      const int32_t sv = s[j + (size_t)k * i];
      sj[d + i] = sv;   // index m - m' >= 0
      sj[i] = -sv;      // index m - m' + d (wrapped, negated)
    }
    __syncthreads();
    for (uint32_t m = threadIdx.x; m < d; m += blockDim.x) {
      int64_t part = 0;
      for (uint32_t mp = 0; mp < d; ++mp) part += (int64_t)sh[mp] * sj[d + m - mp];
      acc += part % (int64_t)q0;  // |part| < d * q0 < 2^40
    }
  }
  for (uint32_t m = threadIdx.x; m < d; m += blockDim.x) {
    const uint32_t b = out_b[(size_t)(y / k) * N + (y % k) + (size_t)k * m];
    int64_t v = (acc + b) % (int64_t)q0;
    if (v < 0) v += q0;
    phase[(size_t)blockIdx.x * d + m] = v > q0 / 2 ? v - q0 : v;
  }
}
cudaError_t launch_decrypt_mlwe(const RingDims& R, const int32_t* s, const uint32_t* out_b, const uint32_t* out_a,
                                uint32_t n_out, uint32_t row0, uint32_t n_rows, int64_t* phase, cudaStream_t st) {
  if (R.d > 256) return cudaErrorInvalidValue;  // one thread per m
  size_t smem = 3 * (size_t)R.d * sizeof(uint32_t);
  decrypt_mlwe_kernel<<<n_rows, R.d, smem, st>>>(s, out_b, out_a, R.d, R.k, R.N, R.q[0], row0, phase);
  return cudaGetLastError();
}

// Fast MLWE decryption through the RLWE view: row y's phase is component 0 of A_y s (degree N) plus b',
// with A_y[k m - j] = a'_y[j][m] (negacyclic) -- one NTT product per row instead of k length-d convolutions.
// A [rows][N] (q0 residues) from the a' rows [row0, row0 + rows): one CTA per (32 positions m, row)
__global__ void __launch_bounds__(256) mlwe_rows_to_poly_kernel(const uint32_t* __restrict__ out_a, uint32_t row0,
                                                                uint32_t d, uint32_t k, uint32_t N, uint32_t q0,
                                                                uint32_t* __restrict__ A) {
  __shared__ uint32_t tile[256 * 33];   // [j][m], k <= 256
  const uint32_t m0 = blockIdx.x * 32, r = blockIdx.y;
  const uint32_t* src = out_a + (size_t)(row0 + r) * N + m0;
  for (uint32_t i = threadIdx.x; i < 32 * k; i += blockDim.x) tile[(i >> 5) * 33 + (i & 31)] = src[(size_t)d * (i >> 5) + (i & 31)];
  __syncthreads();
  uint32_t* dst = A + (size_t)r * N;
  for (uint32_t i = threadIdx.x; i < 32 * k; i += blockDim.x) {
    const uint32_t mm = i / k, j = k - 1 - (i % k);
    uint32_t v = tile[j * 33 + mm];
    int64_t c = (int64_t)k * (m0 + mm) - j;
    if (c < 0) {
      c += N;
      v = v ? q0 - v : 0;
    }
    dst[c] = v;
  }
}
// phase [rows][d] = centred (prod[r][k m] + b'_y[m]) mod q0   (prod = A_y s, coefficient form)
__global__ void mlwe_phase_kernel(const uint32_t* __restrict__ prod, const uint32_t* __restrict__ out_b, uint32_t row0,
                                  uint32_t rows, uint32_t d, uint32_t k, uint32_t N, uint32_t q0,
                                  int64_t* __restrict__ phase) {
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < rows * d; x += gridDim.x * blockDim.x) {
    const uint32_t r = x / d, m = x % d, y = row0 + r;
    const uint32_t b = out_b[(size_t)(y / k) * N + (y % k) + (size_t)k * m];
    const uint32_t v = add_mod(prod[(size_t)r * N + (size_t)k * m], b, q0);
    phase[x] = v > q0 / 2 ? (int64_t)v - q0 : (int64_t)v;
  }
}
cudaError_t launch_mlwe_rows_to_poly(const RingDims& R, const uint32_t* out_a, uint32_t row0, uint32_t rows, uint32_t* A,
                                     cudaStream_t st) {
  if (R.k > 256 || R.d % 32) return cudaErrorInvalidValue;
  mlwe_rows_to_poly_kernel<<<dim3(R.d / 32, rows), 256, 0, st>>>(out_a, row0, R.d, R.k, R.N, R.q[0], A);
  return cudaGetLastError();
}
cudaError_t launch_mlwe_phase(const RingDims& R, const uint32_t* prod, const uint32_t* out_b, uint32_t row0,
                              uint32_t rows, int64_t* phase, cudaStream_t st) {
  const uint32_t total = rows * R.d;
  mlwe_phase_kernel<<<(total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32, 256, 0, st>>>(
      prod, out_b, row0, rows, R.d, R.k, R.N, R.q[0], phase);
  return cudaGetLastError();
}

// ModRaise (the Half-Bootstrap hand-off): level-0 ciphertexts mod q0 [n_ct][2][N] ->
// the centred lift of every coefficient into each target prime: out [n_ct][n_primes][2][N]
__global__ void mod_raise_kernel(const uint32_t* __restrict__ ct, uint64_t words, uint32_t q0,
                                 const uint32_t* __restrict__ primes, uint32_t n_primes, uint32_t N,
                                 uint32_t* __restrict__ out) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < words; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = x / (2ull * N), w = x % (2ull * N);
    const uint32_t v = ct[x];
    const int64_t c = v > q0 / 2 ? (int64_t)v - q0 : (int64_t)v;
    for (uint32_t i = 0; i < n_primes; ++i) {
      const int64_t p = primes[i];
      int64_t m = c % p;
      if (m < 0) m += p;
      out[(r * n_primes + i) * 2ull * N + w] = (uint32_t)m;
    }
  }
}
cudaError_t launch_mod_raise(const RingDims& R, const uint32_t* ct, uint32_t n_ct, const uint32_t* primes_dev,
                             uint32_t n_primes, uint32_t* out, cudaStream_t st) {
  const uint64_t words = (uint64_t)n_ct * 2 * R.N;
  const uint64_t blocks = (words + 255) / 256;
  mod_raise_kernel<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(ct, words, R.q[0], primes_dev,
                                                                                      n_primes, R.N, out);
  return cudaGetLastError();
}

}  // namespace he
