// he_ntt.cu -- K2: negacyclic NTT / INTT over Z_q[X]/(X^n + 1), n <= 65536, q < 2^31.
//
// Merged-twiddle Cooley-Tukey (natural -> bit-reversed) forward and Gentleman-Sande
// (bit-reversed -> natural, scaled by n^-1) inverse, the same transform the oracle
// restates (oracle/he_oracle.c ntt_fwd/ntt_inv).  n = n1 * n2 with n2 = min(n, 4096):
//   pass "cols": the log2(n1) outer stages act on n2 independent strided columns
//                (element c + n2*v, v < n1), staged through shared memory 64 columns at a time;
//   pass "rows": the log2(n2) inner stages act on n1 contiguous 4096-word blocks, one CTA per
//                block, all stages in shared memory.
// For n <= 4096 only the rows pass runs.  A batch is processed pass-by-pass, so when it
// fits in L2 the intermediate never reaches HBM.  Twiddles use Shoup precomputation.
#include "he_common.cuh"
#include "he_kernels.h"

namespace he {

constexpr int kNttRowsMax = 4096;
constexpr int kColW = 64;

// ---------------------------------------------------------------- host tables
cudaError_t ntt_table_init(NttTable& t, uint32_t n, uint32_t q) {
  t.n = n;
  t.q = q;
  if ((q - 1) % (2ull * n)) return cudaErrorInvalidValue;
  uint64_t psi = 0;
  for (uint64_t g = 2; g < q; ++g) {
    uint64_t c = powmod_h(g, (q - 1) / (2ull * n), q);
    if (powmod_h(c, n, q) == q - 1) {
      psi = c;
      break;
    }
  }
  if (!psi) return cudaErrorInvalidValue;
  const uint64_t psii = powmod_h(psi, q - 2, q);
  const int l = ilog2_h(n);
  uint32_t* h = new uint32_t[4 * (size_t)n];
  uint64_t* pw = new uint64_t[n];
  uint64_t* pwi = new uint64_t[n];
  uint64_t p = 1, pi = 1;
  for (uint32_t i = 0; i < n; ++i) {
    pw[i] = p;
    pwi[i] = pi;
    p = (unsigned __int128)p * psi % q;
    pi = (unsigned __int128)pi * psii % q;
  }
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t f = (uint32_t)pw[bitrev_h(i, l)], v = (uint32_t)pwi[bitrev_h(i, l)];
    h[i] = f;
    h[n + i] = shoup_pre(f, q);
    h[2 * n + i] = v;
    h[3 * n + i] = shoup_pre(v, q);
  }
  delete[] pw;
  delete[] pwi;
  t.ninv = (uint32_t)powmod_h(n, q - 2, q);
  t.ninvp = shoup_pre(t.ninv, q);
  uint32_t* dptr = nullptr;
  cudaError_t e = cudaMalloc(&dptr, 4 * (size_t)n * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(dptr, h, 4 * (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice);
  delete[] h;
  if (e != cudaSuccess) return e;
  t.fw = dptr;
  t.fwp = dptr + n;
  t.iv = dptr + 2 * (size_t)n;
  t.ivp = dptr + 3 * (size_t)n;
  return cudaSuccess;
}

void ntt_table_free(NttTable& t) {
  if (t.fw) cudaFree(t.fw);
  t.fw = t.fwp = t.iv = t.ivp = nullptr;
}

// ---------------------------------------------------------------- kernels
// outer stages over strided columns; forward: m = 1 .. n1/2
__global__ void __launch_bounds__(256) ntt_cols_fwd(uint32_t* __restrict__ data, uint64_t stride, uint32_t n1,
                                                    uint32_t n2, const uint32_t* __restrict__ fw,
                                                    const uint32_t* __restrict__ fwp, uint32_t q) {
  __shared__ uint32_t s[16 * kColW];
  uint32_t* a = data + blockIdx.y * stride;
  const uint32_t c0 = blockIdx.x * kColW;
  for (uint32_t i = threadIdx.x; i < n1 * kColW; i += blockDim.x) {
    uint32_t v = i / kColW, cc = i % kColW;
    s[i] = a[c0 + cc + (size_t)n2 * v];
  }
  __syncthreads();
  for (uint32_t m = 1, t = n1 / 2; m < n1; m <<= 1, t >>= 1) {
    for (uint32_t bf = threadIdx.x; bf < (n1 / 2) * kColW; bf += blockDim.x) {
      uint32_t cc = bf % kColW, p = bf / kColW;
      uint32_t i = p / t, u = p % t, j = 2 * i * t + u;
      uint32_t U = s[j * kColW + cc];
      uint32_t V = shoup_mul(s[(j + t) * kColW + cc], fw[m + i], fwp[m + i], q);
      s[j * kColW + cc] = add_mod(U, V, q);
      s[(j + t) * kColW + cc] = sub_mod(U, V, q);
    }
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < n1 * kColW; i += blockDim.x) {
    uint32_t v = i / kColW, cc = i % kColW;
    a[c0 + cc + (size_t)n2 * v] = s[i];
  }
}

// inner stages over contiguous n2-blocks; forward: m = n1 * 2^s
__global__ void __launch_bounds__(512) ntt_rows_fwd(uint32_t* __restrict__ data, uint64_t stride, uint32_t n1,
                                                    uint32_t n2, const uint32_t* __restrict__ fw,
                                                    const uint32_t* __restrict__ fwp, uint32_t q) {
  __shared__ uint32_t s[kNttRowsMax];
  const uint32_t b = blockIdx.x;
  uint32_t* a = data + blockIdx.y * stride + (size_t)b * n2;
  for (uint32_t i = threadIdx.x; i < n2 / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(s)[i] = reinterpret_cast<const uint4*>(a)[i];
  __syncthreads();
  for (uint32_t m = n1, t = n2 / 2; t >= 1; m <<= 1, t >>= 1) {
    for (uint32_t p = threadIdx.x; p < n2 / 2; p += blockDim.x) {
      uint32_t il = p / t, u = p % t, j = 2 * il * t + u;
      uint32_t i = b * (n2 / (2 * t)) + il;
      uint32_t U = s[j];
      uint32_t V = shoup_mul(s[j + t], fw[m + i], fwp[m + i], q);
      s[j] = add_mod(U, V, q);
      s[j + t] = sub_mod(U, V, q);
    }
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < n2 / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(a)[i] = reinterpret_cast<const uint4*>(s)[i];
}

// inverse inner stages: t = 1 .. n2/2, h = n/(2t); optional final n^-1 scaling (when n1 == 1)
__global__ void __launch_bounds__(512) ntt_rows_inv(uint32_t* __restrict__ data, uint64_t stride, uint32_t n,
                                                    uint32_t n2, const uint32_t* __restrict__ iv,
                                                    const uint32_t* __restrict__ ivp, uint32_t q, uint32_t scale,
                                                    uint32_t scalep, int do_scale) {
  __shared__ uint32_t s[kNttRowsMax];
  const uint32_t b = blockIdx.x;
  uint32_t* a = data + blockIdx.y * stride + (size_t)b * n2;
  for (uint32_t i = threadIdx.x; i < n2 / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(s)[i] = reinterpret_cast<const uint4*>(a)[i];
  __syncthreads();
  for (uint32_t t = 1; t < n2; t <<= 1) {
    const uint32_t h = n / (2 * t);
    for (uint32_t p = threadIdx.x; p < n2 / 2; p += blockDim.x) {
      uint32_t il = p / t, u = p % t, j = 2 * il * t + u;
      uint32_t i = b * (n2 / (2 * t)) + il;
      uint32_t U = s[j], V = s[j + t];
      s[j] = add_mod(U, V, q);
      s[j + t] = shoup_mul(sub_mod(U, V, q), iv[h + i], ivp[h + i], q);
    }
    __syncthreads();
  }
  if (do_scale) {
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) s[i] = shoup_mul(s[i], scale, scalep, q);
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < n2 / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(a)[i] = reinterpret_cast<const uint4*>(s)[i];
}

// inverse outer stages over strided columns: t' = 1 .. n1/2, then n^-1 scaling
__global__ void __launch_bounds__(256) ntt_cols_inv(uint32_t* __restrict__ data, uint64_t stride, uint32_t n1,
                                                    uint32_t n2, const uint32_t* __restrict__ iv,
                                                    const uint32_t* __restrict__ ivp, uint32_t q, uint32_t scale,
                                                    uint32_t scalep) {
  __shared__ uint32_t s[16 * kColW];
  uint32_t* a = data + blockIdx.y * stride;
  const uint32_t c0 = blockIdx.x * kColW;
  for (uint32_t i = threadIdx.x; i < n1 * kColW; i += blockDim.x) {
    uint32_t v = i / kColW, cc = i % kColW;
    s[i] = a[c0 + cc + (size_t)n2 * v];
  }
  __syncthreads();
  for (uint32_t t = 1; t < n1; t <<= 1) {
    const uint32_t h = n1 / (2 * t);
    for (uint32_t bf = threadIdx.x; bf < (n1 / 2) * kColW; bf += blockDim.x) {
      uint32_t cc = bf % kColW, p = bf / kColW;
      uint32_t i = p / t, u = p % t, j = 2 * i * t + u;
      uint32_t U = s[j * kColW + cc], V = s[(j + t) * kColW + cc];
      s[j * kColW + cc] = add_mod(U, V, q);
      s[(j + t) * kColW + cc] = shoup_mul(sub_mod(U, V, q), iv[h + i], ivp[h + i], q);
    }
    __syncthreads();
  }
  for (uint32_t i = threadIdx.x; i < n1 * kColW; i += blockDim.x) {
    uint32_t v = i / kColW, cc = i % kColW;
    a[c0 + cc + (size_t)n2 * v] = shoup_mul(s[i], scale, scalep, q);
  }
}

static void split(uint32_t n, uint32_t& n1, uint32_t& n2) {
  n2 = n < (uint32_t)kNttRowsMax ? n : (uint32_t)kNttRowsMax;
  n1 = n / n2;
}

cudaError_t ntt_forward(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t st) {
  uint32_t n1, n2;
  split(t.n, n1, n2);
  if (n1 > 16 || count == 0) return count ? cudaErrorInvalidValue : cudaSuccess;
  if (n1 > 1) {
    dim3 g(n2 / kColW, count);
    ntt_cols_fwd<<<g, 256, 0, st>>>(data, stride, n1, n2, t.fw, t.fwp, t.q);
  }
  dim3 g2(n1, count);
  ntt_rows_fwd<<<g2, n2 >= 1024 ? 512 : n2 / 2, 0, st>>>(data, stride, n1, n2, t.fw, t.fwp, t.q);
  return cudaGetLastError();
}

cudaError_t ntt_inverse(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t st) {
  uint32_t n1, n2;
  split(t.n, n1, n2);
  if (n1 > 16 || count == 0) return count ? cudaErrorInvalidValue : cudaSuccess;
  dim3 g2(n1, count);
  ntt_rows_inv<<<g2, n2 >= 1024 ? 512 : n2 / 2, 0, st>>>(data, stride, t.n, n2, t.iv, t.ivp, t.q, t.ninv, t.ninvp,
                                                         n1 == 1);
  if (n1 > 1) {
    dim3 g(n2 / kColW, count);
    ntt_cols_inv<<<g, 256, 0, st>>>(data, stride, n1, n2, t.iv, t.ivp, t.q, t.ninv, t.ninvp);
  }
  return cudaGetLastError();
}

}  // namespace he
