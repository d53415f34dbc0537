// he_ntt.cu -- K2: negacyclic NTT / INTT over Z_q[X]/(X^n + 1), n in {64 * 8^i} x {1,2,4,8,16}, q < 2^30.
//
// The transform is the merged-twiddle Cooley-Tukey (natural -> bit-reversed) / Gentleman-Sande
// (bit-reversed -> natural, scaled by n^-1) pair the oracle restates (oracle/he_oracle.c
// ntt_fwd / ntt_inv), so outputs agree word for word.  n = n1 * n2:
//   "cols" pass: the log2(n1) outer stages act on n2 independent strided columns; one column per
//               thread, all n1 (<= 16) elements in registers, twiddles warp-uniform.
//   "rows" pass: the log2(n2) inner stages act on contiguous n2-word blocks (n2 = 8^R <= 4096), one
//               CTA per block, n2/8 threads x 8 register-resident elements; each radix-8 round does
//               3 stages in registers and one shared-memory exchange.
// Butterflies are Harvey-lazy (q < 2^30): values live in [0, 4q) between stages (7 integer ops per
// butterfly), Shoup twiddles come from an interleaved (W, W') table read as 8/16-byte vectors.
// Between the two passes of a batch the intermediate is L2-resident when the batch fits L2.
#include <type_traits>

#include "he_common.cuh"
#include "he_kernels.h"

namespace he {

// ---------------------------------------------------------------- host tables
cudaError_t ntt_table_init(NttTable& t, uint32_t n, uint32_t q) {
  t.n = n;
  t.q = q;
  if ((q - 1) % (2ull * n) || q >= (1u << 30)) return cudaErrorInvalidValue;
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
  uint32_t* h = new uint32_t[4 * (size_t)n];  // fw pairs [n][2], iv pairs [n][2]
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
    h[2 * i] = f;
    h[2 * i + 1] = shoup_pre(f, q);
    h[2 * (size_t)n + 2 * i] = v;
    h[2 * (size_t)n + 2 * i + 1] = shoup_pre(v, q);
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
  t.iv = dptr + 2 * (size_t)n;
  t.fwp = t.ivp = nullptr;
  return cudaSuccess;
}

void ntt_table_free(NttTable& t) {
  if (t.fw) cudaFree(t.fw);
  t.fw = t.fwp = t.iv = t.ivp = nullptr;
}

// ---------------------------------------------------------------- butterflies (q < 2^30)
// CT: X, Y in [0, 4q) -> X' = X + WY, Y' = X - WY, both in [0, 4q)
HE_D void ct_bf(uint32_t& x, uint32_t& y, uint2 w, uint32_t q2, uint32_t q) {
  const uint32_t a = min(x, x - q2);     // [0, 2q): x - 2q wraps above x when x < 2q
  const uint32_t t = y * w.x - __umulhi(y, w.y) * q;  // Shoup, [0, 2q)
  x = a + t;
  y = a + q2 - t;
}
// GS: X, Y in [0, 2q) -> X' = X + Y, Y' = (X - Y) W, both in [0, 2q)
HE_D void gs_bf(uint32_t& x, uint32_t& y, uint2 w, uint32_t q2, uint32_t q) {
  const uint32_t s = x + y;
  const uint32_t d = x + q2 - y;
  x = min(s, s - q2);
  y = d * w.x - __umulhi(d, w.y) * q;
}
HE_D uint32_t reduce4(uint32_t x, uint32_t q) {  // [0, 4q) -> [0, q)
  x = min(x, x - 2 * q);
  return min(x, x - q);
}
HE_D uint2 ldtw(const uint2* tw, uint32_t i) { return __ldg(tw + i); }

// ---------------------------------------------------------------- cols pass (outer stages)
template <int N1>
__global__ void __launch_bounds__(256) ntt_fwd_cols(uint32_t* __restrict__ data, uint64_t stride, uint32_t n2,
                                                    const uint2* __restrict__ tw, uint32_t q) {
  const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n2) return;
  uint32_t* a = data + blockIdx.y * stride + col;
  uint32_t x[N1];
#pragma unroll
  for (int v = 0; v < N1; ++v) x[v] = a[(size_t)n2 * v];
  const uint32_t q2 = 2 * q;
#pragma unroll
  for (int m = 1, t = N1 / 2; m < N1; m <<= 1, t >>= 1) {
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const uint2 w = ldtw(tw, m + i);
#pragma unroll
      for (int u = 0; u < t; ++u) ct_bf(x[2 * i * t + u], x[2 * i * t + u + t], w, q2, q);
    }
  }
#pragma unroll
  for (int v = 0; v < N1; ++v) a[(size_t)n2 * v] = x[v];
}

template <int N1>
__global__ void __launch_bounds__(256) ntt_inv_cols(uint32_t* __restrict__ data, uint64_t stride, uint32_t n2,
                                                    const uint2* __restrict__ tw, uint32_t q, uint32_t ninv,
                                                    uint32_t ninvp) {
  const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n2) return;
  uint32_t* a = data + blockIdx.y * stride + col;
  uint32_t x[N1];
#pragma unroll
  for (int v = 0; v < N1; ++v) x[v] = a[(size_t)n2 * v];
  const uint32_t q2 = 2 * q;
#pragma unroll
  for (int t = 1; t < N1; t <<= 1) {
    const int h = N1 / (2 * t);
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const uint2 w = ldtw(tw, h + i);
#pragma unroll
      for (int u = 0; u < t; ++u) gs_bf(x[2 * i * t + u], x[2 * i * t + u + t], w, q2, q);
    }
  }
#pragma unroll
  for (int v = 0; v < N1; ++v) a[(size_t)n2 * v] = shoup_mul(x[v], ninv, ninvp, q);
}

// ---------------------------------------------------------------- rows pass (inner stages)
// smem index padding: one word per 32 to break the power-of-two strides
HE_D uint32_t pad(uint32_t i) { return i + (i >> 5); }

// forward: rounds of 3 stages, T = N2/8, N2/64, ..., 1
template <int N2>
__global__ void __launch_bounds__(N2 / 8) ntt_fwd_rows(uint32_t* __restrict__ data, uint64_t stride, uint32_t n,
                                                       const uint2* __restrict__ tw, uint32_t q, int final_reduce) {
  __shared__ uint32_t s[N2 + N2 / 32];
  const uint32_t b = blockIdx.x;
  uint32_t* a = data + blockIdx.y * stride + (size_t)b * N2;
  const uint32_t tau = threadIdx.x;
  const uint32_t q2 = 2 * q;
  for (uint32_t i = tau; i < N2 / 4; i += N2 / 8) {
    const uint4 v = reinterpret_cast<const uint4*>(a)[i];
    s[pad(4 * i)] = v.x;
    s[pad(4 * i + 1)] = v.y;
    s[pad(4 * i + 2)] = v.z;
    s[pad(4 * i + 3)] = v.w;
  }
  __syncthreads();
#pragma unroll
  for (int T = N2 / 8; T >= 1; T /= 8) {
    const uint32_t j0 = (tau / T) * 8 * T + (tau % T);
    uint32_t x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = s[pad(j0 + e * T)];
    // global butterfly-group index of this thread's 8T block, and m of the first stage (t = 4T)
    const uint32_t m0 = n / (8 * T);
    const uint32_t i0 = b * (N2 / (8 * T)) + tau / T;
    {
      const uint2 w = ldtw(tw, m0 + i0);
#pragma unroll
      for (int e = 0; e < 4; ++e) ct_bf(x[e], x[e + 4], w, q2, q);
    }
    {
      const uint4 w2 = __ldg(reinterpret_cast<const uint4*>(tw + 2 * m0 + 2 * i0));
      const uint2 wa = make_uint2(w2.x, w2.y), wb = make_uint2(w2.z, w2.w);
      ct_bf(x[0], x[2], wa, q2, q);
      ct_bf(x[1], x[3], wa, q2, q);
      ct_bf(x[4], x[6], wb, q2, q);
      ct_bf(x[5], x[7], wb, q2, q);
    }
    {
      const uint4* p = reinterpret_cast<const uint4*>(tw + 4 * m0 + 4 * i0);
      const uint4 w01 = __ldg(p), w23 = __ldg(p + 1);
      ct_bf(x[0], x[1], make_uint2(w01.x, w01.y), q2, q);
      ct_bf(x[2], x[3], make_uint2(w01.z, w01.w), q2, q);
      ct_bf(x[4], x[5], make_uint2(w23.x, w23.y), q2, q);
      ct_bf(x[6], x[7], make_uint2(w23.z, w23.w), q2, q);
    }
    if (T == 1) {
      // last round: 8 contiguous outputs, straight to global
      if (final_reduce) {
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = reduce4(x[e], q);
      }
      uint4* dst = reinterpret_cast<uint4*>(a + 8 * tau);
      dst[0] = make_uint4(x[0], x[1], x[2], x[3]);
      dst[1] = make_uint4(x[4], x[5], x[6], x[7]);
    } else {
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 8; ++e) s[pad(j0 + e * T)] = x[e];
      __syncthreads();
    }
  }
}

// inverse: rounds of 3 stages, T = 1, 8, 64, ...
template <int N2>
__global__ void __launch_bounds__(N2 / 8) ntt_inv_rows(uint32_t* __restrict__ data, uint64_t stride, uint32_t n,
                                                       const uint2* __restrict__ tw, uint32_t q, uint32_t ninv,
                                                       uint32_t ninvp, int do_scale) {
  __shared__ uint32_t s[N2 + N2 / 32];
  const uint32_t b = blockIdx.x;
  uint32_t* a = data + blockIdx.y * stride + (size_t)b * N2;
  const uint32_t tau = threadIdx.x;
  const uint32_t q2 = 2 * q;
#pragma unroll
  for (int T = 1; T < N2; T *= 8) {
    const uint32_t j0 = (tau / T) * 8 * T + (tau % T);
    uint32_t x[8];
    if (T == 1) {
      const uint4* src = reinterpret_cast<const uint4*>(a + 8 * tau);
      const uint4 v0 = src[0], v1 = src[1];
      x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
      x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = s[pad(j0 + e * T)];
    }
    const uint32_t h0 = n / (2 * T);                 // h of the first stage (t = T)
    const uint32_t i0 = b * (N2 / (8 * T)) + tau / T;
    {
      const uint4* p = reinterpret_cast<const uint4*>(tw + h0 + 4 * i0);
      const uint4 w01 = __ldg(p), w23 = __ldg(p + 1);
      gs_bf(x[0], x[1], make_uint2(w01.x, w01.y), q2, q);
      gs_bf(x[2], x[3], make_uint2(w01.z, w01.w), q2, q);
      gs_bf(x[4], x[5], make_uint2(w23.x, w23.y), q2, q);
      gs_bf(x[6], x[7], make_uint2(w23.z, w23.w), q2, q);
    }
    {
      const uint4 w2 = __ldg(reinterpret_cast<const uint4*>(tw + h0 / 2 + 2 * i0));
      const uint2 wa = make_uint2(w2.x, w2.y), wb = make_uint2(w2.z, w2.w);
      gs_bf(x[0], x[2], wa, q2, q);
      gs_bf(x[1], x[3], wa, q2, q);
      gs_bf(x[4], x[6], wb, q2, q);
      gs_bf(x[5], x[7], wb, q2, q);
    }
    {
      const uint2 w = ldtw(tw, h0 / 4 + i0);
#pragma unroll
      for (int e = 0; e < 4; ++e) gs_bf(x[e], x[e + 4], w, q2, q);
    }
    if (T != 1) __syncthreads();
#pragma unroll
    for (int e = 0; e < 8; ++e) s[pad(j0 + e * T)] = x[e];
    __syncthreads();
  }
  for (uint32_t i = tau; i < N2 / 4; i += N2 / 8) {
    uint32_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t z = s[pad(4 * i + e)];
      v[e] = do_scale ? shoup_mul(z, ninv, ninvp, q) : z;
    }
    reinterpret_cast<uint4*>(a)[i] = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

// ---------------------------------------------------------------- dispatch
template <typename F>
static cudaError_t with_n1(uint32_t n1, F f) {
  switch (n1) {
    case 2: return f(std::integral_constant<int, 2>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 8: return f(std::integral_constant<int, 8>{});
    case 16: return f(std::integral_constant<int, 16>{});
  }
  return cudaErrorInvalidValue;
}
template <typename F>
static cudaError_t with_n2(uint32_t n2, F f) {
  switch (n2) {
    case 64: return f(std::integral_constant<int, 64>{});
    case 512: return f(std::integral_constant<int, 512>{});
    case 4096: return f(std::integral_constant<int, 4096>{});
  }
  return cudaErrorInvalidValue;
}
// n = n1 * n2 with n2 the largest power of 8 <= min(n, 4096), n1 <= 16
static bool split(uint32_t n, uint32_t& n1, uint32_t& n2) {
  for (uint32_t c : {4096u, 512u, 64u}) {
    if (c <= n && n % c == 0 && n / c <= 16) {
      n2 = c;
      n1 = n / c;
      return true;
    }
  }
  return false;
}

cudaError_t ntt_forward(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t st) {
  uint32_t n1, n2;
  if (!split(t.n, n1, n2)) return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  const uint2* tw = reinterpret_cast<const uint2*>(t.fw);
  cudaError_t e = cudaSuccess;
  if (n1 > 1) {
    e = with_n1(n1, [&](auto N1) {
      dim3 g((n2 + 255) / 256, count);
      ntt_fwd_cols<decltype(N1)::value><<<g, 256, 0, st>>>(data, stride, n2, tw, t.q);
      return cudaGetLastError();
    });
    if (e != cudaSuccess) return e;
  }
  return with_n2(n2, [&](auto N2) {
    dim3 g(n1, count);
    ntt_fwd_rows<decltype(N2)::value><<<g, decltype(N2)::value / 8, 0, st>>>(data, stride, t.n, tw, t.q, 1);
    return cudaGetLastError();
  });
}

cudaError_t ntt_inverse(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t st) {
  uint32_t n1, n2;
  if (!split(t.n, n1, n2)) return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  const uint2* tw = reinterpret_cast<const uint2*>(t.iv);
  cudaError_t e = with_n2(n2, [&](auto N2) {
    dim3 g(n1, count);
    ntt_inv_rows<decltype(N2)::value><<<g, decltype(N2)::value / 8, 0, st>>>(data, stride, t.n, tw, t.q, t.ninv,
                                                                             t.ninvp, n1 == 1);
    return cudaGetLastError();
  });
  if (e != cudaSuccess || n1 == 1) return e;
  return with_n1(n1, [&](auto N1) {
    dim3 g((n2 + 255) / 256, count);
    ntt_inv_cols<decltype(N1)::value><<<g, 256, 0, st>>>(data, stride, n2, tw, t.q, t.ninv, t.ninvp);
    return cudaGetLastError();
  });
}

}  // namespace he
