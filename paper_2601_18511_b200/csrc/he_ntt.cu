// he_ntt.cu -- K2: negacyclic NTT / INTT over Z_q[X]/(X^n + 1), n in {64 * 8^i} x {1,2,4,8,16}, q < 2^30.
//
// The transform is the merged-twiddle Cooley-Tukey (natural -> bit-reversed) / Gentleman-Sande
// (bit-reversed -> natural, scaled by n^-1) pair the oracle restates (oracle/he_oracle.c
// ntt_fwd / ntt_inv), so outputs agree word for word.  n = n1 * n2:
//   "cols" pass: the log2(n1) outer stages act on n2 independent strided columns; one column per
//               thread, all n1 (<= 16) elements in registers, twiddles warp-uniform.
//   "rows" pass: the log2(n2) inner stages act on contiguous n2-word blocks (n2 = 16^R <= 4096), one
//               CTA per block, n2/16 threads x 16 register-resident elements; each radix-16 round does
//               4 stages in registers; the first round reads global memory directly and the last writes
//               it directly, so a 4096-point block needs two shared-memory exchanges.
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
    if (i < 16) {
      t.fw16[i] = make_uint2(h[2 * i], h[2 * i + 1]);
      t.iv16[i] = make_uint2(h[2 * (size_t)n + 2 * i], h[2 * (size_t)n + 2 * i + 1]);
    }
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

// ---------------------------------------------------------------- job tables
// One launch transforms up to kNttMaxJobs batches that share the degree, batch count and stride but may differ in
// modulus and base pointer (blockIdx.z = job): the RNS limbs / components of a ciphertext batch in one launch.
constexpr int kNttMaxJobs = 16;
struct NttJobs {
  uint32_t* data[kNttMaxJobs];
  const uint2* tw[kNttMaxJobs];
  uint32_t q[kNttMaxJobs], ninv[kNttMaxJobs], ninvp[kNttMaxJobs];
};

// ---------------------------------------------------------------- cols pass (outer stages)
template <int N1>
__global__ void __launch_bounds__(256) ntt_fwd_cols(const __grid_constant__ NttJobs J, uint64_t stride, uint32_t n2) {
  uint32_t* __restrict__ data = J.data[blockIdx.z];
  const uint2* __restrict__ tw = J.tw[blockIdx.z];
  const uint32_t q = J.q[blockIdx.z];
  const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n2) return;
  uint32_t* a = data + blockIdx.y * stride + col;
  // the N1 - 1 warp-uniform twiddles first (L1/L2 hits), then the strided column loads from HBM
  uint2 w[N1];
#pragma unroll
  for (int i = 1; i < N1; ++i) w[i] = ldtw(tw, i);
  uint32_t x[N1];
#pragma unroll
  for (int v = 0; v < N1; ++v) x[v] = a[(size_t)n2 * v];
  const uint32_t q2 = 2 * q;
#pragma unroll
  for (int m = 1, t = N1 / 2; m < N1; m <<= 1, t >>= 1) {
#pragma unroll
    for (int i = 0; i < m; ++i) {
#pragma unroll
      for (int u = 0; u < t; ++u) ct_bf(x[2 * i * t + u], x[2 * i * t + u + t], w[m + i], q2, q);
    }
  }
#pragma unroll
  for (int v = 0; v < N1; ++v) a[(size_t)n2 * v] = x[v];
}

// single-batch forms with plain parameters (the multi-job form's indexed parameter loads cost the standalone
// 2^16 forward ~8%: 0.254 -> 0.277 ms for 1024 polys); the N1 - 1 twiddles are kernel parameters
// (NttTable::fw16 / iv16: constant-bank operands, no loads)
struct Tw16 {
  uint2 w[16];
};
template <int N1>
__global__ void __launch_bounds__(256) ntt_fwd_cols1(uint32_t* __restrict__ data, uint64_t stride, uint32_t n2,
                                                     const Tw16 tw, uint32_t q) {
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
#pragma unroll
      for (int u = 0; u < t; ++u) ct_bf(x[2 * i * t + u], x[2 * i * t + u + t], tw.w[m + i], q2, q);
    }
  }
#pragma unroll
  for (int v = 0; v < N1; ++v) a[(size_t)n2 * v] = x[v];
}
template <int N1>
__global__ void __launch_bounds__(256) ntt_inv_cols1(uint32_t* __restrict__ data, uint64_t stride, uint32_t n2,
                                                     const Tw16 tw, uint32_t q, uint32_t ninv, uint32_t ninvp) {
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
#pragma unroll
      for (int u = 0; u < t; ++u) gs_bf(x[2 * i * t + u], x[2 * i * t + u + t], tw.w[h + i], q2, q);
    }
  }
#pragma unroll
  for (int v = 0; v < N1; ++v) a[(size_t)n2 * v] = shoup_mul(x[v], ninv, ninvp, q);
}

template <int N1>
__global__ void __launch_bounds__(256) ntt_inv_cols(const __grid_constant__ NttJobs J, uint64_t stride, uint32_t n2) {
  uint32_t* __restrict__ data = J.data[blockIdx.z];
  const uint2* __restrict__ tw = J.tw[blockIdx.z];
  const uint32_t q = J.q[blockIdx.z], ninv = J.ninv[blockIdx.z], ninvp = J.ninvp[blockIdx.z];
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

// One radix-16 round = 4 CT stages on the 16 elements j0 + e*T of this thread (t = 8T .. T), for NP
// transforms at once (same twiddles: NP polys of one batch, block b of each) -- NP-fold ILP per load.
// i0: group index of the thread's 16T block at the round's first stage, m0 = n / (16 T).
template <int NP>
HE_D void ct_round16(uint32_t (&x)[NP][16], const uint2* __restrict__ tw, uint32_t m0, uint32_t i0, uint32_t q2,
                     uint32_t q) {
  {
    const uint2 w = __ldg(tw + m0 + i0);
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int p = 0; p < NP; ++p) ct_bf(x[p][e], x[p][e + 8], w, q2, q);
  }
  {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(tw + 2 * m0 + 2 * i0));
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        ct_bf(x[p][e], x[p][e + 4], make_uint2(w.x, w.y), q2, q);
        ct_bf(x[p][8 + e], x[p][12 + e], make_uint2(w.z, w.w), q2, q);
      }
  }
  {
    const uint4* pp = reinterpret_cast<const uint4*>(tw + 4 * m0 + 4 * i0);
    const uint4 wa = __ldg(pp), wb = __ldg(pp + 1);
    const uint2 ws[4] = {make_uint2(wa.x, wa.y), make_uint2(wa.z, wa.w), make_uint2(wb.x, wb.y), make_uint2(wb.z, wb.w)};
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        ct_bf(x[p][4 * g], x[p][4 * g + 2], ws[g], q2, q);
        ct_bf(x[p][4 * g + 1], x[p][4 * g + 3], ws[g], q2, q);
      }
  }
  {
    const uint4* pp = reinterpret_cast<const uint4*>(tw + 8 * m0 + 8 * i0);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint4 w = __ldg(pp + h);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        ct_bf(x[p][4 * h], x[p][4 * h + 1], make_uint2(w.x, w.y), q2, q);
        ct_bf(x[p][4 * h + 2], x[p][4 * h + 3], make_uint2(w.z, w.w), q2, q);
      }
    }
  }
}
// One radix-16 GS round = 4 stages t = T .. 8T; h0 = n / (2T).
template <int NP>
HE_D void gs_round16(uint32_t (&x)[NP][16], const uint2* __restrict__ tw, uint32_t h0, uint32_t i0, uint32_t q2,
                     uint32_t q) {
  {
    const uint4* pp = reinterpret_cast<const uint4*>(tw + h0 + 8 * i0);
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint4 w = __ldg(pp + h);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        gs_bf(x[p][4 * h], x[p][4 * h + 1], make_uint2(w.x, w.y), q2, q);
        gs_bf(x[p][4 * h + 2], x[p][4 * h + 3], make_uint2(w.z, w.w), q2, q);
      }
    }
  }
  {
    const uint4* pp = reinterpret_cast<const uint4*>(tw + h0 / 2 + 4 * i0);
    const uint4 wa = __ldg(pp), wb = __ldg(pp + 1);
    const uint2 ws[4] = {make_uint2(wa.x, wa.y), make_uint2(wa.z, wa.w), make_uint2(wb.x, wb.y), make_uint2(wb.z, wb.w)};
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        gs_bf(x[p][4 * g], x[p][4 * g + 2], ws[g], q2, q);
        gs_bf(x[p][4 * g + 1], x[p][4 * g + 3], ws[g], q2, q);
      }
  }
  {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(tw + h0 / 4 + 2 * i0));
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        gs_bf(x[p][e], x[p][e + 4], make_uint2(w.x, w.y), q2, q);
        gs_bf(x[p][8 + e], x[p][12 + e], make_uint2(w.z, w.w), q2, q);
      }
  }
  {
    const uint2 w = __ldg(tw + h0 / 8 + i0);
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int p = 0; p < NP; ++p) gs_bf(x[p][e], x[p][e + 8], w, q2, q);
  }
}

// smem offset of element j0 + e T relative to pad(j0) for the thread layouts of the rounds below
// (j0 = (tau / T) 16 T + tau % T with T in {1, 16, 256}: j0 % 32 + e T never carries past the
// next multiple of 32 except through e T itself, so the offset is a compile-time constant)
template <int T>
HE_D constexpr uint32_t poff(int e) {
  return T >= 32 ? (uint32_t)(e * T + e * T / 32) : (T == 16 ? (uint32_t)(16 * e + e / 2) : (uint32_t)e);
}

// 4096-point exchange layout (no padding): word i at i ^ 4 sx(i / 32), sx(X) = (X mod 4) | 4 (bit 3 of X) -- an
// XOR of the 16-byte granule inside each 128-byte row.  The three access patterns of the rounds are then all
// conflict-free: (A) tau + 256 e (32 consecutive words per warp), (B) j0 + 16 e with j0 = 256 (tau / 16) + tau % 16
// (the two half-warps land in opposite 64-byte halves of the row; with the additive pad they shared 8 banks), and
// (C) the 16 consecutive words of thread tau as 4 x 16-byte accesses (8 lanes per quarter-warp on 8 granules).
HE_D uint32_t swz_a(uint32_t tau, int e) { return (tau ^ (((tau >> 5) & 3) << 2) ^ ((e & 1) << 4)) + 256 * e; }
HE_D uint32_t swz_b(uint32_t tau, int e) {
  return 256 * (tau >> 4) + ((tau & 15) ^ (4 * ((e >> 1) & 3))) + 32 * (e >> 1) + 16 * ((e & 1) ^ ((tau >> 4) & 1));
}
HE_D uint32_t swz_c(uint32_t tau, int v) {   // granule v (words 4 v .. 4 v + 3) of thread tau's 16
  const uint32_t sx = ((tau >> 1) & 3) | (((tau >> 4) & 1) << 2);
  return 32 * (tau >> 1) + 4 * ((4 * (tau & 1) + v) ^ sx);
}
constexpr int kNttSwz = 4096;                 // the rows size that uses the swizzled exchange layout
template <int N2>
constexpr int rows_smem_words() { return N2 == kNttSwz ? N2 : N2 + N2 / 32; }

// forward: rounds of 4 stages, T = N2/16, N2/256, ..., 1; first round straight from global.  NP transforms
// (polys blockIdx.y * NP .. + NP - 1 of the batch, block b of each) per CTA share every twiddle load.
template <int N2, int NP, int MINB = 1>
__global__ void __launch_bounds__(N2 / 16, MINB) ntt_fwd_rows(const __grid_constant__ NttJobs J, uint64_t stride,
                                                        uint32_t n, int final_reduce) {
  uint32_t* __restrict__ data = J.data[blockIdx.z];
  const uint2* __restrict__ tw = J.tw[blockIdx.z];
  const uint32_t q = J.q[blockIdx.z];
  __shared__ __align__(16) uint32_t s[NP][rows_smem_words<N2>()];
  // block b of each poly = blockIdx.y: consecutive CTAs share b, so the CTAs resident on an SM read the same
  // twiddle slice (L1 hits even when the table is the 512 KB of a 2^16 transform)
  const uint32_t b = blockIdx.y;
  uint32_t* a[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) a[p] = data + ((size_t)blockIdx.x * NP + p) * stride + (size_t)b * N2;
  const uint32_t tau = threadIdx.x;
  const uint32_t q2 = 2 * q;
  uint32_t x[NP][16];
#pragma unroll
  for (int p = 0; p < NP; ++p)
#pragma unroll
    for (int e = 0; e < 16; ++e) x[p][e] = a[p][tau + e * (N2 / 16)];  // coalesced across the warp
  ct_round16<NP>(x, tw, n / N2, b, q2, q);
  if constexpr (N2 == kNttSwz) {
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int e = 0; e < 16; ++e) s[p][swz_a(tau, e)] = x[p][e];
    __syncthreads();
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int e = 0; e < 16; ++e) x[p][e] = s[p][swz_b(tau, e)];
    ct_round16<NP>(x, tw, n / 256, b * 16 + tau / 16, q2, q);
    // each thread writes back exactly the words it read; rounds 2 -> 3 stay inside the half-warp's 256-word
    // sub-block, so one __syncwarp orders the store before the round-3 loads
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int e = 0; e < 16; ++e) s[p][swz_b(tau, e)] = x[p][e];
    __syncwarp();
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const uint4 w = *reinterpret_cast<const uint4*>(&s[p][swz_c(tau, v)]);
        x[p][4 * v] = w.x, x[p][4 * v + 1] = w.y, x[p][4 * v + 2] = w.z, x[p][4 * v + 3] = w.w;
      }
    ct_round16<NP>(x, tw, n / 16, b * (N2 / 16) + tau, q2, q);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (final_reduce) {
#pragma unroll
        for (int e = 0; e < 16; ++e) x[p][e] = reduce4(x[p][e], q);
      }
      uint4* dst = reinterpret_cast<uint4*>(a[p] + 16 * tau);
#pragma unroll
      for (int v = 0; v < 4; ++v) dst[v] = make_uint4(x[p][4 * v], x[p][4 * v + 1], x[p][4 * v + 2], x[p][4 * v + 3]);
    }
    return;
  } else if constexpr (N2 == 16) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (final_reduce) {
#pragma unroll
        for (int e = 0; e < 16; ++e) x[p][e] = reduce4(x[p][e], q);
      }
      uint4* dst = reinterpret_cast<uint4*>(a[p]);
#pragma unroll
      for (int v = 0; v < 4; ++v) dst[v] = make_uint4(x[p][4 * v], x[p][4 * v + 1], x[p][4 * v + 2], x[p][4 * v + 3]);
    }
    return;
  } else {
    {
      constexpr int T = N2 / 16;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        uint32_t* ps = s[p] + pad(tau);
#pragma unroll
        for (int e = 0; e < 16; ++e) ps[poff<T>(e)] = x[p][e];
      }
      __syncthreads();
    }
    if constexpr (N2 == 4096) {
      constexpr int T = 16;
      const uint32_t j0 = (tau / T) * 16 * T + (tau % T);
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e) x[p][e] = s[p][pad(j0) + poff<T>(e)];
      ct_round16<NP>(x, tw, n / (16 * T), b * (N2 / (16 * T)) + tau / T, q2, q);
      // rounds 2 -> 3 exchange within the 256-word sub-block of this half-warp: no CTA barrier
      __syncwarp();
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e) s[p][pad(j0) + poff<T>(e)] = x[p][e];
      __syncwarp();
    }
    {
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e) x[p][e] = s[p][pad(16 * tau) + e];
      ct_round16<NP>(x, tw, n / 16, b * (N2 / 16) + tau, q2, q);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (final_reduce) {
#pragma unroll
          for (int e = 0; e < 16; ++e) x[p][e] = reduce4(x[p][e], q);
        }
        uint4* dst = reinterpret_cast<uint4*>(a[p] + 16 * tau);
#pragma unroll
        for (int v = 0; v < 4; ++v) dst[v] = make_uint4(x[p][4 * v], x[p][4 * v + 1], x[p][4 * v + 2], x[p][4 * v + 3]);
      }
    }
  }
}

// inverse: rounds of 4 stages, T = 1, 16, 256, ...; first round straight from global (16 contiguous words),
// last round straight to global (coalesced), optional n^-1 scaling
template <int N2, int NP, int MINB = 1>
__global__ void __launch_bounds__(N2 / 16, MINB) ntt_inv_rows(const __grid_constant__ NttJobs J, uint64_t stride,
                                                        uint32_t n, int do_scale) {
  uint32_t* __restrict__ data = J.data[blockIdx.z];
  const uint2* __restrict__ tw = J.tw[blockIdx.z];
  const uint32_t q = J.q[blockIdx.z], ninv = J.ninv[blockIdx.z], ninvp = J.ninvp[blockIdx.z];
  __shared__ __align__(16) uint32_t s[NP][rows_smem_words<N2>()];
  // block b of each poly = blockIdx.y: consecutive CTAs share b, so the CTAs resident on an SM read the same
  // twiddle slice (L1 hits even when the table is the 512 KB of a 2^16 transform)
  const uint32_t b = blockIdx.y;
  uint32_t* a[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) a[p] = data + ((size_t)blockIdx.x * NP + p) * stride + (size_t)b * N2;
  const uint32_t tau = threadIdx.x;
  const uint32_t q2 = 2 * q;
  uint32_t x[NP][16];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const uint4* src = reinterpret_cast<const uint4*>(a[p] + 16 * tau);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint4 w = src[v];
      x[p][4 * v] = w.x;
      x[p][4 * v + 1] = w.y;
      x[p][4 * v + 2] = w.z;
      x[p][4 * v + 3] = w.w;
    }
  }
  gs_round16<NP>(x, tw, n / 2, b * (N2 / 16) + tau, q2, q);
  if constexpr (N2 == kNttSwz) {
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        *reinterpret_cast<uint4*>(&s[p][swz_c(tau, v)]) = make_uint4(x[p][4 * v], x[p][4 * v + 1], x[p][4 * v + 2], x[p][4 * v + 3]);
    __syncwarp();   // rounds 1 -> 2 stay inside the half-warp's 256-word sub-block
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int e = 0; e < 16; ++e) x[p][e] = s[p][swz_b(tau, e)];
    gs_round16<NP>(x, tw, n / 32, b * 16 + tau / 16, q2, q);
    // each thread writes back exactly the words it read: no barrier before the store
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int e = 0; e < 16; ++e) s[p][swz_b(tau, e)] = x[p][e];
    __syncthreads();
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int e = 0; e < 16; ++e) x[p][e] = s[p][swz_a(tau, e)];
    gs_round16<NP>(x, tw, n / 512, b, q2, q);
  } else if constexpr (N2 > 16) {
    {
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e) s[p][pad(16 * tau) + e] = x[p][e];
      if constexpr (N2 == 4096) __syncwarp();   // rounds 1 -> 2 stay inside the half-warp's 256-word sub-block
      else __syncthreads();
    }
    if constexpr (N2 == 4096) {
      constexpr int T = 16;
      const uint32_t j0 = (tau / T) * 16 * T + (tau % T);
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e) x[p][e] = s[p][pad(j0) + poff<T>(e)];
      gs_round16<NP>(x, tw, n / (2 * T), b * (N2 / (16 * T)) + tau / T, q2, q);
      __syncthreads();
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e) s[p][pad(j0) + poff<T>(e)] = x[p][e];
      __syncthreads();
    }
    {
      constexpr int T = N2 / 16;
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e) x[p][e] = s[p][pad(tau) + poff<T>(e)];
      gs_round16<NP>(x, tw, n / (2 * T), b, q2, q);
    }
  }
  {
    constexpr int T = N2 / 16;
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int e = 0; e < 16; ++e) a[p][tau + e * T] = do_scale ? shoup_mul(x[p][e], ninv, ninvp, q) : x[p][e];
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
    case 16: return f(std::integral_constant<int, 16>{});
    case 256: return f(std::integral_constant<int, 256>{});
    case 4096: return f(std::integral_constant<int, 4096>{});
  }
  return cudaErrorInvalidValue;
}
// n = n1 * n2 with n2 the largest power of 16 <= min(n, 4096), n1 <= 16
static bool split(uint32_t n, uint32_t& n1, uint32_t& n2) {
  for (uint32_t c : {4096u, 256u, 16u}) {
    if (c <= n && n % c == 0 && n / c <= 16) {
      n2 = c;
      n1 = n / c;
      return true;
    }
  }
  return false;
}

static NttJobs make_jobs(const NttTable* const* t, uint32_t* const* data, int njobs, bool inverse) {
  NttJobs J{};
  for (int i = 0; i < njobs; ++i) {
    J.data[i] = data[i];
    J.tw[i] = reinterpret_cast<const uint2*>(inverse ? t[i]->iv : t[i]->fw);
    J.q[i] = t[i]->q;
    J.ninv[i] = t[i]->ninv;
    J.ninvp[i] = t[i]->ninvp;
  }
  return J;
}
static NttJobs shift_jobs(NttJobs J, int njobs, uint64_t off) {
  for (int i = 0; i < njobs; ++i) J.data[i] += off;
  return J;
}

cudaError_t ntt_forward_multi(const NttTable* const* t, uint32_t* const* data, int njobs, uint32_t count,
                              uint64_t stride, cudaStream_t st, bool rows_only, bool reduce) {
  if (njobs < 1 || njobs > kNttMaxJobs) return cudaErrorInvalidValue;
  const uint32_t n = t[0]->n;
  for (int i = 1; i < njobs; ++i)
    if (t[i]->n != n) return cudaErrorInvalidValue;
  uint32_t n1, n2;
  if (!split(n, n1, n2)) return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  const NttJobs J = make_jobs(t, data, njobs, false);
  cudaError_t e = cudaSuccess;
  if (n1 > 1 && !rows_only) {
    e = with_n1(n1, [&](auto N1) {
      dim3 g((n2 + 255) / 256, count, njobs);
      if (njobs == 1) {
        Tw16 tw;
        for (int i = 0; i < 16; ++i) tw.w[i] = t[0]->fw16[i];
        ntt_fwd_cols1<decltype(N1)::value><<<g, 256, 0, st>>>(J.data[0], stride, n2, tw, J.q[0]);
      }
      else ntt_fwd_cols<decltype(N1)::value><<<g, 256, 0, st>>>(J, stride, n2);
      return cudaGetLastError();
    });
    if (e != cudaSuccess) return e;
  }
  return with_n2(n2, [&](auto N2) {
    constexpr int K = decltype(N2)::value;
    if (count / 2) {
      // 4096-point blocks: compiled for 4 resident CTAs per SM (<= 64 registers, 32 warps); measured against
      // 3 / 5 CTAs and one poly per CTA at 6 / 7
      dim3 g(count / 2, n1, njobs);
      if constexpr (K == 4096) ntt_fwd_rows<K, 2, 4><<<g, K / 16, 0, st>>>(J, stride, n, reduce);
      else ntt_fwd_rows<K, 2><<<g, K / 16, 0, st>>>(J, stride, n, reduce);
    }
    if (count & 1) {
      dim3 g(1, n1, njobs);
      ntt_fwd_rows<K, 1><<<g, K / 16, 0, st>>>(shift_jobs(J, njobs, (uint64_t)(count - 1) * stride), stride, n,
                                               reduce);
    }
    return cudaGetLastError();
  });
}

cudaError_t ntt_inverse_multi(const NttTable* const* t, uint32_t* const* data, int njobs, uint32_t count,
                              uint64_t stride, cudaStream_t st) {
  if (njobs < 1 || njobs > kNttMaxJobs) return cudaErrorInvalidValue;
  const uint32_t n = t[0]->n;
  for (int i = 1; i < njobs; ++i)
    if (t[i]->n != n) return cudaErrorInvalidValue;
  uint32_t n1, n2;
  if (!split(n, n1, n2)) return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  const NttJobs J = make_jobs(t, data, njobs, true);
  cudaError_t e = with_n2(n2, [&](auto N2) {
    constexpr int K = decltype(N2)::value;
    if (count / 2) {
      dim3 g(count / 2, n1, njobs);
      if constexpr (K == 4096) ntt_inv_rows<K, 2, 4><<<g, K / 16, 0, st>>>(J, stride, n, n1 == 1);
      else ntt_inv_rows<K, 2><<<g, K / 16, 0, st>>>(J, stride, n, n1 == 1);
    }
    if (count & 1) {
      dim3 g(1, n1, njobs);
      ntt_inv_rows<K, 1><<<g, K / 16, 0, st>>>(shift_jobs(J, njobs, (uint64_t)(count - 1) * stride), stride, n, n1 == 1);
    }
    return cudaGetLastError();
  });
  if (e != cudaSuccess || n1 == 1) return e;
  return with_n1(n1, [&](auto N1) {
    dim3 g((n2 + 255) / 256, count, njobs);
    if (njobs == 1) {
      Tw16 tw;
      for (int i = 0; i < 16; ++i) tw.w[i] = t[0]->iv16[i];
      ntt_inv_cols1<decltype(N1)::value><<<g, 256, 0, st>>>(J.data[0], stride, n2, tw, J.q[0], J.ninv[0], J.ninvp[0]);
    } else {
      ntt_inv_cols<decltype(N1)::value><<<g, 256, 0, st>>>(J, stride, n2);
    }
    return cudaGetLastError();
  });
}

cudaError_t ntt_forward(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t st,
                        bool rows_only) {
  const NttTable* tp = &t;
  return ntt_forward_multi(&tp, &data, 1, count, stride, st, rows_only);
}

cudaError_t ntt_inverse(const NttTable& t, uint32_t* data, uint32_t count, uint64_t stride, cudaStream_t st) {
  const NttTable* tp = &t;
  return ntt_inverse_multi(&tp, &data, 1, count, stride, st);
}

}  // namespace he
