// he_spectral.cu -- the spectral form of the MLWE PCMM's a-part GEMM (K7 = S1..S4).
//
// The a-part of the MLWE PCMM is, per limb q and output row y,
//   v[y][d + d j + m] = sum_r sum_t W~[y][k r + t] * a_r[t - j + k m]        (negacyclic read)
// i.e. for every input RLWE ct r a length-k correlation of the weight row segment
// g_{y,r}[t] = W~[y][k r + t] with a_r, sampled at c = k m - j.  The GEMM of K1 spends
// n_out * n_in * d * k word-MACs on it because it ignores that every column of the
// decomposed a-matrix is a twisted shift of the same polynomial.  Here the correlation is
// evaluated blockwise by overlap-save with a cyclic NTT of length L = 2k over Z_q:
//   window  win_{r,m}[u] = a_r[k m - k + 1 + u],  u < L            (S2, per op)
//   filter  g'_{y,r}[u]  = g_{y,r}[-u mod L]                        (S1, plan time)
//   C^_y,m[f] = sum_r  G^_{y,r}[f] * A^_{r,m}[f]   mod q,  f < L    (S3, tcgen05 GEMM per f)
//   v[y][d + d (k-1-u) + m] = INTT(C^_{y,m})[u],  u < k            (S4, + rescale)
// The values are the same residues K1 produces (exact modular arithmetic, no rounding), so
// the output is bit-identical; the work drops from d*k to ~2*L*n_in/k MACs per output word
// (128x fewer word-MACs at the Llama shapes), at the cost of full-width (not 2-digit)
// spectral weights and an L x n_out x d spectral intermediate per limb.
//
// S3 runs per frequency f a modular GEMM  C^_f (n_out x d) = G^_f (n_out x R) * A^_f (R x d),
// R = n_in / k, on tcgen05 kind::i8 exactly like K1: both operands split into D balanced
// int8 digit planes (D = 4 for q0 < 2^30, 3 for q1 ~ 2^20), one MMA per weight digit against
// the D stacked data planes writing at TMEM column offset 32 a, so digit pair (a, b) lands in
// the int32 accumulator of shift s = a + b (2D-1 accumulators per word); the epilogue sums
// acc_s * (2^(8 s) mod q) in int64 and Montgomery-reduces.  CTA pairs (cta_group::2), tiles of
// 256 rows x 32 columns, two TMEM accumulator buffers so the epilogue of one tile overlaps
// the MMAs of the next.  A operand (G^): 16-byte K chunks stored as no-swizzle core-matrix tiles
// (gidx); B operand (A^): K = R padded to 64 bytes, 64-byte swizzle.  Tiles run y-tile-major in
// runs of 4 consecutive frequencies per CTA pair; C^ lands in [row][group of 8 blocks][f][8]
// (cidx), one contiguous run per S4 unit.
#include <cuda.h>
#include <cstdlib>
#include "he_common.cuh"
#include "he_tc.cuh"
#include "he_kernels.h"

namespace he {

// C^ (S3 -> S4) layout: [y][group of 8 blocks][f][8], so the 8 blocks x L frequencies of one (row, group) -- the
// unit of the fast S4 -- are one contiguous L x 32-byte region per limb
HE_HD size_t cidx(uint32_t y, uint32_t f, uint32_t blk, uint32_t L, uint32_t nbp) {
  return (((size_t)y * (nbp >> 3) + (blk >> 3)) * L + f) * 8 + (blk & 7);
}

// ---------------------------------------------------------------- host tables
cudaError_t spec_table_init(SpecTable& t, uint32_t L, uint32_t q) {
  t.L = L;
  t.q = q;
  if (L < 4 || (L & (L - 1)) || (q - 1) % L) return cudaErrorInvalidValue;
  uint64_t w = 0;
  for (uint64_t g = 2; g < q; ++g) {
    const uint64_t c = powmod_h(g, (q - 1) / L, q);
    if (powmod_h(c, L / 2, q) != 1) {
      w = c;
      break;
    }
  }
  if (!w) return cudaErrorInvalidValue;
  const uint64_t wi = powmod_h(w, q - 2, q);
  // fast-inverse tables (he_spectral.cu S4): L = 512 -> 16 round-2 lanes (stages 4..8), L = 1024 -> 32 lanes
  // (stages 5..9); entry [i][lane] of stage s = w^-((lane + lanes i) << (log2(L/2) - s)) at lanes (2^(s - s0) - 1)
  const int lg = ilog2_h(L / 2), s0 = L == 512 ? 4 : 5, lanes = 1 << s0;
  const size_t nr2 = (L == 512 || L == 1024) ? (size_t)lanes * ((1u << (lg + 1 - s0)) - 1) : 0;
  uint32_t* h = new uint32_t[2 * (size_t)L + 4 * nr2];  // fw pairs [L/2][2], iv pairs [L/2][2], r2 pairs, f2 pairs
  uint64_t p = 1, pi = 1;
  for (uint32_t j = 0; j < L / 2; ++j) {
    h[2 * j] = (uint32_t)p;
    h[2 * j + 1] = shoup_pre((uint32_t)p, q);
    h[L + 2 * j] = (uint32_t)pi;
    h[L + 2 * j + 1] = shoup_pre((uint32_t)pi, q);
    p = p * w % q;
    pi = pi * wi % q;
  }
  for (int st = s0; st <= lg && nr2; ++st) {
    const int len = 1 << (st - s0), base = lanes * (len - 1);
    for (int i = 0; i < len; ++i)
      for (int lo = 0; lo < lanes; ++lo) {
        const uint32_t j = (uint32_t)(lo + lanes * i) << (lg - st);
        // L = 1024 inverse tables: entries i, i + 1 (i even) of a lane adjacent, so S4 reads them as one 16-byte
        // load: [base + 2 lanes (i / 2) + 2 lo + i % 2]; the single-entry first stage and L = 512 stay [i][lane]
        const size_t ri = (L == 1024 && len >= 2) ? base + 2 * lanes * (i >> 1) + 2 * lo + (i & 1)
                                                  : base + lanes * i + lo;
        h[2 * (size_t)L + 2 * ri] = h[L + 2 * j];
        h[2 * (size_t)L + 2 * ri + 1] = h[L + 2 * j + 1];
        h[2 * (size_t)L + 2 * nr2 + 2 * (base + lanes * i + lo)] = h[2 * j];        // forward (f2)
        h[2 * (size_t)L + 2 * nr2 + 2 * (base + lanes * i + lo) + 1] = h[2 * j + 1];
      }
  }
  // r1: round-1 (register) stages s = 1 .. s0 - 1, off = 1 .. 2^s - 1 at (2^s - s - 1) + off - 1
  for (int st = 1; st < s0 && nr2; ++st)
    for (int off = 1; off < (1 << st); ++off) {
      const uint32_t j = (uint32_t)off << (lg - st);
      t.r1[(1 << st) - st - 1 + off - 1] = make_uint2(h[L + 2 * j], h[L + 2 * j + 1]);
      t.f1[(1 << st) - st - 1 + off - 1] = make_uint2(h[2 * j], h[2 * j + 1]);
    }
  t.linv = (uint32_t)powmod_h(L, q - 2, q);
  t.linvp = shoup_pre(t.linv, q);
  uint32_t* dptr = nullptr;
  const size_t words = 2 * (size_t)L + 4 * nr2;
  cudaError_t e = cudaMalloc(&dptr, words * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(dptr, h, words * sizeof(uint32_t), cudaMemcpyHostToDevice);
  delete[] h;
  if (e != cudaSuccess) return e;
  t.fw = reinterpret_cast<uint2*>(dptr);
  t.iv = reinterpret_cast<uint2*>(dptr + L);
  t.r2 = nr2 ? reinterpret_cast<uint2*>(dptr + 2 * L) : nullptr;
  t.f2 = nr2 ? reinterpret_cast<uint2*>(dptr + 2 * L + 2 * nr2) : nullptr;
  return cudaSuccess;
}

void spec_table_free(SpecTable& t) {
  if (t.fw) cudaFree(t.fw);
  t.fw = t.iv = t.r2 = t.f2 = nullptr;
}

// ---------------------------------------------------------------- cooperative cyclic NTTs in shared memory
// cnt transforms of length L at x + b * ld.  Forward: DIF (natural -> bit-reversed),
// X[f] = sum_i x[i] w^(f i).  Inverse: DIT (bit-reversed -> natural) with the L^-1 scaling
// left to the caller.  Values fully reduced in [0, q).
HE_D void cyc_fwd_smem(uint32_t* x, int cnt, int ld, int L, const uint2* __restrict__ tw, uint32_t q) {
  const int half = L / 2, lh = __ffs(half) - 1;    // L is a power of two: shifts, not divisions
  for (int ll = lh; ll >= 0; --ll) {
    const int len = 1 << ll, step_sh = lh - ll;
    for (int i = threadIdx.x; i < cnt * half; i += blockDim.x) {
      const int b = i >> lh, j = i & (half - 1);
      const int off = j & (len - 1);
      uint32_t* p = x + b * ld + ((j >> ll) << (ll + 1)) + off;
      const uint32_t u = p[0], v = p[len];
      const uint2 w = __ldg(tw + (off << step_sh));
      p[0] = add_mod(u, v, q);
      p[len] = shoup_mul(sub_mod(u, v, q), w.x, w.y, q);
    }
    __syncthreads();
  }
}
HE_D void cyc_inv_smem(uint32_t* x, int cnt, int ld, int L, const uint2* __restrict__ tw, uint32_t q) {
  const int half = L / 2;
  for (int len = 1, step = half; len < L; len <<= 1, step >>= 1) {
    for (int i = threadIdx.x; i < cnt * half; i += blockDim.x) {
      const int b = i / half, j = i % half;
      const int off = j % len;
      uint32_t* p = x + b * ld + (j / len) * 2 * len + off;
      const uint2 w = __ldg(tw + off * step);
      const uint32_t u = p[0], v = shoup_mul(p[len], w.x, w.y, q);
      p[0] = add_mod(u, v, q);
      p[len] = sub_mod(u, v, q);
    }
    __syncthreads();
  }
}

HE_D void write_digits(uint32_t v, uint32_t q, int D, int8_t* dst, uint64_t plane_stride) {
  const uint32_t c = v > (q >> 1) ? v - q : v;        // two's complement of the centred residue
  const uint32_t w = (c + 0x80808080u) ^ 0x80808080u;  // byte p = balanced digit p (he_crypto.cu K3)
  for (int p = 0; p < D; ++p) dst[(size_t)p * plane_stride] = (int8_t)(w >> (8 * p));
}

// ---------------------------------------------------------------- S1: spectral weights (plan time)
// G^ int8 (balanced digit a of the transformed filter g'_{y,r}), stored as S3's A-operand tiles: plane f D + a,
// 128-row tile yt, then kg / 16 chunks of 128 rows x 16 bytes (no-swizzle UMMA core matrices, K-major), so one
// TMA box of 256-byte lines copies a whole (plane, row tile) into shared memory as is (gidx).
// One CTA per (row y, chunk of kSpecRChunk input cts).
HE_HD size_t gidx(uint32_t plane, uint32_t y, uint32_t r, uint32_t n_out, uint32_t kg) {
  const uint32_t yt = (n_out + 127) / 128;
  return (((size_t)plane * yt + (y >> 7)) * (kg >> 4) + (r >> 4)) * 2048 + (y & 127) * 16 + (r & 15);
}
constexpr int kSpecRChunk = 16;
__global__ void __launch_bounds__(256) spec_weights_kernel(const int8_t* __restrict__ wdig, uint32_t d_w, uint32_t n_out,
                                                           uint32_t n_in, uint32_t k, uint32_t L, uint32_t q, int D,
                                                           uint32_t r_pad, const uint2* __restrict__ tw, uint32_t linv,
                                                           uint32_t linvp, int8_t* __restrict__ out) {
  extern __shared__ uint32_t xs[];  // [kSpecRChunk][L]
  const uint32_t y = blockIdx.x, r0 = blockIdx.y * kSpecRChunk;
  const uint32_t R = n_in / k;
  const int cnt = (int)min((uint32_t)kSpecRChunk, R - r0);
  for (int i = threadIdx.x; i < cnt * (int)L; i += blockDim.x) xs[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < cnt * (int)k; i += blockDim.x) {
    const int b = i / (int)k, t = i % (int)k;
    const size_t x = (size_t)(r0 + b) * k + t;
    int64_t w = 0;
    for (int a = (int)d_w - 1; a >= 0; --a) w = w * 256 + wdig[((size_t)a * n_out + y) * n_in + x];
    int64_t m = w % (int64_t)q;
    if (m < 0) m += q;
    xs[b * L + ((L - t) & (L - 1))] = (uint32_t)m;  // g'[-t mod L] = g[t]
  }
  __syncthreads();
  cyc_fwd_smem(xs, cnt, (int)L, (int)L, tw, q);
  const uint64_t plane = gidx(1, 0, 0, n_out, r_pad);   // bytes per digit plane (r_pad = kg here)
  for (int i = threadIdx.x; i < cnt * (int)L; i += blockDim.x) {
    const int f = i / cnt, b = i % cnt;  // consecutive threads: consecutive r (bytes)
    int8_t* dst = out + gidx((uint32_t)f * D, y, r0 + b, n_out, r_pad);
    write_digits(shoup_mul(xs[b * L + f], linv, linvp, q), q, D, dst, plane);  // L^-1 of the INTT folded in
  }
}

// ---------------------------------------------------------------- S2: spectral data windows (per op)
// A^[f][b][blk][r_pad] int8, block blk covering outputs c' = ob blk .. ob blk + ob - 1 (c' = k m - j + k - 1)
// from the window a_r[ob blk - (k - 1) + u], u < L.  One CTA per (block, chunk of input cts).
__global__ void __launch_bounds__(256) spec_data_kernel(const uint32_t* __restrict__ ct, uint32_t n_ct, uint32_t limb,
                                                        uint32_t k, uint32_t ob, uint32_t nbp, uint32_t N, uint32_t L,
                                                        uint32_t q, int D, uint32_t r_pad, const uint2* __restrict__ tw,
                                                        int8_t* __restrict__ out) {
  extern __shared__ uint32_t xs[];  // [kSpecRChunk][L]
  const uint32_t m = blockIdx.x, r0 = blockIdx.y * kSpecRChunk;
  const int cnt = (int)min((uint32_t)kSpecRChunk, n_ct - r0);
  for (int i = threadIdx.x; i < cnt * (int)L; i += blockDim.x) {
    const int b = i / (int)L, u = i % (int)L;
    const uint32_t* a = ct + ((size_t)(r0 + b) * 2 + limb) * 2 * N;
    int64_t I = (int64_t)ob * m - (int64_t)k + 1 + u;
    uint32_t v;
    if (I < 0) {
      const uint32_t w = a[I + N];
      v = w ? q - w : 0u;
    } else if (I >= (int64_t)N) {
      const uint32_t w = a[I - N];
      v = w ? q - w : 0u;
    } else {
      v = a[I];
    }
    xs[i] = v;
  }
  __syncthreads();
  cyc_fwd_smem(xs, cnt, (int)L, (int)L, tw, q);
  const uint64_t plane = (uint64_t)nbp * r_pad;
  for (int i = threadIdx.x; i < cnt * (int)L; i += blockDim.x) {
    const int f = i / cnt, b = i % cnt;
    int8_t* dst = out + ((size_t)f * D * nbp + m) * r_pad + r0 + b;
    write_digits(xs[b * L + f], q, D, dst, plane);
  }
}


// Fast S2 for L = 1024: one warp per window, 32 register elements per lane, forward DIF (natural ->
// bit-reversed) in two register rounds -- stages 512 .. 32 apart on elements l + 32 e (per-stage lane
// tables f2), a per-warp smem transpose, stages 16 .. 1 apart on the lane's 32 contiguous elements
// (lane-uniform twiddles f1 as kernel parameters) -- then the digits of 16 windows x 1024 frequencies.
// GS: X, Y in [0, 2q) -> X' = X + Y, Y' = (X - Y) W, both in [0, 2q)
HE_D void gs_bf(uint32_t& x, uint32_t& y, uint2 w, uint32_t q2, uint32_t q) {
  const uint32_t s = x + y;
  const uint32_t d = x + q2 - y;
  x = min(s, s - q2);
  y = d * w.x - __umulhi(d, w.y) * q;
}
struct SpecFwdConst {
  const uint2* f2;
  uint2 f1[26];
};
constexpr int kS2Ld = 1057;   // per-warp region pitch: 1024 + 32 + 1 (odd: conflict-free digit read-out)
struct SpecData2 {   // both limbs of S2 in one launch (blockIdx.z = limb)
  SpecFwdConst cf[2];
  uint32_t q[2];
  int D[2];
  int8_t* out[2];
};
__global__ void __launch_bounds__(512) spec_data1024_kernel(const uint32_t* __restrict__ ct, uint32_t n_ct,
                                                            uint32_t k, uint32_t ob, uint32_t nbp, uint32_t N,
                                                            uint32_t r_pad, const __grid_constant__ SpecData2 sd) {
  extern __shared__ uint32_t xs[];                      // [16 windows][1057]
  const uint32_t limb = blockIdx.z;
  const SpecFwdConst& cf = sd.cf[limb];
  const uint32_t q = sd.q[limb];
  const int D = sd.D[limb];
  int8_t* __restrict__ out = sd.out[limb];
  const uint32_t m = blockIdx.x, r0 = blockIdx.y * 16;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t q2 = 2 * q;
  const uint32_t r = r0 + w;
  uint32_t* col = xs + w * kS2Ld;
  if (r < n_ct) {
    const uint32_t* a = ct + ((size_t)r * 2 + limb) * 2 * N;
    const int64_t I0 = (int64_t)ob * m - (int64_t)k + 1;
    uint32_t x[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const int64_t I = I0 + lane + 32 * e;
      uint32_t v;
      if (I < 0) {
        const uint32_t t = a[I + N];
        v = t ? q - t : 0u;
      } else if (I >= (int64_t)N) {
        const uint32_t t = a[I - N];
        v = t ? q - t : 0u;
      } else {
        v = a[I];
      }
      x[e] = v;
    }
    // round 1: len = 512 .. 32 (element distance 16 .. 1), twiddle w^((l + 32 i) << (9 - s))
#pragma unroll
    for (int s = 9; s >= 5; --s) {
      const int h = 1 << (s - 5), base = 32 * (h - 1);
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if (e & h) continue;
        gs_bf(x[e], x[e + h], __ldg(cf.f2 + base + 32 * (e & (h - 1)) + lane), q2, q);
      }
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) col[lane + 33 * e] = x[e];    // pad(l + 32 e)
    __syncwarp();
#pragma unroll
    for (int e = 0; e < 32; ++e) x[e] = col[33 * lane + e];    // pad(32 l + e)
    __syncwarp();
    // round 2: len = 16 .. 1 on the lane's contiguous elements, twiddle w^(off << (9 - s)), off = e mod len
#pragma unroll
    for (int s = 4; s >= 0; --s) {
      const int h = 1 << s;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if (e & h) continue;
        const int off = e & (h - 1);
        if (off == 0) {
          const uint32_t sm = x[e] + x[e + h], df = x[e] + q2 - x[e + h];
          x[e] = min(sm, sm - q2);
          x[e + h] = min(df, df - q2);
        } else {
          gs_bf(x[e], x[e + h], cf.f1[(1 << s) - s - 1 + off - 1], q2, q);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) col[32 * lane + e] = min(x[e], x[e] - q);   // position p, [0, q)
  }
  __syncthreads();
  // digits: for each position p the 16 windows' words are 16 consecutive bytes of every digit plane -- one
  // thread per p builds them in registers and stores each digit's 16 bytes at once (windows r >= n_ct: zeros)
  const uint32_t cnt = min(16u, n_ct - r0);
  const uint64_t plane = (uint64_t)nbp * r_pad;
  for (uint32_t p = threadIdx.x; p < 1024; p += 512) {
    uint32_t wv[16];
#pragma unroll
    for (int rl = 0; rl < 16; ++rl) {
      const uint32_t v = (uint32_t)rl < cnt ? xs[rl * kS2Ld + p] : 0u;   // lanes: consecutive p, distinct banks
      const uint32_t c = v > (q >> 1) ? v - q : v;
      wv[rl] = (c + 0x80808080u) ^ 0x80808080u;                          // balanced base-256 digits as bytes
    }
    int8_t* dst = out + ((size_t)p * D * nbp + m) * r_pad + r0;
    for (int d = 0; d < D; ++d) {
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {   // byte d of windows 4 j .. 4 j + 3
        const uint32_t sh = 8 * d;
        o[j] = ((wv[4 * j] >> sh) & 0xFF) | (((wv[4 * j + 1] >> sh) & 0xFF) << 8) |
               (((wv[4 * j + 2] >> sh) & 0xFF) << 16) | (((wv[4 * j + 3] >> sh) & 0xFF) << 24);
      }
      *reinterpret_cast<uint4*>(dst + (size_t)d * plane) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// ---------------------------------------------------------------- S4: inverse transform + rescale + store
// One CTA per (row y, group of 32 blocks m).  C^ limb i: cidx layout (row-major in y).
constexpr int kSpecMGroup = 32;
__global__ void __launch_bounds__(256) spec_inverse_kernel(const uint32_t* __restrict__ c0, const uint32_t* __restrict__ c1,
                                                           uint32_t nbp, uint32_t row0, uint32_t d, uint32_t k,
                                                           uint32_t L, SpecInvConst cst, uint32_t* __restrict__ out_a) {
  extern __shared__ uint32_t sm[];
  const uint32_t ld = L + 1;
  uint32_t* xs = sm;                       // [32 m][L + 1]
  uint32_t* keep = sm + kSpecMGroup * ld;  // [32 m][k + 1]: limb-1 result
  const uint32_t y = row0 + blockIdx.y, m0 = blockIdx.x * kSpecMGroup;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int limb = 1; limb >= 0; --limb) {
    const uint32_t* src = limb ? c1 : c0;
    const uint32_t q = cst.q[limb];
    for (uint32_t f = warp; f < L; f += nw) xs[lane * ld + f] = src[cidx(y, f, m0 + lane, L, nbp)];
    __syncthreads();
    cyc_inv_smem(xs, kSpecMGroup, (int)ld, (int)L, cst.iv[limb], q);
    if (limb) {
      for (uint32_t i = threadIdx.x; i < kSpecMGroup * k; i += blockDim.x) {
        const uint32_t mm = i / k, u = i % k;
        keep[mm * (k + 1) + u] = xs[mm * ld + u];
      }
      __syncthreads();
    }
  }
  const uint32_t q0 = cst.q[0], q1 = cst.q[1];
  const uint32_t N = d * k;
  for (uint32_t i = threadIdx.x; i < kSpecMGroup * k; i += blockDim.x) {
    const uint32_t mm = i & 31, u = i >> 5;
    const uint32_t x0 = xs[mm * ld + u];
    const uint32_t x1 = keep[mm * (k + 1) + u];
    uint32_t t;
    if (x1 > (q1 >> 1)) t = csub(x0 + (q1 - x1), q0);
    else t = sub_mod(x0, x1, q0);
    const uint32_t j = k - 1 - u;
    const size_t o = (size_t)(y - row0) * N + (size_t)d * j + m0 + mm;
    if (cst.out1) {  // level-1 words of both limbs
      out_a[o] = x0;
      cst.out1[o] = x1;
      continue;
    }
    out_a[o] = shoup_mul(t, cst.q1inv, cst.q1invp, q0);
  }
}

// Fast S4 for L = 512 (k = 256): one warp per column m, both limbs interleaved (ILP), 16
// register-resident elements per lane and limb.
//   round 1: lane l holds positions 16 l + e (e < 16): DIT stages len = 1, 2, 4, 8 in registers
//            (lane-uniform twiddles; twiddle-1 butterflies skip the multiply);
//   round 2: lane l = (l_lo, l_hi) holds l_lo + 16 e + 256 l_hi: stages len = 16 .. 128 in registers,
//            stage len = 256 across lanes l ^ 16 -- only its lower half (outputs u < 256) is formed.
//            Round-2 twiddles come from a per-stage [i][l_lo] table (one 128-B line per access).
// Harvey-lazy butterflies (values in [0, 4q)); the L^-1 of the inverse is folded into G^ (S1).
// 16 columns per CTA, both limbs resident in smem; row pitch 546 words with pad(p) = p + p/16
// keeps the transposing loads, both rounds and the row-ordered read-out conflict-free.
constexpr int kInv512Cols = 16;
constexpr int kInv512Ld = 546;
HE_D uint32_t pad16(uint32_t p) { return p + (p >> 4); }
HE_D void dit_bf(uint32_t& x, uint32_t& y, uint2 w, uint32_t q2, uint32_t q) {  // X, Y in [0, 4q)
  const uint32_t a = min(x, x - q2);
  const uint32_t t = y * w.x - __umulhi(y, w.y) * q;
  x = a + t;
  y = a + q2 - t;
}
HE_D void dit_bf1(uint32_t& x, uint32_t& y, uint32_t q2) {  // twiddle 1, X, Y in [0, 4q)
  const uint32_t a = min(x, x - q2), b = min(y, y - q2);
  x = a + b;
  y = a + q2 - b;
}
struct Inv512Limb {
 uint32_t* col;        // smem column (pitch-padded, bit-reversed positions)
  const uint2* r2;      // round-2 table: stage s at 16 (2^(s-4) - 1), entry [i][l_lo]
  uint32_t q;
};
// -> out[l][e] = INTT value u = l_lo + 16 (e + 8 l_hi) of limb l, e < 8
HE_D void inv512_pair(const Inv512Limb (&L)[2], const SpecInvConst& cst, uint32_t lane, uint32_t (&out)[2][8]) {
  uint32_t x[2][16];
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int e = 0; e < 16; ++e) x[l][e] = L[l].col[17 * lane + e];
#pragma unroll
  for (int e = 0; e < 16; e += 2)
#pragma unroll
    for (int l = 0; l < 2; ++l) dit_bf1(x[l][e], x[l][e + 1], 2 * L[l].q);
#pragma unroll
  for (int s = 1; s < 4; ++s) {
    const int len = 1 << s;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      if (e & len) continue;
      const int off = e & (len - 1);
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        if (off == 0) dit_bf1(x[l][e], x[l][e + len], 2 * L[l].q);
        else dit_bf(x[l][e], x[l][e + len], cst.r1[l][(1 << s) - s - 1 + off - 1], 2 * L[l].q, L[l].q);
      }
    }
  }
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int e = 0; e < 16; ++e) L[l].col[17 * lane + e] = x[l][e];
  __syncwarp();
  const uint32_t lo = lane & 15, hi = lane >> 4;
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int e = 0; e < 16; ++e) x[l][e] = L[l].col[lo + 17 * e + 272 * hi];
#pragma unroll
  for (int s = 4; s < 8; ++s) {
    const int len = 1 << (s - 4);
    const int base = 16 * (len - 1);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      if (e & len) continue;
      const int i = e & (len - 1);
#pragma unroll
      for (int l = 0; l < 2; ++l)
        dit_bf(x[l][e], x[l][e + len], __ldg(L[l].r2 + base + 16 * i + lo), 2 * L[l].q, L[l].q);
    }
  }
  // stage len = 256, pruned to the outputs u < 256 (X + W Y): lanes l and l ^ 16 swap half their elements
  // so lane (lo, hi) holds the pairs of positions lo + 16 (e + 8 hi), e < 8, and forms those 8 outputs
#pragma unroll
  for (int e = 0; e < 8; ++e) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const uint32_t q = L[l].q, q2 = 2 * q;
      const uint32_t send = hi ? x[l][e] : x[l][e + 8];
      const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 16);
      const uint32_t X = hi ? recv : x[l][e], Y = hi ? x[l][e + 8] : recv;
      const uint2 w = __ldg(L[l].r2 + 240 + 16 * (e + 8 * hi) + lo);
      const uint32_t t = Y * w.x - __umulhi(Y, w.y) * q;  // [0, 2q)
      uint32_t v = min(X, X - q2) + t;                    // [0, 4q)
      v = min(v, v - q2);
      out[l][e] = min(v, v - q);
    }
  }
}

__global__ void __launch_bounds__(256, 3) spec_inverse512_kernel(const uint32_t* __restrict__ c0,
                                                                 const uint32_t* __restrict__ c1, uint32_t nbp,
                                                                 uint32_t row0, uint32_t d, SpecInvConst cst,
                                                                 uint32_t* __restrict__ out_a) {
  extern __shared__ uint32_t sm[];
  uint32_t* xs0 = sm;                                // [16 m][546]
  uint32_t* xs1 = sm + kInv512Cols * kInv512Ld;      // [16 m][546]
  const uint32_t y = row0 + blockIdx.y, m0 = blockIdx.x * kInv512Cols;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // phase A: C^ (cidx layout) positions p of blocks m0 .. m0 + 15 of both limbs -> xs[m][pad(p)]
  // (16-byte loads; pitch 546 = 2 mod 32 makes the 4 scattered stores per load conflict-free)
  {
    const uint32_t mq = lane & 3;
    const size_t stride = (size_t)64 * 8;            // 64 rows p
    const uint32_t p_first = warp * 8 + (lane >> 2);
    const size_t g = cidx(y, p_first, m0 + 4 * mq, 512, nbp);
    const uint4* g0 = reinterpret_cast<const uint4*>(c0 + g);
    const uint4* g1 = reinterpret_cast<const uint4*>(c1 + g);
#pragma unroll 4
    for (uint32_t it = 0; it < 8; ++it) {
      const uint32_t o = 4 * mq * kInv512Ld + pad16(p_first + 64 * it);
      const uint4 v0 = __ldg(g0 + it * (stride / 4)), v1 = __ldg(g1 + it * (stride / 4));
      xs0[o] = v0.x; xs0[o + kInv512Ld] = v0.y; xs0[o + 2 * kInv512Ld] = v0.z; xs0[o + 3 * kInv512Ld] = v0.w;
      xs1[o] = v1.x; xs1[o + kInv512Ld] = v1.y; xs1[o + 2 * kInv512Ld] = v1.z; xs1[o + 3 * kInv512Ld] = v1.w;
    }
  }
  __syncthreads();
  const uint32_t q0 = cst.q[0], q1 = cst.q[1];
  for (uint32_t m = warp; m < kInv512Cols; m += 8) {
    const Inv512Limb L[2] = {{xs0 + m * kInv512Ld, cst.r2[0], q0}, {xs1 + m * kInv512Ld, cst.r2[1], q1}};
    uint32_t x[2][8];
    inv512_pair(L, cst, lane, x);
    const uint32_t u0 = (lane & 15) + 128 * (lane >> 4);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (cst.out1) {  // level-1 mode: both limbs, no rescale
        xs0[m * kInv512Ld + u0 + 16 * e] = x[0][e];
        xs1[m * kInv512Ld + u0 + 16 * e] = x[1][e];
        continue;
      }
      uint32_t t;
      if (x[1][e] > (q1 >> 1)) t = csub(x[0][e] + (q1 - x[1][e]), q0);
      else t = sub_mod(x[0][e], x[1][e], q0);
      xs1[m * kInv512Ld + u0 + 16 * e] = shoup_mul(t, cst.q1inv, cst.q1invp, q0);  // u = lo + 16 (e + 8 hi)
    }
  }
  __syncthreads();
  // phase C: a'[y][d j + m0 + m] = res[m][u = 255 - j]: 64-byte row segments
  const uint32_t N = d * 256;
  const size_t off = (size_t)(y - row0) * N + m0;
  const uint32_t* res = cst.out1 ? xs0 : xs1;
  for (uint32_t i = threadIdx.x; i < 256 * kInv512Cols; i += 256) {
    const uint32_t m = i & 15, j = i >> 4;
    out_a[off + (size_t)d * j + m] = res[m * kInv512Ld + 255 - j];
    if (cst.out1) cst.out1[off + (size_t)d * j + m] = xs1[m * kInv512Ld + 255 - j];
  }
}


// Fast S4 for L = 1024 (k = 256, blocks of ob = 768 outputs = 3 MLWE positions m): one warp per block,
// limbs in sequence, 32 register-resident elements per lane.
//   round 1: lane l holds positions 32 l + e: DIT stages len = 1 .. 16 in registers (lane-uniform twiddles);
//   round 2: lane l holds l + 32 e: stages len = 32 .. 512 in registers (per-stage lane tables); the last
//            stage forms only the outputs u < 768.
// 8 blocks per CTA, both limbs in smem (pitch 1148 = 4 mod 8, position p at pin36(p): conflict-free transposing
// stores, 16-byte round-1 loads/stores); a' rows of 3 x 8 positions are written as 96-byte segments.
HE_D void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
HE_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
HE_D void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
constexpr int kInv1kBlocks = 8;
constexpr uint32_t kLlamaQ0 = 1073479681u, kLlamaQ1 = 1179649u;   // HeParams.llama() (S4 specialisation)
constexpr uint64_t cx_powmod(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1;
  for (a %= q; e; e >>= 1, a = a * a % q)
    if (e & 1) r = r * a % q;
  return r;
}
constexpr int kInv1kLd = 1148;   // pin36(1023) + 1, = 4 mod 8
// position p at p + 4 (p / 32): rows of 32 positions at pitch 36 words, so a lane's 32 round-1 positions are
// 16-byte aligned (8 x LDS/STS.128, conflict-free per quarter-warp) and the round-2 reads p = l + 32 e hit 32 banks
HE_D uint32_t pin36(uint32_t p) { return p + 4 * (p >> 5); }
HE_D void ld_row32(const uint32_t* c, uint32_t (&x)[32]) {
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const uint4 w = reinterpret_cast<const uint4*>(c)[v];
    x[4 * v] = w.x, x[4 * v + 1] = w.y, x[4 * v + 2] = w.z, x[4 * v + 3] = w.w;
  }
}
HE_D void st_row32(uint32_t* c, const uint32_t (&x)[32]) {
#pragma unroll
  for (int v = 0; v < 8; ++v) reinterpret_cast<uint4*>(c)[v] = make_uint4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
}
// -> x[l][e] = INTT value u = lane + 32 e of limb l for e < 24, reduced to [0, q); both limbs in lockstep
struct Inv1kLimb {
  uint32_t* col;
  const uint2* r2;
  uint32_t q;
};
// Lazy q1 limb (LAZY1, when 42 q1 < 2^32 -- the 21-bit q1): no correction of x in its butterflies (values grow
// by at most 2 q per twiddled stage and double per twiddle-1 stage: < 42 q after the 10 stages), one Barrett
// reduction at the end.  Outputs: limb 0 in [0, 2 q0), limb 1 in [0, q1).
HE_D void bfl(uint32_t& x, uint32_t& y, uint2 w, uint32_t q2, uint32_t q) {  // DIT, x not corrected
  const uint32_t t = y * w.x - __umulhi(y, w.y) * q;
  const uint32_t a = x;
  x = a + t;
  y = a + q2 - t;
}
template <bool LAZY1, uint32_t KQ0 = 0, uint32_t KQ1 = 0>
HE_D void inv1024_pair(const Inv1kLimb (&L_)[2], const SpecInvConst& cst, uint32_t lane, uint32_t (&x)[2][32]) {
  // KQ0 / KQ1 != 0: the moduli as compile-time constants (immediate operands of the q products)
  const Inv1kLimb L[2] = {{L_[0].col, L_[0].r2, KQ0 ? KQ0 : L_[0].q}, {L_[1].col, L_[1].r2, KQ1 ? KQ1 : L_[1].q}};
#pragma unroll
  for (int l = 0; l < 2; ++l) ld_row32(L[l].col + 36 * lane, x[l]);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int len = 1 << s;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      if (e & len) continue;
      const int off = e & (len - 1);
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const bool lazy = LAZY1 && l == 1;
        if (off == 0) {
          if (lazy) {  // inputs < 2^s q: K = 2^s q keeps x + K - y >= 0
            const uint32_t u = x[l][e], v = x[l][e + len];
            x[l][e] = u + v;
            x[l][e + len] = u + (L[l].q << s) - v;
          } else if (s == 0 || (s == 1 && (e & 1) == 0)) {
            // no corrections needed: S3 stores C^ reduced to [0, q), and the even positions after the first stage
            // hold x + y < 2 q (only the odd ones, x - y + 2 q, reach 3 q)
            const uint32_t u = x[l][e], v = x[l][e + len];
            x[l][e] = u + v;
            x[l][e + len] = u + 2 * L[l].q - v;
          } else {
            dit_bf1(x[l][e], x[l][e + len], 2 * L[l].q);
          }
        } else {
          const uint2 w = cst.r1[l][(1 << s) - s - 1 + off - 1];
          if (lazy) bfl(x[l][e], x[l][e + len], w, 2 * L[l].q, L[l].q);
          else dit_bf(x[l][e], x[l][e + len], w, 2 * L[l].q, L[l].q);
        }
      }
    }
  }
#pragma unroll
  for (int l = 0; l < 2; ++l) st_row32(L[l].col + 36 * lane, x[l]);
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int e = 0; e < 32; ++e) x[l][e] = L[l].col[lane + 36 * e];
  __syncwarp();
#pragma unroll
  for (int s = 5; s < 9; ++s) {
    const int len = 1 << (s - 5);
    const int base = 32 * (len - 1);
    // this stage's len twiddles of the lane, entries (2 i, 2 i + 1) as one 16-byte load (spec_table_init layout)
    uint2 tw[2][8];
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      if (len == 1) {
        tw[l][0] = L[l].r2[lane];
      } else {
#pragma unroll
        for (int i = 0; i < len / 2; ++i) {
          const uint4 v = *reinterpret_cast<const uint4*>(L[l].r2 + base + 64 * i + 2 * lane);
          tw[l][2 * i] = make_uint2(v.x, v.y);
          tw[l][2 * i + 1] = make_uint2(v.z, v.w);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      if (e & len) continue;
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const uint2 w = tw[l][e & (len - 1)];
        if (LAZY1 && l == 1) bfl(x[l][e], x[l][e + len], w, 2 * L[l].q, L[l].q);
        else dit_bf(x[l][e], x[l][e + len], w, 2 * L[l].q, L[l].q);
      }
    }
  }
  // len = 512: pairs (e, e + 16); the upper output u = lane + 32 e + 512 is needed only for e < 8
#pragma unroll
  for (int e = 0; e < 16; ++e) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const bool lazy = LAZY1 && l == 1;
      const uint32_t q = L[l].q, q2 = 2 * q;
      const uint4 wv = *reinterpret_cast<const uint4*>(L[l].r2 + 480 + 64 * (e >> 1) + 2 * lane);
      const uint2 w = (e & 1) ? make_uint2(wv.z, wv.w) : make_uint2(wv.x, wv.y);
      if (e < 8) {
        if (lazy) bfl(x[l][e], x[l][e + 16], w, q2, q);
        else dit_bf(x[l][e], x[l][e + 16], w, q2, q);
      } else {
        const uint32_t t = x[l][e + 16] * w.x - __umulhi(x[l][e + 16], w.y) * q;
        x[l][e] = (lazy ? x[l][e] : min(x[l][e], x[l][e] - q2)) + t;
      }
    }
  }
  // limb 1 leaves as r = (x1 + h) mod q1, h = (q1 - 1) / 2: r - h is the centred representative the rescale needs
  const uint32_t q1 = L[1].q, h = q1 >> 1;
  const uint32_t q1bar = KQ1 ? (uint32_t)(0x100000000ull / KQ1) : cst.q1bar;
#pragma unroll
  for (int e = 0; e < 24; ++e) {
    x[0][e] = min(x[0][e], x[0][e] - 2 * L[0].q);   // [0, 2 q0)
    uint32_t v = x[1][e] + h;
    if (LAZY1) {
      v -= __umulhi(v, q1bar) * q1;                   // v < 43 q1 < 2^32: quotient off by at most one -> [0, 2 q1)
    } else {
      v = min(v, v - 2 * q1);
      v = min(v, v - 2 * q1);                         // x1 < 4 q1: [0, 2 q1)
    }
    x[1][e] = min(v, v - q1);                         // [0, q1)
  }
}

template <bool LAZY1, uint32_t KQ0 = 0, uint32_t KQ1 = 0>
__global__ void __launch_bounds__(256, 2) spec_inverse1024_kernel(const uint32_t* __restrict__ c0,
                                                                  const uint32_t* __restrict__ c1, uint32_t n_out,
                                                                  uint32_t row0, uint32_t nbp, uint32_t nblk,
                                                                  uint32_t d, SpecInvConst cst,
                                                                  uint32_t* __restrict__ out_a, OutPeers peers) {
  extern __shared__ uint32_t sm[];
  uint32_t* xs0 = sm;                                  // [8 blocks][1060]
  uint32_t* xs1 = sm + kInv1kBlocks * kInv1kLd;
  uint2* tws = reinterpret_cast<uint2*>(xs1 + kInv1kBlocks * kInv1kLd);   // round-2 lane tables [2][992]
  const uint32_t y = row0 + blockIdx.y, b0 = blockIdx.x * kInv1kBlocks;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // phase A: C^[y][b0 / 8][p][0 .. 7] of both limbs -> xs[b][pin36(p)]; one warp access = 512 contiguous bytes.
  // The round-2 lane tables are copied with cp.async after the unit's loads are issued (no register staging,
  // no wait in front of the loads)
  {
    const uint32_t bq = lane & 1, ps = lane >> 1;
    const size_t g = cidx(y, warp * 16 + ps, b0 + 4 * bq, 1024, nbp);   // the unit is one contiguous 32 KB run
    const size_t stride = (size_t)128 * 8 / 4;   // 128 rows p, in uint4
    const uint4* g0 = reinterpret_cast<const uint4*>(c0 + g);
    const uint4* g1 = reinterpret_cast<const uint4*>(c1 + g);
    uint4 v0[8], v1[8];   // all 16 loads in flight before the first store
#pragma unroll
    for (uint32_t it = 0; it < 8; ++it) {
      v0[it] = __ldg(g0 + it * stride);
      v1[it] = __ldg(g1 + it * stride);
    }
    for (uint32_t i = threadIdx.x; i < 496; i += 256) {   // 992 uint2 = 496 uint4 per limb
      cp_async16(reinterpret_cast<uint4*>(tws) + i, reinterpret_cast<const uint4*>(cst.r2[0]) + i);
      cp_async16(reinterpret_cast<uint4*>(tws + 992) + i, reinterpret_cast<const uint4*>(cst.r2[1]) + i);
    }
    cp_async_commit();
#pragma unroll
    for (uint32_t it = 0; it < 8; ++it) {
      const uint32_t o = 4 * bq * kInv1kLd + pin36(warp * 16 + ps + 128 * it);
      xs0[o] = v0[it].x; xs0[o + kInv1kLd] = v0[it].y; xs0[o + 2 * kInv1kLd] = v0[it].z; xs0[o + 3 * kInv1kLd] = v0[it].w;
      xs1[o] = v1[it].x; xs1[o + kInv1kLd] = v1[it].y; xs1[o + 2 * kInv1kLd] = v1[it].z; xs1[o + 3 * kInv1kLd] = v1[it].w;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const uint32_t b = warp;
  if (b0 + b < nblk) {
    const uint32_t q0 = KQ0 ? KQ0 : cst.q[0], q1 = KQ1 ? KQ1 : cst.q[1];
    const Inv1kLimb L[2] = {{xs0 + b * kInv1kLd, tws, q0}, {xs1 + b * kInv1kLd, tws + 992, q1}};
    uint32_t x[2][32];
    inv1024_pair<LAZY1, KQ0, KQ1>(L, cst, lane, x);
    const uint32_t h = q1 >> 1;
    if (cst.out1) {  // level-1 mode: both limbs, no rescale
#pragma unroll
      for (int e = 0; e < 24; ++e) {
        xs0[b * kInv1kLd + lane + 32 * e + (e >> 3)] = min(x[0][e], x[0][e] - q0);
        const uint32_t r = x[1][e];   // (x1 + h) mod q1
        xs1[b * kInv1kLd + lane + 32 * e + (e >> 3)] = min(r - h, r + q1 - h);
      }
    } else
#pragma unroll
    for (int e = 0; e < 24; ++e) {
      // (x0 - [x1]_centred) q1^-1 mod q0 with [x1]_centred = r - h: t = x0 + (q0 + h) - r in (0, 3 q0 + h),
      // one Shoup product (any 32-bit input) -> [0, 2 q0), one correction
      constexpr uint32_t kInv = KQ0 ? (uint32_t)cx_powmod(KQ1, KQ0 - 2, KQ0) : 0u;
      const uint32_t qi = KQ0 ? kInv : cst.q1inv;
      const uint32_t qip = KQ0 ? (uint32_t)(((uint64_t)kInv << 32) / KQ0) : cst.q1invp;
      const uint32_t t = x[0][e] + (q0 + h) - x[1][e];
      const uint32_t v = t * qi - __umulhi(t, qip) * q0;
      // u = lane + 32 e stored at u + u / 256 (the three thirds of a block one bank apart for phase C)
      xs1[b * kInv1kLd + lane + 32 * e + (e >> 3)] = min(v, v - q0);
    }
  }
  __syncthreads();
  // phase C: block b covers c' = 768 (b0 + b) + u  <->  m = 3 (b0 + b) + u / 256, j = 255 - u % 256
  // lane ml < 24 owns position m = 3 b0 + ml (block ml / 3, third ml % 3); the 8 warps stride over j
  const uint32_t N = d * 256, m = 3 * b0 + lane;
  if (lane < 24 && m < d) {
    const uint32_t bl = lane / 3, r3 = lane - 3 * bl, src = bl * kInv1kLd + 257 * r3 + 255;
    if (cst.out1) {
      const size_t o = (size_t)(y - row0) * N + m;
      for (uint32_t j = warp; j < 256; j += 8) {
        out_a[o + (size_t)d * j] = xs0[src - j];
        cst.out1[o + (size_t)d * j] = xs1[src - j];
      }
    } else if (peers.n == 0) {
      uint32_t* dst = out_a + (size_t)(y - row0) * N + m;
#pragma unroll 4
      for (uint32_t j = warp; j < 256; j += 8) dst[(size_t)d * j] = xs1[src - j];
    } else {  // fused all-gather: the same words into every rank's full output at row dst_row0 + (y - row0)
      const size_t yd = (size_t)peers.dst_row0 + (y - row0);
      for (uint32_t j = warp; j < 256; j += 8) {
        const uint32_t v = xs1[src - j];
        for (int pr = 0; pr < peers.n; ++pr) peers.a[pr][yd * N + (size_t)d * j + m] = v;
      }
    }
  }
}

// ---------------------------------------------------------------- S3: per-frequency modular GEMM (tcgen05)
constexpr int kSpecBN = 32;   // blocks m per tile
constexpr int kSpecBK = 64;   // K bytes per stage
constexpr int kSpecEpiWarps = 16;
constexpr int kSpecEpiCols = kSpecBN / (kSpecEpiWarps / 4);  // columns per epilogue thread
constexpr int kSpecThreads = 64 + 32 * kSpecEpiWarps;

HE_D void named_bar_sync(uint32_t id, uint32_t n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
HE_D void tma_store_3d(const void* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
HE_D void tma_store_4d_hint(const void* map, const void* src, int x, int y, int z, int w, uint64_t hint) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;"
               ::"l"(map), "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z), "r"(w), "l"(hint)
               : "memory");
}

HE_D void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
HE_D void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
HE_D void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// UMMA smem descriptor, K-major, 64-byte swizzle: rows of 64 B, 8-row atoms (SBO = 512 B)
HE_D uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(512u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;  // SWIZZLE_64B
  return d;
}

template <int D>
struct SpecCfg {
  static constexpr int S = 2 * D - 1;
  static constexpr int kChunk = kSpecBN / 2;                // B rows per TMA box (half a plane)
  static constexpr int kABytes = D * 128 * kSpecBK;         // per CTA per stage
  static constexpr int kBBytes = D * kChunk * kSpecBK;      // per CTA per stage
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOutBytes = 128 * kSpecBN * 4;       // one staged C^ tile (128 rows x 32 u32)
  static constexpr int kStages = (176 * 1024) / kStageBytes > 8 ? 8 : (176 * 1024) / kStageBytes;
  static constexpr int kZeroBytes = 8192;
  static constexpr int kSmemBytes = kStages * kStageBytes + 2 * kOutBytes + kZeroBytes + 1024 + 256;
  static constexpr int kBuf = 256;                          // TMEM column stride of the two buffers
  static_assert(S * kSpecBN <= kBuf, "shift accumulators exceed one TMEM buffer");
  static_assert(kStages >= 2, "not enough shared memory");
};

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kSpecThreads, 1)
    spec_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const SpecGemmArgs args) {
  using C = SpecCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint8_t* sOut = sB + C::kStages * C::kBBytes;       // [2][128 rows][128 B], 128-B swizzled (TMA store)
  uint8_t* sZero = sOut + 2 * C::kOutBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sZero + C::kZeroBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int m_tiles = args.nb / kSpecBN;
  const int y_tiles = (args.n_rows + 255) / 256;
  const int num_tiles = m_tiles * y_tiles * args.L;
  const int num_kb = args.r_pad / kSpecBK;
  // G^ bytes of K block kb (kg <= r_pad; the last block may be partial)
  auto kg_kb = [&](int kb) { const int r = args.kg - kb * kSpecBK; return r < kSpecBK ? (r > 0 ? r : 0) : kSpecBK; };

  for (int i = threadIdx.x; i < C::kZeroBytes / 16; i += kSpecThreads)
    reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 2 * kSpecEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc_2sm(tmem_slot, 512);
    tmem_relinquish_2sm();
  }
  fence_proxy_async();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // tile -> (y tile, f / 4, m tile, f % 4): each CTA pair takes runs of 4 consecutive tiles (4 consecutive
  // frequencies of one (y tile, m tile)), so an epilogue warp writes the 4 x 32-byte pieces of each row's
  // C^ group run ([y][group][f][8]) back to back -- full 128-byte lines -- while the pairs working at one time
  // still cover the 3 m tiles of a run of frequencies of the same 256 rows (G^_f read once from DRAM);
  // divisions by 32-bit reciprocals (exact for operands < 2^16)
  const uint32_t m_magic = (uint32_t)((0xFFFFFFFFull + m_tiles) / m_tiles);
  const uint32_t lg_l4 = 29 - __clz(args.L);   // log2(L / 4), L a power of two >= 4
  auto pair_tile = [&](int it) { return ((pair + (it >> 2) * npairs) << 2) + (it & 3); };
  auto tile_coords = [&](int tile, int& f, int& y0, int& m0) {
    const uint32_t rest = (uint32_t)tile >> 2;
    const uint32_t r2 = m_tiles == 1 ? rest : __umulhi(rest, m_magic);
    m0 = (int)(rest - r2 * (uint32_t)m_tiles) * kSpecBN;
    f = (int)(((r2 & ((uint32_t)(args.L >> 2) - 1)) << 2) | ((uint32_t)tile & 3));
    y0 = args.row0 + (int)(r2 >> lg_l4) * 256;
  };

  if (warp == 0) {
    // ======================= TMA producer (both CTAs) =======================
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0_remote = mapa_rank(&full[0], 0);
      for (int it = 0, tile; (tile = pair_tile(it)) < num_tiles; ++it) {
        int f, y0, m0;
        tile_coords(tile, f, y0, m0);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], 2 * (uint32_t)(D * 128 * kg_kb(kb) + C::kBBytes));
          else mbar_arrive_cluster(full0_remote + stage * 8);
          uint8_t* a_dst = sA + stage * C::kABytes;
          uint8_t* b_dst = sB + stage * C::kBBytes;
          // A: this CTA's 128-row tile of each digit plane, kg_kb(kb) / 16 chunks of 2 KB stored contiguously
          // (gidx): one box of kg_kb / 2 lines of 256 bytes
#pragma unroll
          for (int a = 0; a < D; ++a)
            tma_load_3d_2sm(a_dst + a * 128 * kSpecBK, &tmA, &full[stage], 0, kb * (kSpecBK / 2),
                            (f * D + a) * ((args.n_out + 127) / 128) + (y0 + (int)rank * 128) / 128, args.hint_g);
          // stacked operand [P0 | P1 | .. | P(D-1)] x 32 rows: this CTA holds chunks [rank*D, rank*D + D)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const int g = (int)rank * D + c;
            tma_load_3d_2sm(b_dst + c * C::kChunk * kSpecBK, &tmB, &full[stage], kb * kSpecBK,
                            m0 + (g & 1) * C::kChunk, f * D + (g >> 1), args.hint_a);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA) =======================
    if (leader) {
      constexpr uint32_t kIdesc = idesc_i8(256, D * kSpecBN);
      constexpr uint32_t kIdescZ = idesc_i8(256, C::S * kSpecBN);
      const uint64_t zdesc = desc_noswz(smem_u32(sZero), 128, 256);
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int tile; (tile = pair_tile(iter)) < num_tiles; ++iter) {
        const int buf = iter & 1;
        const uint32_t acc = tmem_base + buf * C::kBuf;
        if (iter >= 2) mbar_wait(&tmem_empty[buf], ((iter >> 1) - 1) & 1);
        tc_fence_after();
        if (elect_one()) mma_i8_2sm(acc, zdesc, zdesc, kIdescZ, 0);
        __syncwarp();
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_base = smem_u32(sA + stage * C::kABytes);
            const uint32_t b_base = smem_u32(sB + stage * C::kBBytes);
            // K steps of 32 bytes = A chunks (2 kk, 2 kk + 1): LBO 2 KB between K chunks, SBO 128 B between
            // 8-row groups. A chunk past kg is stale smem (the next digit's / stage's bytes) whose products meet
            // A^'s zero padding (rows r >= R are zero), so it adds nothing; K steps wholly past kg are skipped.
            for (int kk = 0; kk < (kg_kb(kb) + 31) / 32; ++kk) {
              const uint64_t bd = desc_sw64(b_base + kk * 32);
#pragma unroll
              for (int a = 0; a < D; ++a)
                mma_i8_2sm(acc + a * kSpecBN, desc_noswz(a_base + a * 128 * kSpecBK + kk * 4096, 2048, 128), bd,
                           kIdesc, 1);
            }
            tc_commit_2sm_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) tc_commit_2sm_mc(&tmem_full[buf], 0x3);
        __syncwarp();
      }
    }
  } else {
    // ======================= epilogue (both CTAs, 16 warps) =======================
    const uint32_t ew = warp - 2;
    const uint32_t quarter = warp & 3;
    const uint32_t part = ew / 4;                      // columns [kSpecEpiCols part, .. + kSpecEpiCols)
    const uint32_t lane_addr = (quarter * 32) << 16;
    const uint32_t tmem_empty_remote = mapa_rank(&tmem_empty[0], 0);
    const uint32_t q = args.q;
    int iter = 0;
    for (int tile; (tile = pair_tile(iter)) < num_tiles; ++iter) {
      const int buf = iter & 1;
      int f, y0, m0;
      tile_coords(tile, f, y0, m0);
      mbar_wait(&tmem_full[buf], (iter >> 1) & 1);
      tc_fence_after();
      const int y = y0 + (int)rank * 128 + (int)(quarter * 32 + lane);
      uint32_t acc[C::S][kSpecEpiCols];
      const uint32_t col = tmem_base + lane_addr + buf * C::kBuf + part * kSpecEpiCols;
#pragma unroll
      for (int s = 0; s < C::S; ++s)
#pragma unroll
        for (int c8 = 0; c8 < kSpecEpiCols / 8; ++c8) tmem_ld_x8(col + s * kSpecBN + 8 * c8, acc[s] + 8 * c8);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tmem_empty_remote + buf * 8);  // accumulators drained
      // sum_s acc_s 2^(8 s) mod q: shifts paired exactly in int32 (t_i = acc_2i + 256 acc_2i+1, plan-time
      // bound |t_i| < 2^31), v = off + sum_i t_i (2^(16 i + 32) mod q) in int64 (off: a multiple of q above
      // |sum|), one Montgomery reduction (v + ((v mod 2^32)(-q^-1) mod 2^32) q) / 2^32 in [0, 3q), two csubs
      uint32_t res[kSpecEpiCols];
      constexpr int T = (C::S + 1) / 2;
#pragma unroll
      for (int e = 0; e < kSpecEpiCols; ++e) {
        int64_t v = (int64_t)args.off64;
#pragma unroll
        for (int i = 0; i < T; ++i) {
          const int32_t lo = (int32_t)acc[2 * i][e];
          const int32_t t = (2 * i + 1 < C::S) ? lo + ((int32_t)acc[2 * i + 1][e] << 8) : lo;
          v += (int64_t)t * (int64_t)args.pw[i];
        }
        const uint32_t m = (uint32_t)v * args.qninv;
        uint32_t t = (uint32_t)(((uint64_t)v + (uint64_t)m * q) >> 32);   // [0, 3q)
        t = min(t, t - 2 * q);
        res[e] = min(t, t - q);
      }
      // each warp stages its 32 rows x 8 words (1 KB, double-buffered) and TMA-stores them itself: no
      // cross-warp barrier; the buffer of tile iter-2 must have been read out by its bulk store first
      uint8_t* so = sOut + buf * C::kOutBytes + ew * (32 * kSpecEpiCols * 4);
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
#pragma unroll
      for (int c = 0; c < kSpecEpiCols / 4; ++c)
        *reinterpret_cast<uint4*>(so + lane * (kSpecEpiCols * 4) + c * 16) =
            make_uint4(res[4 * c], res[4 * c + 1], res[4 * c + 2], res[4 * c + 3]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_4d_hint(&tmC, so, 0, f, (m0 + (int)part * kSpecEpiCols) >> 3, y0 + (int)rank * 128 + (int)quarter * 32,
                          args.hint_c);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait_all();
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
}

// debug/reference form of S3 on CUDA cores (HE_SPEC_SIMPLE=1): same digit operands, exact int64 sums
__global__ void spec_gemm_simple_kernel(const int8_t* __restrict__ G, const int8_t* __restrict__ A, SpecGemmArgs args,
                                        int D) {
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t yy = blockIdx.y, f = blockIdx.z;
  if (m >= (uint32_t)args.nb) return;
  const uint32_t y = args.row0 + yy;
  const uint32_t q = args.q;
  uint64_t accq = 0;
  for (int r = 0; r < args.r_pad; ++r) {
    int64_t gv = 0, av = 0;
    for (int a = D - 1; a >= 0; --a) {
      gv = gv * 256 + (r < args.kg ? G[gidx(f * D + a, y, r, args.n_out, args.kg)] : 0);
      av = av * 256 + A[(((size_t)f * D + a) * args.nb + m) * args.r_pad + r];
    }
    int64_t gm = gv % (int64_t)q, am = av % (int64_t)q;
    if (gm < 0) gm += q;
    if (am < 0) am += q;
    accq = (accq + (uint64_t)gm * (uint64_t)am) % q;
  }
  args.out[cidx(y, f, m, args.L, args.nb)] = (uint32_t)accq;
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_spec_weights(const int8_t* wdig, uint32_t d_w, uint32_t n_out, uint32_t n_in, uint32_t k,
                                const SpecTable& t, int D, uint32_t r_pad, int8_t* out, cudaStream_t s) {
  const uint32_t R = n_in / k;
  dim3 grid(n_out, (R + kSpecRChunk - 1) / kSpecRChunk);
  const size_t smem = (size_t)kSpecRChunk * t.L * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(spec_weights_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  spec_weights_kernel<<<grid, 256, smem, s>>>(wdig, d_w, n_out, n_in, k, t.L, t.q, D, r_pad, t.fw, t.linv, t.linvp,
                                              out);
  return cudaGetLastError();
}

cudaError_t launch_spec_data(const RingDims& Rg, const uint32_t* ct, uint32_t n_ct, uint32_t limb, const SpecTable& t,
                             int D, uint32_t r_pad, uint32_t ob, uint32_t nblk, uint32_t nbp, int8_t* out,
                             cudaStream_t s) {
  if (t.L == 1024 && t.f2) {
    dim3 grid(nblk, (n_ct + 15) / 16, 1);
    const size_t smem = (size_t)16 * kS2Ld * sizeof(uint32_t);
    cudaError_t e = cudaFuncSetAttribute(spec_data1024_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    SpecData2 sd{};
    sd.cf[0].f2 = t.f2;
    for (int i = 0; i < 26; ++i) sd.cf[0].f1[i] = t.f1[i];
    sd.q[0] = t.q;
    sd.D[0] = D;
    // one limb per call: the kernel reads limb blockIdx.z of the ciphertexts, so shift the base to this limb
    sd.out[0] = out;
    spec_data1024_kernel<<<grid, 512, smem, s>>>(ct + (size_t)limb * 2 * Rg.N, n_ct, Rg.k, ob, nbp, Rg.N, r_pad, sd);
    return cudaGetLastError();
  }
  dim3 grid(nblk, (n_ct + kSpecRChunk - 1) / kSpecRChunk);
  const size_t smem = (size_t)kSpecRChunk * t.L * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(spec_data_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  spec_data_kernel<<<grid, 256, smem, s>>>(ct, n_ct, limb, Rg.k, ob, nbp, Rg.N, t.L, t.q, D, r_pad, t.fw, out);
  return cudaGetLastError();
}

cudaError_t launch_spec_data2(const RingDims& Rg, const uint32_t* ct, uint32_t n_ct, const SpecTable (&t)[2],
                              const int (&D)[2], uint32_t r_pad, uint32_t ob, uint32_t nblk, uint32_t nbp,
                              int8_t* const (&out)[2], cudaStream_t s) {
  if (t[0].L != 1024 || !t[0].f2 || !t[1].f2) {
    for (uint32_t L = 0; L < 2; ++L) {
      cudaError_t e = launch_spec_data(Rg, ct, n_ct, L, t[L], D[L], r_pad, ob, nblk, nbp, out[L], s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  dim3 grid(nblk, (n_ct + 15) / 16, 2);
  const size_t smem = (size_t)16 * kS2Ld * sizeof(uint32_t);
  cudaError_t e = cudaFuncSetAttribute(spec_data1024_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  SpecData2 sd{};
  for (int L = 0; L < 2; ++L) {
    sd.cf[L].f2 = t[L].f2;
    for (int i = 0; i < 26; ++i) sd.cf[L].f1[i] = t[L].f1[i];
    sd.q[L] = t[L].q;
    sd.D[L] = D[L];
    sd.out[L] = out[L];
  }
  spec_data1024_kernel<<<grid, 512, smem, s>>>(ct, n_ct, Rg.k, ob, nbp, Rg.N, r_pad, sd);
  return cudaGetLastError();
}

cudaError_t launch_spec_inverse(const RingDims& Rg, const uint32_t* c0, const uint32_t* c1, uint32_t n_out,
                                uint32_t row0, uint32_t rows, uint32_t L, uint32_t nblk, uint32_t nbp,
                                const SpecInvConst& cst, uint32_t* out_a, const OutPeers& peers, cudaStream_t s) {
  if (peers.n > 0 && L != 1024) return cudaErrorNotSupported;  // fused output only on the L = 1024 fast path
  if (peers.n > 0 && cst.out1) return cudaErrorNotSupported;
  if (L == 1024) {
    if (Rg.k != 256) return cudaErrorInvalidValue;
    const size_t smem = (size_t)2 * kInv1kBlocks * kInv1kLd * sizeof(uint32_t) + 2 * 992 * sizeof(uint2);
    SpecInvConst c2 = cst;
    c2.q1bar = (uint32_t)(0x100000000ull / cst.q[1]);
    static const bool strict = getenv("HE_S4_STRICT") != nullptr;  // A/B switch: corrected q1 butterflies
    const bool lazy = !strict && 42ull * cst.q[1] < 0x100000000ull;
    static const bool kq_off = getenv("HE_S4_RUNTIME_Q") != nullptr;  // A/B switch: moduli as kernel parameters
    auto kern = lazy ? spec_inverse1024_kernel<true> : spec_inverse1024_kernel<false>;
    if (lazy && !kq_off && cst.q[0] == kLlamaQ0 && cst.q[1] == kLlamaQ1)
      kern = spec_inverse1024_kernel<true, kLlamaQ0, kLlamaQ1>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((nblk + kInv1kBlocks - 1) / kInv1kBlocks, rows);
    kern<<<grid, 256, smem, s>>>(c0, c1, n_out, row0, nbp, nblk, Rg.d, c2, out_a, peers);
    return cudaGetLastError();
  }
  static const bool generic = getenv("HE_SPEC_INV_GENERIC") != nullptr;  // debug: the simple S4
  if (L == 512 && Rg.k == 256 && Rg.d % kInv512Cols == 0 && !generic) {
    dim3 grid(Rg.d / kInv512Cols, rows);
    const size_t smem = (size_t)2 * kInv512Cols * kInv512Ld * sizeof(uint32_t);
    cudaError_t e = cudaFuncSetAttribute(spec_inverse512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    spec_inverse512_kernel<<<grid, 256, smem, s>>>(c0, c1, nbp, row0, Rg.d, cst, out_a);
    return cudaGetLastError();
  }
  if (Rg.d % kSpecMGroup) return cudaErrorInvalidValue;
  dim3 grid(Rg.d / kSpecMGroup, rows);
  const size_t smem = ((size_t)kSpecMGroup * (L + 1) + (size_t)kSpecMGroup * (Rg.k + 1)) * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(spec_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  spec_inverse_kernel<<<grid, 256, smem, s>>>(c0, c1, nbp, row0, Rg.d, Rg.k, L, cst, out_a);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_spec_gemm_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                      const SpecGemmArgs& a, int grid, cudaStream_t s) {
  using C = SpecCfg<D>;
  auto kern = spec_gemm_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kSpecThreads, C::kSmemBytes, s>>>(tmA, tmB, tmC, a);
  return cudaGetLastError();
}

cudaError_t launch_spec_gemm(int D, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                             const SpecGemmArgs& a, int sm_count, cudaStream_t s) {
  const int tiles = (a.nb / kSpecBN) * ((a.n_rows + 255) / 256) * a.L;
  const int pairs = sm_count / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);
  switch (D) {
    case 1: return launch_spec_gemm_t<1>(tmA, tmB, tmC, a, grid, s);
    case 2: return launch_spec_gemm_t<2>(tmA, tmB, tmC, a, grid, s);
    case 3: return launch_spec_gemm_t<3>(tmA, tmB, tmC, a, grid, s);
    case 4: return launch_spec_gemm_t<4>(tmA, tmB, tmC, a, grid, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_spec_gemm_simple(int D, const int8_t* G, const int8_t* A, const SpecGemmArgs& a, cudaStream_t s) {
  dim3 grid((a.nb + 127) / 128, a.n_rows, a.L);
  spec_gemm_simple_kernel<<<grid, 128, 0, s>>>(G, A, a, D);
  return cudaGetLastError();
}

}  // namespace he
