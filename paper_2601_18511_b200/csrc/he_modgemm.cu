// he_modgemm.cu -- K1: the per-RNS-limb modular GEMM of the MLWE PCMM on tcgen05 int8 tensor cores.
//
//   v_i[y][n] = sum_x W~[y][x] * C_i[x][n]  mod q_i      (i = 0, 1;  SURVEY.md App. B.3)
//   out[y][n] = rescale(v_0, v_1) = ((v_0 - [v_1]_centred) * q_1^-1) mod q_0
//
// W~ (integer, |W~| < 2^31) is split into D_W balanced 8-bit digit planes, the centred
// ciphertext words C_i into D_i planes (he_decompose.cu).  One tile = 128 output rows x
// 32 GEMM columns x both limbs.  For weight digit a and limb i, ONE tcgen05.mma multiplies
// the A plane a against the D_i ciphertext planes stacked along N ([C_i,0 | C_i,1 | ...]),
// writing at TMEM column offset a*32: the product of digit pair (a, b) lands in the
// accumulator of shift s = a + b.  So each limb needs only D_W + D_i - 1 int32
// accumulators per output word (not D_W * D_i), and the MMA N is D_i * 32 (128 / 96).
// The epilogue reduces each shift accumulator mod q_i (Shoup), recombines sum_s 2^(8s),
// rescales the two limbs into one level-0 word, and stores b' already composed into RLWE
// order and a' in MLWE row-major order.  Nothing but the level-0
// result ever reaches HBM.
//
// Warp roles (192 threads, 1 CTA per SM, persistent over tiles, m-fastest raster so the
// 32 M-blocks sharing one ciphertext N-block run together and the B tile is L2-hot):
//   warp 0  TMA producer (A: weight digits, EVICT_LAST; B: ciphertext digits, EVICT_FIRST)
//   warp 1  TMEM allocator + single-thread MMA issuer
//   warps 2-5 epilogue (TMEM lane quarter = warp % 4)
#include <cuda.h>
#include "he_common.cuh"
#include "he_tc.cuh"
#include "he_kernels.h"

namespace he {

constexpr int kBM = 128;   // output rows per tile (TMEM lanes)
constexpr int kBN = 32;    // GEMM columns per tile
constexpr int kBK = 128;   // K bytes per pipeline stage (one 128-B swizzle row)
constexpr int kThreads = 192;

template <int DW, int D0, int D1>
struct GemmCfg {
  static constexpr int S0 = DW + D0 - 1;                 // shift accumulators, limb 0
  static constexpr int S1 = DW + D1 - 1;                 // shift accumulators, limb 1
  static constexpr int kTmemCols = (S0 + S1) * kBN;
  static constexpr int kTmemAlloc = kTmemCols <= 32 ? 32 : kTmemCols <= 64 ? 64 : kTmemCols <= 128 ? 128
                                  : kTmemCols <= 256 ? 256 : 512;
  static constexpr int kABytes = DW * kBM * kBK;         // per stage
  static constexpr int kBBytes = (D0 + D1) * kBN * kBK;  // per stage
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024) / kStageBytes > 6 ? 6 : (200 * 1024) / kStageBytes;
  static constexpr int kZeroBytes = 8192;                // zero operand for accumulator clearing
  static constexpr int kSmemBytes = kStages * kStageBytes + kZeroBytes + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(kTmemCols <= 512, "too many shift accumulators for TMEM");
  static_assert(kStages >= 2, "not enough shared memory for two stages");
  static_assert(S0 * kBN <= 256 && S1 * kBN <= 256, "zeroing MMA N out of range");
};

template <int DW, int D0, int D1>
__global__ void __launch_bounds__(kThreads, 1)
    modgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs args) {
  using C = GemmCfg<DW, D0, D1>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the 128-B swizzle atoms
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sA = smem;                                   // [stage][DW][128 rows][128 B]
  uint8_t* sB = smem + C::kStages * C::kABytes;         // [stage][D0+D1][32 rows][128 B]
  uint8_t* sZero = sB + C::kStages * C::kBBytes;        // 8 KB of zeros
  uint64_t* full = reinterpret_cast<uint64_t*>(sZero + C::kZeroBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int m_tiles = (args.n_out + kBM - 1) / kBM;
  const int n_tiles = args.width / kBN;
  const int num_tiles = m_tiles * n_tiles;
  const int num_kb = (args.n_in + kBK - 1) / kBK;

  for (int i = threadIdx.x; i < C::kZeroBytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 4 * 32);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, C::kTmemAlloc);
    tmem_relinquish();
  }
  fence_proxy_async();  // zero tile visible to the tensor-core (async) proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile % m_tiles) * kBM;
        const int n0 = (tile / m_tiles) * kBN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::kStageBytes);
          uint8_t* a_dst = sA + stage * C::kABytes;
          uint8_t* b_dst = sB + stage * C::kBBytes;
#pragma unroll
          for (int a = 0; a < DW; ++a)
            tma_load_3d(a_dst + a * kBM * kBK, &tmA, &full[stage], kb * kBK, m0, a, kEvictLast);
#pragma unroll
          for (int p = 0; p < D0 + D1; ++p)
            tma_load_3d(b_dst + p * kBN * kBK, &tmB, &full[stage], kb * kBK, n0, p, kEvictFirst);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    constexpr uint32_t kIdesc0 = idesc_i8(kBM, D0 * kBN);
    constexpr uint32_t kIdesc1 = idesc_i8(kBM, D1 * kBN);
    constexpr uint32_t kIdescZ0 = idesc_i8(kBM, C::S0 * kBN);
    constexpr uint32_t kIdescZ1 = idesc_i8(kBM, C::S1 * kBN);
    const uint32_t reg0 = tmem_base;                     // limb-0 shift accumulators
    const uint32_t reg1 = tmem_base + C::S0 * kBN;       // limb-1 shift accumulators
    const uint64_t zdesc = desc_noswz(smem_u32(sZero), 128, 256);
    int stage = 0;
    uint32_t phase = 0;
    int iter = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++iter) {
      if (iter > 0) mbar_wait(tmem_empty, (iter - 1) & 1);  // epilogue drained the accumulators
      tc_fence_after();
      if (elect_one()) {
        // clear all shift accumulators: D = 0 * B
        mma_i8(reg0, zdesc, zdesc, kIdescZ0, 0);
        mma_i8(reg1, zdesc, zdesc, kIdescZ1, 0);
      }
      __syncwarp();
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_base = smem_u32(sA + stage * C::kABytes);
          const uint32_t b_base = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
          for (int kk = 0; kk < kBK / 32; ++kk) {
            const uint64_t b0 = desc_sw128(b_base + kk * 32);
            const uint64_t b1 = desc_sw128(b_base + D0 * kBN * kBK + kk * 32);
#pragma unroll
            for (int a = 0; a < DW; ++a) {
              const uint64_t ad = desc_sw128(a_base + a * kBM * kBK + kk * 32);
              mma_i8(reg0 + a * kBN, ad, b0, kIdesc0, 1);
              mma_i8(reg1 + a * kBN, ad, b1, kIdesc1, 1);
            }
          }
          tc_commit(&empty[stage]);  // frees the smem slot when these MMAs retire
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) tc_commit(tmem_full);
      __syncwarp();
    }
  } else {
    // ======================= epilogue =======================
    const uint32_t quarter = warp & 3;                   // TMEM lanes this warp may access
    const uint32_t row_in_tile = quarter * 32 + lane;
    const uint32_t lane_addr = (quarter * 32) << 16;
    const int N = args.d * args.k;
    const int logk = ilog2_h(args.k);
    (void)logk;
    const GemmEpiConst& c = args.c;
    int iter = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++iter) {
      const int m0 = (tile % m_tiles) * kBM;
      const int n0 = (tile / m_tiles) * kBN;
      mbar_wait(tmem_full, iter & 1);
      tc_fence_after();
      const int y = m0 + (int)row_in_tile;
      const bool row_ok = y < args.n_out;
#pragma unroll 1
      for (int c8 = 0; c8 < kBN / 8; ++c8) {
        uint32_t acc0[C::S0][8], acc1[C::S1][8];
#pragma unroll
        for (int s = 0; s < C::S0; ++s) tmem_ld_x8(tmem_base + lane_addr + s * kBN + c8 * 8, acc0[s]);
#pragma unroll
        for (int s = 0; s < C::S1; ++s) tmem_ld_x8(tmem_base + lane_addr + (C::S0 + s) * kBN + c8 * 8, acc1[s]);
        tmem_ld_wait();
        uint32_t res[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          // limb 0: sum_s 2^(8s) * acc_s  mod q0
          uint32_t x0 = 0, x1 = 0;
#pragma unroll
          for (int s = 0; s < C::S0; ++s) {
            const uint32_t v = acc0[s][e];
            const uint32_t u = ((int32_t)v < 0) ? v + c.offs[0] : v;   // == acc (mod q0), < 2^32
            x0 = add_mod(x0, shoup_mul(u, c.pw[0][s], c.pwp[0][s], c.q[0]), c.q[0]);
          }
#pragma unroll
          for (int s = 0; s < C::S1; ++s) {
            const uint32_t v = acc1[s][e];
            const uint32_t u = ((int32_t)v < 0) ? v + c.offs[1] : v;
            x1 = add_mod(x1, shoup_mul(u, c.pw[1][s], c.pwp[1][s], c.q[1]), c.q[1]);
          }
          // rescale: ((x0 - [x1]_centred) * q1^-1) mod q0
          uint32_t t;
          if (x1 > (c.q[1] >> 1)) {
            t = csub(x0 + (c.q[1] - x1), c.q[0]);              // x0 + |x1c|
          } else {
            t = sub_mod(x0, x1, c.q[0]);
          }
          res[e] = shoup_mul(t, c.q1inv, c.q1invp, c.q[0]);
        }
        if (row_ok) {
          const int n = n0 + c8 * 8;
          if (n < args.d) {
            // b' composed into RLWE order: b_rlwe[y / k][(y % k) + k * m]
            uint32_t* dst = args.out_b + (size_t)(y / args.k) * N + (y % args.k);
#pragma unroll
            for (int e = 0; e < 8; ++e) dst[(size_t)args.k * (n + e)] = res[e];
          } else {
            uint4* dst = reinterpret_cast<uint4*>(args.out_a + (size_t)y * (N) + (n - args.d));
            dst[0] = make_uint4(res[0], res[1], res[2], res[3]);
            dst[1] = make_uint4(res[4], res[5], res[6], res[7]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(tmem_empty);
    }
  }

  __syncwarp();  // reconverge each role warp before the CTA barrier
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemAlloc);
  }
}

// ======================================================================================
// K1 v2: CTA pair (cta_group::2).  One pair-tile = 256 rows (128 per CTA) x 48 GEMM columns x
// both limbs.  Each CTA stages its 128 weight rows (A) and HALF of every stacked ciphertext
// operand (B, split along N between the pair), so the tensor cores of the two SMs share
// operands and each SM reads ~80 B/clk of shared memory per MMA cycle instead of ~134.
// The leader CTA issues all MMAs; commits are multicast to both CTAs' barriers.
// 8 epilogue warps per CTA (two per TMEM lane quarter) halve the drain time of the single
// accumulator buffer.  Raster: groups of kGroupM pair-rows sweep all N blocks, so the weight
// planes of a group stay L2-resident while the ciphertext planes stream.
constexpr int kEpiWarps = 8;
constexpr int kThreads2 = 64 + 32 * kEpiWarps;

// tile width: 48 GEMM columns when the shift accumulators fit TMEM (d_w <= 2), else 32
__host__ __device__ constexpr int gemm2_bn(int dw, int d0, int d1) {
  return ((2 * dw + d0 + d1 - 2) * 48 <= 512 && (dw + d0 - 1) * 48 <= 256 && (dw + d1 - 1) * 48 <= 256) ? 48 : 32;
}

// sum_s 2^(8 s) acc_s mod q for one output word.  S <= 5: exact signed int64 sum (plan-time
// bound K 2^14 sum_s pairs(s) 2^(8s) < 2^62) and one Barrett reduction; else per-shift Shoup.
template <int S>
__device__ __forceinline__ uint32_t recombine(const uint32_t (*acc)[8], int e, const GemmEpiConst& c, int L) {
  const uint32_t q = c.q[L];
  if constexpr (S <= 5) {
    int64_t v = (int32_t)acc[0][e];
#pragma unroll
    for (int s = 1; s < S; ++s) v += (int64_t)(int32_t)acc[s][e] << (8 * s);
    const uint64_t u = (uint64_t)v + c.off64[L];
    const uint64_t qh = __umul64hi(u, c.mu[L]);
    return csub((uint32_t)(u - qh * q), q);
  } else {
    uint32_t x = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const uint32_t v = acc[s][e];
      const uint32_t u = ((int32_t)v < 0) ? v + c.offs[L] : v;
      x = add_mod(x, shoup_mul(u, c.pw[L][s], c.pwp[L][s], q), q);
    }
    return x;
  }
}

template <int DW, int D0, int D1, int BN>
struct Gemm2Cfg {
  static constexpr int kBN2 = BN;
  static constexpr int kChunk = kBN2 / 2;  // TMA box rows for B (half a digit plane)
  static constexpr int S0 = DW + D0 - 1, S1 = DW + D1 - 1;
  static constexpr int kTmemCols = (S0 + S1) * kBN2;
  static constexpr int kTmemAlloc = 512;
  static constexpr int kABytes = DW * kBM * kBK;                    // per CTA per stage
  static constexpr int kB0Rows = D0 * kChunk, kB1Rows = D1 * kChunk; // per CTA (half of D_i * 48)
  static constexpr int kBBytes = (kB0Rows + kB1Rows) * kBK;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (224 * 1024 - 9472) / kStageBytes > 6 ? 6 : (224 * 1024 - 9472) / kStageBytes;
  static constexpr int kZeroBytes = 8192;
  static constexpr int kSmemBytes = kStages * kStageBytes + kZeroBytes + 1024 + 256;
  static_assert(kTmemCols <= 512, "too many shift accumulators for TMEM");
  static_assert(kStages >= 2, "not enough shared memory");
  static_assert(S0 * kBN2 <= 256 && S1 * kBN2 <= 256, "zeroing MMA N out of range");
};

template <int DW, int D0, int D1, int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    modgemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmBa, const GemmArgs args) {
  using C = Gemm2Cfg<DW, D0, D1, BN>;
  constexpr int kBN2 = C::kBN2;
  constexpr int kChunk = C::kChunk;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint8_t* sZero = sB + C::kStages * C::kBBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sZero + C::kZeroBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tmem_full = empty + C::kStages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int m_tiles = (args.n_out + 2 * kBM - 1) / (2 * kBM);
  const int n_tiles = (args.width + kBN2 - 1) / kBN2;
  const int num_tiles = m_tiles * n_tiles;
  const int num_kb = (args.n_in + kBK - 1) / kBK;
  const int gm = args.group_m < m_tiles ? args.group_m : m_tiles;

  for (int i = threadIdx.x; i < C::kZeroBytes / 16; i += kThreads2)
    reinterpret_cast<uint4*>(sZero)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmBa);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 2);      // leader's expect_tx arrive + the peer's remote arrive
      mbar_init(&empty[s], 1);     // one multicast commit
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 2 * kEpiWarps);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc_2sm(tmem_slot, C::kTmemAlloc);
    tmem_relinquish_2sm();
  }
  fence_proxy_async();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // tile -> (m block of 256 rows, n block of kBN2 columns), M-grouped raster.  Fused path: the
  // a-part column tiles are visited as (m-range, j mod 16, j / 16) so that consecutive tiles read
  // the same rows of the same 16-byte-shifted digit copy (L2 reuse across key components j).
  auto tile_mn = [&](int tile, int& m0, int& n0) {
    const int per_group = gm * n_tiles;
    const int g = tile / per_group, r = tile % per_group;
    const int rows_in_group = (m_tiles - g * gm) < gm ? (m_tiles - g * gm) : gm;
    m0 = (g * gm + r % rows_in_group) * (2 * kBM);
    const int v = r / rows_in_group;
    if (!args.fused) {
      n0 = v * kBN2;
    } else {
      const int nb_b = args.d / kBN2;                  // b-part tiles first
      if (v < nb_b) {
        n0 = v * kBN2;
      } else {
        const int va = v - nb_b, J = args.k, jh_n = J / 16;
        const int mb = va / J, rem = va % J;
        const int j = 16 * (rem % jh_n) + rem / jh_n;
        n0 = args.d + args.d * j + kBN2 * mb;
      }
    }
  };

  if (warp == 0) {
    // ======================= TMA producer (both CTAs) =======================
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0_remote = mapa_rank(&full[0], 0);
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        int m0, n0;
        tile_mn(tile, m0, n0);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], 2 * C::kStageBytes);
          else mbar_arrive_cluster(full0_remote + stage * 8);
          uint8_t* a_dst = sA + stage * C::kABytes;
          uint8_t* b_dst = sB + stage * C::kBBytes;
#pragma unroll
          for (int a = 0; a < DW; ++a)
            tma_load_3d_2sm(a_dst + a * kBM * kBK, &tmA, &full[stage], kb * kBK, m0 + (int)rank * kBM, a, args.hint_a);
          // stacked limb-i operand [C0|C1|..] (D_i * kBN2 rows): this CTA holds chunks [rank*D_i, (rank+1)*D_i)
          const int r_ct = (kb * kBK) / args.k, t0 = (kb * kBK) % args.k;
          auto load_chunk = [&](uint8_t* dst, int plane, int n_c) {
            if (!args.fused) {
              tma_load_3d_2sm(dst, &tmB, &full[stage], kb * kBK, n_c, plane, args.hint_b);
            } else if (n_c < args.d) {             // b part: b_r[t + k m], rows m = n_c ..
              tma_load_4d_2sm(dst, &tmB, &full[stage], t0, n_c, r_ct, plane, args.hint_b);
            } else {                               // a part: a_r[t - j + k m] from the shift copy
              const int j = (n_c - args.d) / args.d, m = (n_c - args.d) % args.d;
              const int sh = (16 - (j & 15)) & 15;
              const int I0 = t0 - j + args.k * (m + 1) - sh;
              tma_load_4d_2sm(dst, &tmBa, &full[stage], I0 % args.k, I0 / args.k, r_ct, plane * 16 + sh, args.hint_b);
            }
          };
#pragma unroll
          for (int c = 0; c < D0; ++c) {
            const int g = (int)rank * D0 + c;
            load_chunk(b_dst + c * kChunk * kBK, g >> 1, n0 + (g & 1) * kChunk);
          }
#pragma unroll
          for (int c = 0; c < D1; ++c) {
            const int g = (int)rank * D1 + c;
            load_chunk(b_dst + (C::kB0Rows + c * kChunk) * kBK, D0 + (g >> 1), n0 + (g & 1) * kChunk);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA only) =======================
    if (leader) {
      constexpr uint32_t kIdesc0 = idesc_i8(2 * kBM, D0 * kBN2);
      constexpr uint32_t kIdesc1 = idesc_i8(2 * kBM, D1 * kBN2);
      constexpr uint32_t kIdescZ0 = idesc_i8(2 * kBM, C::S0 * kBN2);
      constexpr uint32_t kIdescZ1 = idesc_i8(2 * kBM, C::S1 * kBN2);
      const uint32_t reg0 = tmem_base;
      const uint32_t reg1 = tmem_base + C::S0 * kBN2;
      const uint64_t zdesc = desc_noswz(smem_u32(sZero), 128, 256);
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs, ++iter) {
        if (iter > 0) mbar_wait(tmem_empty, (iter - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          mma_i8_2sm(reg0, zdesc, zdesc, kIdescZ0, 0);
          mma_i8_2sm(reg1, zdesc, zdesc, kIdescZ1, 0);
        }
        __syncwarp();
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_base = smem_u32(sA + stage * C::kABytes);
            const uint32_t b_base = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
            for (int kk = 0; kk < kBK / 32; ++kk) {
              const uint64_t b0 = desc_sw128(b_base + kk * 32);
              const uint64_t b1 = desc_sw128(b_base + C::kB0Rows * kBK + kk * 32);
#pragma unroll
              for (int a = 0; a < DW; ++a) {
                const uint64_t ad = desc_sw128(a_base + a * kBM * kBK + kk * 32);
                mma_i8_2sm(reg0 + a * kBN2, ad, b0, kIdesc0, 1);
                mma_i8_2sm(reg1 + a * kBN2, ad, b1, kIdesc1, 1);
              }
            }
            tc_commit_2sm_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) tc_commit_2sm_mc(tmem_full, 0x3);
        __syncwarp();
      }
    }
  } else {
    // ======================= epilogue (both CTAs, 8 warps) =======================
    const uint32_t ew = warp - 2;
    const uint32_t quarter = warp & 3;
    const uint32_t half = ew / 4;                      // which 3 of the 6 column chunks
    const uint32_t lane_addr = (quarter * 32) << 16;
    const int N = args.d * args.k;
    const GemmEpiConst& c = args.c;
    const uint32_t tmem_empty_remote = mapa_rank(tmem_empty, 0);
    int iter = 0;
    for (int tile = pair; tile < num_tiles; tile += npairs, ++iter) {
      int m0, n0;
      tile_mn(tile, m0, n0);
      mbar_wait(tmem_full, iter & 1);
      tc_fence_after();
      const int y = m0 + (int)rank * kBM + (int)(quarter * 32 + lane);
      const bool row_ok = y < args.n_out;
#pragma unroll 1
      for (int cc = 0; cc < kBN2 / 16; ++cc) {
        const int c8 = (int)half * (kBN2 / 16) + cc;
        const int n = n0 + c8 * 8;
        if (n >= args.width) break;  // warp-uniform
        uint32_t acc0[C::S0][8], acc1[C::S1][8];
#pragma unroll
        for (int s = 0; s < C::S0; ++s) tmem_ld_x8(tmem_base + lane_addr + s * kBN2 + c8 * 8, acc0[s]);
#pragma unroll
        for (int s = 0; s < C::S1; ++s) tmem_ld_x8(tmem_base + lane_addr + (C::S0 + s) * kBN2 + c8 * 8, acc1[s]);
        tmem_ld_wait();
        if (args.epi_skip) continue;
        uint32_t res[8];
        if (args.out1_b) {  // level-1 mode: both limbs' words, no rescale (same layouts)
          uint32_t r1[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            res[e] = recombine<C::S0>(acc0, e, c, 0);
            r1[e] = recombine<C::S1>(acc1, e, c, 1);
          }
          if (row_ok) {
            if (n < args.d) {
              const size_t o = (size_t)(y / args.k) * N + (y % args.k);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                args.out_b[o + (size_t)args.k * (n + e)] = res[e];
                args.out1_b[o + (size_t)args.k * (n + e)] = r1[e];
              }
            } else {
              const size_t o = (size_t)y * N + (n - args.d);
              uint4* d0 = reinterpret_cast<uint4*>(args.out_a + o);
              uint4* d1 = reinterpret_cast<uint4*>(args.out1_a + o);
              d0[0] = make_uint4(res[0], res[1], res[2], res[3]);
              d0[1] = make_uint4(res[4], res[5], res[6], res[7]);
              d1[0] = make_uint4(r1[0], r1[1], r1[2], r1[3]);
              d1[1] = make_uint4(r1[4], r1[5], r1[6], r1[7]);
            }
          }
          continue;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t x0 = recombine<C::S0>(acc0, e, c, 0);
          const uint32_t x1 = recombine<C::S1>(acc1, e, c, 1);
          uint32_t t;
          if (x1 > (c.q[1] >> 1)) t = csub(x0 + (c.q[1] - x1), c.q[0]);
          else t = sub_mod(x0, x1, c.q[0]);
          res[e] = shoup_mul(t, c.q1inv, c.q1invp, c.q[0]);
        }
        if (row_ok) {
          const int np = args.peers.n > 0 ? args.peers.n : 1;
          const size_t yd = args.peers.n > 0 ? (size_t)args.peers.dst_row0 + y : (size_t)y;
          for (int pr = 0; pr < np; ++pr) {
            if (n < args.d) {
              uint32_t* ob = args.peers.n > 0 ? args.peers.b[pr] : args.out_b;
              uint32_t* dst = ob + (yd / args.k) * N + (yd % args.k);
#pragma unroll
              for (int e = 0; e < 8; ++e) dst[(size_t)args.k * (n + e)] = res[e];
            } else {
              uint32_t* oa = args.peers.n > 0 ? args.peers.a[pr] : args.out_a;
              uint4* dst = reinterpret_cast<uint4*>(oa + yd * N + (n - args.d));
              dst[0] = make_uint4(res[0], res[1], res[2], res[3]);
              dst[1] = make_uint4(res[4], res[5], res[6], res[7]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tmem_empty_remote);
    }
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, C::kTmemAlloc);
  }
}

template <int DW, int D0, int D1, int BN>
static cudaError_t launch2_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmBa,
                             const GemmArgs& args, int grid, cudaStream_t stream) {
  using C = Gemm2Cfg<DW, D0, D1, BN>;
  auto kern = modgemm2_kernel<DW, D0, D1, BN>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads2, C::kSmemBytes, stream>>>(tmA, tmB, tmBa, args);
  return cudaGetLastError();
}

template <int DW, int D0, int D1>
static cudaError_t launch_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& args, int grid,
                            cudaStream_t stream) {
  using C = GemmCfg<DW, D0, D1>;
  auto kern = modgemm_kernel<DW, D0, D1>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, C::kSmemBytes, stream>>>(tmA, tmB, args);
  return cudaGetLastError();
}

int gemm2_tile_n(int dw, int d0, int d1) { return gemm2_bn(dw, d0, d1); }

int gemm_smem_bytes(int dw, int d0, int d1) {
#define HE_CASE(a, b, c) \
  if (dw == a && d0 == b && d1 == c) return GemmCfg<a, b, c>::kSmemBytes;
  HE_GEMM_INSTANCES(HE_CASE)
#undef HE_CASE
  return -1;
}

cudaError_t launch_modgemm(int variant, int dw, int d0, int d1, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmBa, const GemmArgs& args, int grid, cudaStream_t stream) {
#define HE_CASE(a, b, c)                                                                   \
  if (dw == a && d0 == b && d1 == c) {                                                    \
    if (variant == 1) return launch_t<a, b, c>(tmA, tmB, args, grid, stream);            \
    if constexpr (gemm2_bn(a, b, c) == 48)                                                \
      if (args.tile_n == 48) return launch2_t<a, b, c, 48>(tmA, tmB, tmBa, args, grid, stream); \
    if (args.tile_n == 32) return launch2_t<a, b, c, 32>(tmA, tmB, tmBa, args, grid, stream);   \
    return cudaErrorInvalidValue;                                                         \
  }
  HE_GEMM_INSTANCES(HE_CASE)
#undef HE_CASE
  return cudaErrorInvalidValue;
}

}  // namespace he
