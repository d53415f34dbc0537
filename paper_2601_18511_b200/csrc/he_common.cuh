// he_common.cuh -- shared device helpers: counter-based RNG, modular arithmetic, PTX wrappers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HE_HD __host__ __device__ __forceinline__
#define HE_D __device__ __forceinline__

namespace he {

// ---------------------------------------------------------------- RNG
// Keyed splitmix64 counter generator.  Restated bit-for-bit from the oracle
// (oracle/he_oracle.c: mix64 / or_rng_key / draw) so GPU encryption is
// reproducible and checkable word-for-word against the CPU restatement.
HE_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
HE_HD uint64_t rng_key(uint64_t seed, uint64_t stream) {
  return mix64((seed * 0xD1B54A32D192ED03ULL) ^ mix64(stream + 0x9E3779B97F4A7C15ULL));
}
HE_HD uint64_t rng_draw(uint64_t key, uint64_t idx) { return mix64(key + (idx + 1) * 0x9E3779B97F4A7C15ULL); }

// ---------------------------------------------------------------- secure sampling (ChaCha20, RFC 8439)
// A context created with a 256-bit secret key (he_context_set_rng_key) samples secrets, masks a,
// errors and key-switching keys from ChaCha20 instead: a per-seed subkey
//   K_seed = ChaCha20_block(K, counter 0xFFFFFFFF, nonce (seed_lo, seed_hi, 0x5EED5EED))[0..8)
// and draw idx of stream = the first 64 bits of ChaCha20_block(K_seed, (uint32)idx,
// nonce (stream_lo, stream_hi, idx >> 32)).  Without a key (the seeded test path) the splitmix draws above
// are used, which the oracle restates bit for bit.
struct RngCtx {
  uint32_t key[8];
  uint32_t secure;
};
HE_HD uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
HE_HD void chacha_qr(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  a += b; d ^= a; d = rotl32(d, 16);
  c += d; b ^= c; b = rotl32(b, 12);
  a += b; d ^= a; d = rotl32(d, 8);
  c += d; b ^= c; b = rotl32(b, 7);
}
HE_HD void chacha20_block(const uint32_t key[8], uint32_t counter, uint32_t n0, uint32_t n1, uint32_t n2,
                          uint32_t out[16]) {
  uint32_t x[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key[0], key[1], key[2], key[3],
                    key[4],      key[5],      key[6],      key[7],      counter, n0, n1, n2};
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = x[i];
#pragma unroll 1
  for (int r = 0; r < 10; ++r) {
    chacha_qr(w[0], w[4], w[8], w[12]);
    chacha_qr(w[1], w[5], w[9], w[13]);
    chacha_qr(w[2], w[6], w[10], w[14]);
    chacha_qr(w[3], w[7], w[11], w[15]);
    chacha_qr(w[0], w[5], w[10], w[15]);
    chacha_qr(w[1], w[6], w[11], w[12]);
    chacha_qr(w[2], w[7], w[8], w[13]);
    chacha_qr(w[3], w[4], w[9], w[14]);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) out[i] = w[i] + x[i];
}
struct Rng {
  uint64_t det;
  uint32_t k[8];
  uint32_t s0, s1;
  uint32_t secure;
};
HE_HD Rng rng_make(const RngCtx& rc, uint64_t seed, uint64_t stream) {
  Rng r;
  r.secure = rc.secure;
  r.det = rng_key(seed, stream);
  r.s0 = (uint32_t)stream;
  r.s1 = (uint32_t)(stream >> 32);
  if (rc.secure) {
    uint32_t b[16];
    chacha20_block(rc.key, 0xFFFFFFFFu, (uint32_t)seed, (uint32_t)(seed >> 32), 0x5EED5EEDu, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) r.k[i] = b[i];
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) r.k[i] = 0;
  }
  return r;
}
HE_HD uint64_t rng_next(const Rng& r, uint64_t idx) {
  if (!r.secure) return rng_draw(r.det, idx);
  uint32_t b[16];
  chacha20_block(r.k, (uint32_t)idx, r.s0, r.s1, (uint32_t)(idx >> 32), b);
  return (uint64_t)b[0] | ((uint64_t)b[1] << 32);
}

constexpr uint64_t kStreamSecret = 0x5EC0000000000000ULL;
HE_HD uint64_t stream_a(uint32_t r, uint32_t limb) { return 0xA000000000000000ULL | ((uint64_t)r << 8) | limb; }
HE_HD uint64_t stream_e(uint32_t r) { return 0xE000000000000000ULL | ((uint64_t)r << 8); }

HE_HD int32_t cbd21(uint64_t x) {
  return __builtin_popcountll(x & 0x1FFFFFULL) - __builtin_popcountll((x >> 21) & 0x1FFFFFULL);
}
HE_D int32_t cbd21_d(uint64_t x) { return __popcll(x & 0x1FFFFFULL) - __popcll((x >> 21) & 0x1FFFFFULL); }
HE_HD int32_t ternary(uint64_t x) {
  uint32_t b = (uint32_t)(x & 3u);
  return b == 1 ? 1 : (b == 2 ? -1 : 0);
}

// ---------------------------------------------------------------- modular arithmetic (q < 2^31)
HE_HD uint32_t shoup_pre(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
// x * w mod q in [0, 2q) for any x < 2^32, w < q < 2^31 (Shoup).
HE_D uint32_t shoup_lazy(uint32_t x, uint32_t w, uint32_t wp, uint32_t q) {
  uint32_t hi = __umulhi(x, wp);
  return x * w - hi * q;
}
HE_D uint32_t csub(uint32_t x, uint32_t q) { return x >= q ? x - q : x; }
HE_D uint32_t shoup_mul(uint32_t x, uint32_t w, uint32_t wp, uint32_t q) { return csub(shoup_lazy(x, w, wp, q), q); }
HE_D uint32_t add_mod(uint32_t a, uint32_t b, uint32_t q) { return csub(a + b, q); }
HE_D uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t q) { return a >= b ? a - b : a + q - b; }
HE_D uint32_t mul_mod(uint32_t a, uint32_t b, uint32_t q) { return (uint32_t)(((uint64_t)a * b) % q); }
HE_D uint32_t from_i64(int64_t v, uint32_t q) {
  int64_t r = v % (int64_t)q;
  return (uint32_t)(r < 0 ? r + q : r);
}
HE_HD uint64_t powmod_h(uint64_t a, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = (uint64_t)((unsigned __int128)r * a % q);
    a = (uint64_t)((unsigned __int128)a * a % q);
    e >>= 1;
  }
  return r;
}

// balanced base-256 digit i of a centred residue c: c = sum_i d_i 256^i, d_i in [-128, 127]
HE_D void balanced_digits4(int32_t c, int8_t* d, int nd) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nd) {
      int32_t di = (int32_t)(int8_t)(c & 0xFF);
      d[i] = (int8_t)di;
      c = (c - di) >> 8;
    }
  }
}

HE_HD uint32_t bitrev_h(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int t = 0; t < bits; ++t) r |= ((x >> t) & 1u) << (bits - 1 - t);
  return r;
}
HE_HD int ilog2_h(uint32_t x) {
  int l = 0;
  while ((1u << l) < x) ++l;
  return l;
}
// sigma(t) = f(bitReverse(t, log k), log k)  (hesim bitrev.py:24-45)
HE_HD uint32_t sigma_h(uint32_t t, int logk) {
  uint32_t b = bitrev_h(t, logk);
  return (b >> 1) | ((b & 1u) << (logk - 1));
}

}  // namespace he
