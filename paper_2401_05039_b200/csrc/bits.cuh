// bits.cuh — small pure helpers used by the search kernel (host+device so
// they can be unit-tested on the CPU build machine: tests/test_bits_host.py).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define MBE_HD __host__ __device__ __forceinline__
#else
#define MBE_HD inline
#endif

// splitmix64 finalizer: the library's own copy (the oracle keeps a separate one).
MBE_HD uint64_t mbe_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

MBE_HD uint64_t mbe_rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

// H(A,B) of one biclique from its side sums/sizes.
// L' is a subset of V (non-candidate side), R' of U (candidate side).
MBE_HD uint64_t mbe_biclique_hash(int cand_side, uint64_t sL, uint32_t nL, uint64_t sR, uint32_t nR) {
  uint64_t sA = cand_side == 1 ? sR : sL, sB = cand_side == 1 ? sL : sR;
  uint64_t nA = cand_side == 1 ? nR : nL, nB = cand_side == 1 ? nL : nR;
  return mbe_mix64(sA ^ mbe_rotl64(sB, 32) ^ (nA << 32) ^ nB);
}

MBE_HD uint32_t mbe_popc(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __popc(x);
#else
  return (uint32_t)__builtin_popcount(x);
#endif
}

// Column compression (bit gather) of one 32-bit word by a fixed mask m:
// compress(x, m) packs the bits of x at the set positions of m into the low
// bits, in position order.  The five shift masks depend on m only, so they
// are prepared once per task and reused for every row (Warren, Hacker's
// Delight, "compress" with the parallel-suffix method).
struct MbeCompress32 {
  uint32_t m;
  uint32_t mv[5];
};

MBE_HD MbeCompress32 mbe_compress_prep(uint32_t m) {
  MbeCompress32 c;
  c.m = m;
  uint32_t mk = ~m << 1;
  for (int i = 0; i < 5; ++i) {
    uint32_t mp = mk ^ (mk << 1);
    mp ^= mp << 2;
    mp ^= mp << 4;
    mp ^= mp << 8;
    mp ^= mp << 16;
    uint32_t v = mp & m;
    c.mv[i] = v;
    m = (m ^ v) | (v >> (1 << i));
    mk = mk & ~mp;
  }
  return c;
}

MBE_HD uint32_t mbe_compress_apply(const MbeCompress32& c, uint32_t x) {
  x &= c.m;
  for (int i = 0; i < 5; ++i) {
    uint32_t t = x & c.mv[i];
    x = (x ^ t) | (t >> (1 << i));
  }
  return x;
}

// Multi-word compression: W input words (mask words m[0..W)) into the low
// popc(m) bits of up to 4 output words.
template <int W>
struct MbeCompress {
  MbeCompress32 c[W];
  uint32_t off[W];  // output bit offset of word w = Σ_{w'<w} popc(m[w'])
};

template <int W>
MBE_HD MbeCompress<W> mbe_compress_prep_w(const uint32_t* m) {
  MbeCompress<W> c;
  uint32_t o = 0;
  for (int w = 0; w < W; ++w) {
    c.c[w] = mbe_compress_prep(m[w]);
    c.off[w] = o;
    o += mbe_popc(m[w]);
  }
  return c;
}

template <int W>
MBE_HD void mbe_compress_apply_w(const MbeCompress<W>& c, const uint32_t* x, uint32_t* out /* [4] */) {
  out[0] = out[1] = out[2] = out[3] = 0;
  for (int w = 0; w < W; ++w) {
    uint32_t y = mbe_compress_apply(c.c[w], x[w]);
    uint32_t o = c.off[w];
    uint32_t q = o >> 5, r = o & 31;
    out[q] |= y << r;
    if (r && q + 1 < 4) out[q + 1] |= y >> (32 - r);
  }
}

// Words per bit row for a frame with n columns (1, 2, 4, 8 or 16).
MBE_HD uint32_t mbe_words_for(uint32_t n) {
  return n <= 32 ? 1u : (n <= 64 ? 2u : (n <= 128 ? 4u : (n <= 256 ? 8u : 16u)));
}
