// crc_math.h -- GF(2) arithmetic for the reference's CRC-32 (zlib polynomial,
// reflected 0xEDB88320, init/xorout 0xFFFFFFFF: include/gpucrsim/crc32.hpp:12-34).
//
// Representation (zlib's): a 32-bit word is a polynomial of degree < 32 with
// the coefficient of x^k in bit 31-k.  The raw CRC register r (before the
// final inversion) evolves per byte b as r <- Z(r ^ b) with
// Z(r) = T[r & 0xff] ^ (r >> 8); Z^n(r) = r * x^(8n) mod P.  Everything the
// kernels need is a linear map of this kind, so it is tabulated here on the
// host and uploaded once per context.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define POS_HD __host__ __device__ __forceinline__
#else
#define POS_HD inline
#endif

namespace posdump {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr uint32_t kXPow0 = 0x80000000u;  // x^0
constexpr uint32_t kXInv = 0xDB710641u;   // x^-1 = ((P-1)/x): (kPoly << 1) | 1

// a(x) * b(x) mod P  (zlib multmodp).
POS_HD uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// x^(8n) mod P.
POS_HD uint32_t x8nmodp(uint64_t n) {
  uint32_t sq = 1u << 30;  // x^1
  sq = multmodp(sq, sq);   // x^2
  sq = multmodp(sq, sq);   // x^4
  sq = multmodp(sq, sq);   // x^8
  uint32_t p = kXPow0;
  while (n) {
    if (n & 1) p = multmodp(sq, p);
    sq = multmodp(sq, sq);
    n >>= 1;
  }
  return p;
}

// x^(-8n) mod P.
POS_HD uint32_t xinv8nmodp(uint64_t n) {
  uint32_t sq = kXInv;
  sq = multmodp(sq, sq);
  sq = multmodp(sq, sq);
  sq = multmodp(sq, sq);  // x^-8
  uint32_t p = kXPow0;
  while (n) {
    if (n & 1) p = multmodp(sq, p);
    sq = multmodp(sq, sq);
    n >>= 1;
  }
  return p;
}

// crc32 of `len` zero bytes == raw-to-final offset: crc = raw ^ zeros_crc(len).
POS_HD uint32_t zeros_crc(uint64_t len) { return ~multmodp(x8nmodp(len), 0xFFFFFFFFu); }

// zlib crc32_combine: crc(A||B) from crc(A), crc(B), len(B).
POS_HD uint32_t crc32_combine(uint32_t a, uint32_t b, uint64_t len_b) {
  return multmodp(x8nmodp(len_b), a) ^ b;
}

// Slicing table of Z^N: tab[k*256 + e] = Z^N(e << 8k), so
// Z^N(r) = tab[0][r&255] ^ tab[1][(r>>8)&255] ^ tab[2][(r>>16)&255] ^ tab[3][r>>24].
inline void build_advance_table(uint64_t n_bytes, uint32_t* tab /*1024*/) {
  uint32_t xn = x8nmodp(n_bytes);
  for (uint32_t k = 0; k < 4; ++k)
    for (uint32_t e = 0; e < 256; ++e) tab[k * 256 + e] = multmodp(xn, e << (8 * k));
}

}  // namespace posdump
