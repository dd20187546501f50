// host_crc.h -- the reference's CRC-32 (crc32.hpp:12-34) over HOST bytes, for
// the one check of the path whose bytes live only on the host: finalize's
// dedup_consistent over the image's host pages (cr.hpp:692-708).
// Slice-by-8 table walk per thread; long ranges are split over host threads
// and joined with crc32_combine (crc_math.h).  Device bytes never come here:
// they are hashed by k_hash_chunks.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "crc_math.h"

namespace posdump {

struct HostCrcTables {
  uint32_t t[8][256];
  HostCrcTables() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
      t[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int s = 1; s < 8; ++s) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xff];
  }
};

inline const HostCrcTables& host_crc_tables() {
  static const HostCrcTables tabs;
  return tabs;
}

// crc32_update(crc, p, n) (crc32.hpp:26-32): continues a FINAL crc.
inline uint32_t host_crc32_update(uint32_t crc, const uint8_t* p, uint64_t n) {
  const auto& T = host_crc_tables().t;
  uint32_t c = ~crc;
  while (n && (reinterpret_cast<uintptr_t>(p) & 7)) {
    c = T[0][(c ^ *p++) & 0xff] ^ (c >> 8);
    --n;
  }
  while (n >= 8) {
    uint64_t w;
    std::memcpy(&w, p, 8);
    const uint32_t lo = (uint32_t)w ^ c, hi = (uint32_t)(w >> 32);
    c = T[7][lo & 0xff] ^ T[6][(lo >> 8) & 0xff] ^ T[5][(lo >> 16) & 0xff] ^ T[4][lo >> 24] ^
        T[3][hi & 0xff] ^ T[2][(hi >> 8) & 0xff] ^ T[1][(hi >> 16) & 0xff] ^ T[0][hi >> 24];
    p += 8;
    n -= 8;
  }
  while (n--) c = T[0][(c ^ *p++) & 0xff] ^ (c >> 8);
  return ~c;
}

// crc32(p, n), ranges >= 64 MiB on up to `threads` host threads.
inline uint32_t host_crc32(const uint8_t* p, uint64_t n, unsigned threads = 16) {
  const uint64_t piece = 16ull << 20;
  unsigned nt = (unsigned)std::min<uint64_t>(threads ? threads : 1, n / piece);
  if (nt < 4) return host_crc32_update(0, p, n);
  std::vector<uint32_t> part(nt);
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      const uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
      part[t] = host_crc32_update(0, p + lo, hi - lo);
    });
  for (auto& th : pool) th.join();
  uint32_t crc = part[0];
  for (unsigned t = 1; t < nt; ++t) crc = crc32_combine(crc, part[t], n * (t + 1) / nt - n * t / nt);
  return crc;
}

}  // namespace posdump
