// gpucrsim/crc32.hpp -- DROP-IN replacement of the reference's CRC-32
// (proj/include/gpucrsim/crc32.hpp:12-34): same functions, same digest
// (zlib: reflected 0xEDB88320, init / xorout 0xFFFFFFFF), but bytes that are
// the host mirror of a device-resident GpuBuffer (gpucrsim/buffer.hpp) are
// hashed ON THE DEVICE by libposdump (pos_crc32 / pos_crc32_update:
// k_hash_chunks + the GF(2) fold) -- scan_dedup (cr.hpp:419) and
// note_h2d_provenance (process.hpp:518) hash a whole buffer's content.
// Host-only bytes (host pages in dedup_consistent, cr.hpp:692-708; image
// sections in read_image, image.hpp:349) stay on the host: slice-by-8.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <cstring>

#include "gpucrsim/buffer.hpp"

namespace gpucrsim {

namespace detail {
inline const std::array<std::array<uint32_t, 256>, 8>& crc32_slices() {
  static const auto tabs = [] {
    std::array<std::array<uint32_t, 256>, 8> t{};
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int s = 1; s < 8; ++s) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xFF];
    return t;
  }();
  return tabs;
}
inline const std::array<uint32_t, 256>& crc32_table() { return crc32_slices()[0]; }

inline uint32_t host_crc32_update(uint32_t crc, const uint8_t* p, size_t n) {
  const auto& t = crc32_slices();
  uint32_t c = ~crc;
  for (; n >= 8; p += 8, n -= 8) {
    uint32_t lo, hi;
    std::memcpy(&lo, p, 4);
    std::memcpy(&hi, p + 4, 4);
    lo ^= c;
    c = t[7][lo & 0xFF] ^ t[6][(lo >> 8) & 0xFF] ^ t[5][(lo >> 16) & 0xFF] ^ t[4][lo >> 24] ^ t[3][hi & 0xFF] ^
        t[2][(hi >> 8) & 0xFF] ^ t[1][(hi >> 16) & 0xFF] ^ t[0][hi >> 24];
  }
  while (n--) c = t[0][(c ^ *p++) & 0xFF] ^ (c >> 8);
  return ~c;
}
}  // namespace detail

// crc32_update continues a FINAL crc (crc32.hpp:26-32).
inline uint32_t crc32_update(uint32_t crc, const void* data, size_t n) {
  if (n) {
    if (const uint64_t dev = devmem::device_of(data, n)) {
      uint32_t out = 0;
      devmem::ck(pos_crc32_update(crc, dev, n, &out, nullptr), "device crc32");
      return out;
    }
  }
  return detail::host_crc32_update(crc, static_cast<const uint8_t*>(data), n);
}

inline uint32_t crc32(const void* data, size_t n) { return crc32_update(0, data, n); }

}  // namespace gpucrsim
