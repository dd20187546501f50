/*
 * posdump_oracle.c -- CPU restatement of the reference's buffer-dump path.
 *
 * TEST INFRASTRUCTURE ONLY (see posdump_oracle.h).  Plain C, scalar, single
 * threaded: it is the checker the CUDA path is compared against, never the
 * thing shipped or measured as the product.
 *
 * Citations are path:line relative to /root/reference/proj.
 */
#include "posdump_oracle.h"

#include <string.h>

/* ---- CRC-32 ------------------------------------------------------------- */

static uint32_t g_table[256];
static int g_table_ready = 0;

/* Table build: include/gpucrsim/crc32.hpp:12-23 (reflected poly 0xEDB88320). */
static void build_table(void) {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    g_table[i] = c;
  }
  g_table_ready = 1;
}

/* Byte-serial update: include/gpucrsim/crc32.hpp:26-32.  `crc` is a finalised
 * CRC, so chained updates equal the CRC of the concatenation. */
uint32_t or_crc32_update(uint32_t crc, const void* data, size_t n) {
  if (!g_table_ready) build_table();
  const uint8_t* p = (const uint8_t*)data;
  crc = ~crc;
  for (size_t i = 0; i < n; ++i) crc = g_table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
  return ~crc;
}

/* include/gpucrsim/crc32.hpp:34 */
uint32_t or_crc32(const void* data, size_t n) { return or_crc32_update(0, data, n); }

/* GF(2) helpers for the combine (zlib's published crc32_combine algorithm:
 * multiply crc(A) by x^(8*len(B)) modulo the CRC polynomial, xor crc(B)). */
static uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
  }
  return p;
}

static uint32_t x8nmodp(uint64_t n) { /* x^(8n) mod P, reflected */
  uint32_t sq = 1u << 30;          /* x^1 */
  for (int i = 0; i < 3; ++i) sq = multmodp(sq, sq); /* x^8 */
  uint32_t p = 1u << 31;          /* x^0 */
  while (n) {
    if (n & 1) p = multmodp(sq, p);
    sq = multmodp(sq, sq);
    n >>= 1;
  }
  return p;
}

uint32_t or_crc32_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b) {
  return multmodp(x8nmodp(len_b), crc_a) ^ crc_b;
}

/* ---- SplitMix64 / fill / FNV ------------------------------------------ */

/* Rng::next: include/gpucrsim/rng.hpp:15-20 */
uint64_t or_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* include/gpucrsim/rng.hpp:35-40 */
uint64_t or_mix64(uint64_t a, uint64_t b) {
  uint64_t z = a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2));
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* fill_bytes: include/gpucrsim/rng.hpp:43-54 (little-endian 8-byte words,
 * the tail takes the low bytes of one more draw). */
void or_fill_bytes(uint64_t seed, uint8_t* out, size_t n) {
  uint64_t st = seed;
  size_t i = 0;
  while (i + 8 <= n) {
    uint64_t v = or_splitmix_next(&st);
    for (int k = 0; k < 8; ++k) out[i++] = (uint8_t)(v >> (8 * k));
  }
  if (i < n) {
    uint64_t v = or_splitmix_next(&st);
    for (int k = 0; i < n; ++k) out[i++] = (uint8_t)(v >> (8 * k));
  }
}

/* Bytes [off, off+n) of fill_bytes(seed) over a buffer of at least off+n
 * bytes (rng.hpp:43-54): byte i is byte i%8 of the (i/8+1)-th next(), i.e.
 * the SplitMix64 state seed + (i/8+1)*gamma (rng.hpp:15-20) -- random access
 * into a state the size of a GPU without generating its prefix. */
void or_fill_bytes_at(uint64_t seed, uint64_t off, uint8_t* out, size_t n) {
  for (size_t i = 0; i < n;) {
    const uint64_t w = (off + i) / 8;
    uint64_t st = seed + w * 0x9e3779b97f4a7c15ull;
    const uint64_t v = or_splitmix_next(&st);
    for (unsigned k = (unsigned)((off + i) % 8); k < 8 && i < n; ++k) out[i++] = (uint8_t)(v >> (8 * k));
  }
}

/* include/gpucrsim/rng.hpp:63-70 */
uint64_t or_fnv1a(const void* data, size_t n, uint64_t h) {
  const uint8_t* p = (const uint8_t*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* ---- chunk geometry ----------------------------------------------------- */

/* chunk_states sized ceil(size / chunk_size): include/gpucrsim/buffer.hpp:119 */
uint32_t or_chunk_count(uint64_t size, uint64_t chunk_size) {
  return (uint32_t)((size + chunk_size - 1) / chunk_size);
}

/* GpuBuffer::chunk_bytes: include/gpucrsim/buffer.hpp:46-49 (short tail). */
uint64_t or_chunk_bytes(uint64_t size, uint64_t chunk_size, uint32_t idx) {
  uint64_t start = (uint64_t)idx * chunk_size;
  uint64_t rest = size - start;
  return rest < chunk_size ? rest : chunk_size;
}

/* ---- O2 --------------------------------------------------------------- */

uint32_t or_chunk_digests(const uint8_t* content, uint64_t size, uint64_t chunk_size,
                          uint32_t* out) {
  uint32_t n = or_chunk_count(size, chunk_size);
  for (uint32_t c = 0; c < n; ++c)
    out[c] = or_crc32(content + (uint64_t)c * chunk_size, or_chunk_bytes(size, chunk_size, c));
  return n;
}

uint64_t or_dirty_flags(const uint32_t* prev, const uint32_t* cur, uint64_t n, int prev_valid,
                        uint8_t* flags) {
  uint64_t d = 0;
  for (uint64_t i = 0; i < n; ++i) {
    flags[i] = (uint8_t)(!prev_valid || prev[i] != cur[i]);
    d += flags[i];
  }
  return d;
}

void or_pack_bitmap(const uint8_t* flags, uint64_t n, uint32_t* bitmap) {
  uint64_t words = (n + 31) / 32;
  for (uint64_t w = 0; w < words; ++w) bitmap[w] = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (flags[i]) bitmap[i / 32] |= 1u << (i % 32);
}

uint32_t or_fold_digests(const uint32_t* digests, uint64_t size, uint64_t chunk_size) {
  uint32_t n = or_chunk_count(size, chunk_size);
  uint32_t crc = 0;
  for (uint32_t c = 0; c < n; ++c)
    crc = c == 0 ? digests[0]
                 : or_crc32_combine(crc, digests[c], or_chunk_bytes(size, chunk_size, c));
  return crc;
}

/* ---- O1 ----------------------------------------------------------------- */

/* scan_dedup: ok = crc32(content) == up.crc && host untouched
 * (include/gpucrsim/cr.hpp:419-421); no upstream => not a dedup candidate
 * (cr.hpp:390). */
int or_dedup_verdict(int has_upstream, uint32_t crc_now, uint32_t upstream_crc,
                     int host_untouched) {
  return has_upstream && crc_now == upstream_crc && host_untouched;
}

/* ---- POSD pack ---------------------------------------------------------- */

static void put_u32(uint8_t* p, uint32_t v) { memcpy(p, &v, 4); }
static void put_u64(uint8_t* p, uint64_t v) { memcpy(p, &v, 8); }
static uint32_t get_u32(const uint8_t* p) { uint32_t v; memcpy(&v, p, 4); return v; }
static uint64_t get_u64(const uint8_t* p) { uint64_t v; memcpy(&v, p, 8); return v; }
static uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

/* The payload a chunk contributes is the bytes chunk_copied() would copy into
 * captured_[h] (include/gpucrsim/cr.hpp:488-501), in (handle, chunk) order. */
uint64_t or_build_pack(const or_buffer_t* bufs, uint32_t nbufs, uint64_t chunk_size,
                       const uint8_t* flags, uint64_t epoch, uint32_t pack_flags,
                       uint8_t* out) {
  uint64_t n = 0, payload = 0, g = 0;
  for (uint32_t b = 0; b < nbufs; ++b) {
    uint32_t nc = or_chunk_count(bufs[b].size, chunk_size);
    for (uint32_t c = 0; c < nc; ++c, ++g)
      if (flags[g]) {
        ++n;
        payload += round_up(or_chunk_bytes(bufs[b].size, chunk_size, c), 16);
      }
  }
  uint64_t payload_off = round_up(OR_PACK_HEADER + OR_PACK_ENTRY * n, OR_PACK_ALIGN);
  uint64_t total = payload_off + payload;
  if (!out) return total;
  memset(out, 0, total);
  memcpy(out, "POSD", 4);
  put_u32(out + 4, 1);
  put_u64(out + 8, chunk_size);
  put_u32(out + 16, (uint32_t)n);
  put_u32(out + 20, pack_flags);
  put_u64(out + 24, payload_off);
  put_u64(out + 32, payload);
  put_u64(out + 40, epoch);
  put_u64(out + 48, total);
  uint64_t e = 0, off = 0;
  g = 0;
  for (uint32_t b = 0; b < nbufs; ++b) {
    uint32_t nc = or_chunk_count(bufs[b].size, chunk_size);
    for (uint32_t c = 0; c < nc; ++c, ++g) {
      if (!flags[g]) continue;
      uint64_t len = or_chunk_bytes(bufs[b].size, chunk_size, c);
      const uint8_t* src = bufs[b].content + (uint64_t)c * chunk_size;
      uint8_t* ent = out + OR_PACK_HEADER + OR_PACK_ENTRY * e;
      put_u64(ent + 0, bufs[b].handle);
      put_u64(ent + 8, off);
      put_u32(ent + 16, c);
      put_u32(ent + 20, (uint32_t)len);
      put_u32(ent + 24, or_crc32(src, len));
      memcpy(out + payload_off + off, src, len);
      off += round_up(len, 16);
      ++e;
    }
  }
  return total;
}

/* Restore-side scatter: Inline materialize writes bytes at their buffer
 * offsets (include/gpucrsim/cr.hpp:1026-1030 -> buffer.hpp:80-84, which
 * rejects out-of-range writes with InvalidLocator). */
int or_apply_pack(const uint8_t* pack, uint64_t pack_bytes, uint8_t* const* contents,
                  const uint64_t* handles, const uint64_t* sizes, uint32_t nbufs) {
  if (pack_bytes < OR_PACK_HEADER || memcmp(pack, "POSD", 4) != 0) return -1;
  uint64_t cs = get_u64(pack + 8);
  uint32_t n = get_u32(pack + 16);
  uint64_t payload_off = get_u64(pack + 24);
  uint64_t payload = get_u64(pack + 32);
  if (payload_off + payload > pack_bytes) return -1;
  if (OR_PACK_HEADER + (uint64_t)OR_PACK_ENTRY * n > payload_off) return -1;
  for (uint32_t e = 0; e < n; ++e) {
    const uint8_t* ent = pack + OR_PACK_HEADER + OR_PACK_ENTRY * e;
    uint64_t h = get_u64(ent), off = get_u64(ent + 8);
    uint32_t c = get_u32(ent + 16), len = get_u32(ent + 20);
    uint32_t b = 0;
    while (b < nbufs && handles[b] != h) ++b;
    if (b == nbufs) return -1;
    uint64_t dst = (uint64_t)c * cs;
    if (dst + len > sizes[b] || off + len > payload) return -1;
    memcpy(contents[b] + dst, pack + payload_off + off, len);
  }
  return 0;
}
