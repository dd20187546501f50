/*
 * posdump_oracle.h -- CPU restatement of the reference's buffer-dump path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (libposdump.so, the
 * Python package) links, imports or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it, and only as the checker or as the timed CPU baseline.
 *
 * Parity is pinned: every function here is checked by tests/test_oracle.py
 * against golden vectors produced by the reference itself (oracle/_ref, built
 * from /root/reference/proj/include by oracle/Makefile; fixtures committed in
 * tests/golden/ by tests/golden/make_golden.py) and against the reference's
 * own known-answer tests (proj/tests/test_memory.cpp:10-17, :89-99).
 *
 * Citations are path:line relative to /root/reference/proj.
 */
#ifndef POSDUMP_ORACLE_H
#define POSDUMP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- L0 primitives ---------------------------------------------------- */
/* zlib CRC-32: include/gpucrsim/crc32.hpp:12-34 */
uint32_t or_crc32_update(uint32_t crc, const void* data, size_t n);
uint32_t or_crc32(const void* data, size_t n);
/* zlib crc32_combine semantics: crc(A||B) from crc(A), crc(B), len(B). */
uint32_t or_crc32_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b);

/* SplitMix64 / mix64 / fill_bytes / fnv1a: include/gpucrsim/rng.hpp:11-77 */
uint64_t or_splitmix_next(uint64_t* state);
uint64_t or_mix64(uint64_t a, uint64_t b);
void or_fill_bytes(uint64_t seed, uint8_t* out, size_t n);
/* bytes [off, off+n) of fill_bytes(seed) (random access by SplitMix64 state) */
void or_fill_bytes_at(uint64_t seed, uint64_t off, uint8_t* out, size_t n);
uint64_t or_fnv1a(const void* data, size_t n, uint64_t h);

/* ---- chunk geometry: include/gpucrsim/buffer.hpp:44-49, :119 ----------- */
uint32_t or_chunk_count(uint64_t size, uint64_t chunk_size);
uint64_t or_chunk_bytes(uint64_t size, uint64_t chunk_size, uint32_t idx);

/* ---- O2: per-chunk digests and the dirty bitmap ------------------------ */
/* digest[c] = crc32(content + c*cs, chunk_bytes(c))  (the per-chunk
 * form of crc32 applied at cr.hpp:419 / process.hpp:518).  Returns #chunks. */
uint32_t or_chunk_digests(const uint8_t* content, uint64_t size, uint64_t chunk_size,
                          uint32_t* out);
/* flags[i] = !prev_valid || prev[i] != cur[i].  Returns #dirty. */
uint64_t or_dirty_flags(const uint32_t* prev, const uint32_t* cur, uint64_t n, int prev_valid,
                        uint8_t* flags);
/* bitmap word w bit b  <=>  flags[32w+b]. */
void or_pack_bitmap(const uint8_t* flags, uint64_t n, uint32_t* bitmap);
/* whole-buffer CRC folded from chunk digests (== crc32(content, size)). */
uint32_t or_fold_digests(const uint32_t* digests, uint64_t size, uint64_t chunk_size);

/* ---- O1 verdict: cr.hpp:416-425 (scan), cr.hpp:720-721 (record kind) ---- */
int or_dedup_verdict(int has_upstream, uint32_t crc_now, uint32_t upstream_crc,
                     int host_untouched);

/* ---- POSD packed delta (O3 cache format) ------- */
#define OR_PACK_HEADER 64u
#define OR_PACK_ENTRY 32u
#define OR_PACK_ALIGN 256u
typedef struct {
  uint64_t handle;
  const uint8_t* content; /* host copy of the buffer's bytes */
  uint64_t size;
} or_buffer_t;
/* Pack the chunks with flags[g] != 0 (g = global chunk index in buffer
 * order) in (handle, chunk) order.  `out` may be NULL to size only.
 * Returns the pack size in bytes. */
uint64_t or_build_pack(const or_buffer_t* bufs, uint32_t nbufs, uint64_t chunk_size,
                       const uint8_t* flags, uint64_t epoch, uint32_t pack_flags,
                       uint8_t* out);
/* Apply a pack onto host copies of the buffers (restore-side scatter,
 * cr.hpp:1026-1030 write_content semantics).  Returns 0 or -1 if malformed. */
int or_apply_pack(const uint8_t* pack, uint64_t pack_bytes, uint8_t* const* contents,
                  const uint64_t* handles, const uint64_t* sizes, uint32_t nbufs);

#ifdef __cplusplus
}
#endif
#endif
