// kernels.cuh -- sm_100a kernels of the buffer-dump hot path.
//
//   k_hash_chunks<MODE,D2> O2 digest + dirty flags (kModeHash; D2: plus the
//                        opt-in second digest), digest + gather
//                        into a POSD pack (kModeCopy: CoW staging), or digest
//                        of chunks already gathered into a pack (kModeCached:
//                        the STW delta is a pure bulk gather; its hashing
//                        runs after the stop)
//   k_buffer_crc         O1: whole-buffer CRC folded from chunk digests + verdict
//   k_note_upstream      note_h2d_provenance's CRC, folded on the device
//   k_scan_tiles         direct pre-copy: ballot/prefix-sum compaction of the
//                        shipped chunks into copy-engine runs + a POSD index
//                        pack, decoupled look-back over many CTAs
//   k_pack_scan          pack modes: one-CTA compaction (+ fused O1) of the
//                        (handle, chunk)-ordered pack layout and its copy items
//   k_copy_bulk          TMA bulk copies (cp.async.bulk) staged through smem
//   k_copy_simt          16-B vector / byte copies (unaligned items)
//   k_ship_runs          host leg, short runs: SM stores into the mapped image
//   k_pack_items         restore: POSD entries -> scatter copy items
//   k_stage_in           SM loads of the staged STW delta layout
//   k_fill               fill_bytes(seed) (rng.hpp:43-54) into device memory
//   k_clear_written      finalize's written_since_ckpt reset
//
// See DESIGN.md for the data layout and the roofline of each kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "crc_math.h"

namespace posdump {

// ---------------------------------------------------------------------------
// Shared device structures (mirrored on the host in posdump.cu).

struct DevBuf {              // one registered allocation (GpuBuffer, buffer.hpp:27-41)
  uint64_t ptr;              // device address
  uint64_t size;             // bytes
  uint64_t handle;           // BufferHandle
  uint64_t chunk_base;       // global index of chunk 0
  uint32_t nchunks;          // ceil(size / chunk_size) (buffer.hpp:119)
  uint32_t k_tail;           // zeros_crc(last chunk length)
  uint32_t x8_tail;          // x^(8 * last chunk length) mod P
  uint32_t flags;            // kBuf* bits
  uint32_t upstream_crc;     // Upstream::crc
  uint32_t pad;
  uint64_t image;            // device-visible address of the buffer's host image (0: none)
};
static_assert(sizeof(DevBuf) == 64, "DevBuf layout");

enum : uint32_t {
  kBufHasUpstream = 1u,
  kBufHostUntouched = 2u,
  kBufWrittenSinceCkpt = 8u,
  kBufStaged = 16u,  // CoW-staged this epoch: its snapshot is the staged pack
  kBufFresh = 32u,   // joined the snapshot mid-session (cr.hpp:301-306): every chunk dirty until committed
};

struct CopyItem {            // one contiguous copy: chunk -> pack, or pack -> chunk
  uint64_t src;
  uint64_t dst;
  uint64_t len;              // payload bytes
  uint64_t padded;           // bytes to write at dst (len rounded up to 16, zero-filled)
};

// POSD pack layout.
constexpr uint32_t kPackHeader = 64;
constexpr uint32_t kPackEntry = 32;
constexpr uint32_t kPackAlign = 256;
constexpr uint32_t kPackMagic = 0x44534F50u;  // "POSD"
constexpr uint32_t kPackFlagDelta = 1u;        // STW delta pack
constexpr uint32_t kPackFlagDirect = 2u;       // index only: payload went straight to the host image
constexpr uint32_t kPackFlagStaged = 4u;       // CoW staging pack (stage_buffers)

struct HashParams {
  const DevBuf* bufs;
  const uint2* chunk_map;    // [n_chunks] {buffer index, chunk index}
  uint64_t n_items;          // chunks (hash mode) or work items (COPY mode)
  uint64_t chunk_size;
  uint32_t k_full;           // zeros_crc(chunk_size)
  uint32_t pad0;
  const uint32_t* tables;    // [7][1024]: Z^512, Z^4, Z^16, Z^32, Z^64, Z^128, Z^256
  const uint32_t* xinv;      // [512]: x^(-8n) mod P
  uint32_t* digest_cur;
  const uint32_t* digest_prev;
  uint8_t* flags;
  uint32_t* bitmap;
  int prev_valid;
  int skip_clean;            // buffer-level O2 first (cr.hpp:396-401): !written_since_ckpt => not hashed
  // COPY mode
  const uint4* work;         // {g, entry, dst_off lo, dst_off hi}
  uint8_t* pack;             // pack base
  uint64_t payload_off;      // payload offset within the pack
  // Segmented chunks (nseg > 1, divides the warps per CTA): warp unit =
  // (item, segment of seg_bytes); a CTA-local group of warps folds them.
  uint32_t nseg;
  uint32_t seg_bytes;
  uint64_t item_base;        // hash mode: first global chunk of this launch
  const uint32_t* xseg;      // [32]: x^(8 k seg_bytes) mod P
  const uint32_t* lastseg;   // [nbufs]: x^(8 * length of the tail chunk's last segment)
  // Second, non-linear chunk digest for the O2 compare (kModeHash, opt-in):
  // a chunk counts as clean only if its CRC-32 AND this digest are unchanged
  uint32_t* digest2_cur;
  const uint32_t* digest2_prev;
  int d2_prev_valid;
};

// The second digest: a sum over the chunk's 16-B vectors of a multiply-xorshift
// mix of the vector and its position (its 16-B index from the chunk's aligned
// base).  Not GF(2)-linear, so a change that leaves the CRC-32 alone (a
// multiple of its polynomial) changes it with probability 1 - 2^-32.
__device__ __forceinline__ uint32_t d2_mix(uint4 v, uint32_t q) {
  // two multiply-adds (4 was 4 % slower on the wave: profiles/r2/digest2.txt)
  const uint32_t a = (v.x ^ (q * 0x9E3779B1u)) * 0x85EBCA77u + v.y;
  const uint32_t b = (v.z ^ __funnelshift_l(a, a, 13)) * 0xC2B2AE3Du + v.w;
  return b ^ (b >> 15);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Hash kernel geometry.
constexpr int kHashThreads = 512;            // 16 warps, 1 CTA per SM
constexpr int kStepBytes = 512;              // one warp step: 32 lanes x 16 B
constexpr int kUnroll = 6;                   // warp steps per batch (3 KiB per warp)
constexpr uint32_t kRepTableBytes = 131072;  // lane-replicated Z^512: 4 x 256 x 32 lanes x 4 B
constexpr uint32_t kSmallTablesBytes = 6 * 4096;
// The replicated table sits at ABSOLUTE shared address 0x10000, so the PRMT
// that extracts a state byte also supplies the table base (byte 2 = 1) and no
// per-lookup add is needed; the small tables sit at the start of the dynamic
// window (which begins at the ~1 KiB reserved offset).
constexpr uint32_t kRepAbs = 0x10000;
constexpr uint32_t kHashSmem = 0x30000;

// ---------------------------------------------------------------------------
// Load helpers.

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Lane's 16 bytes of warp step `blk` of a region that starts at the 16-B
// aligned address a0, keeping only bytes in [lead, end) (others read as 0).
__device__ __forceinline__ uint4 load_masked(uint64_t a0, uint64_t blk, int lane, uint64_t lead,
                                             uint64_t end) {
  uint64_t off = blk * kStepBytes + (uint64_t)lane * 16;
  if (off >= lead && off + 16 <= end) return ldg_stream((const void*)(a0 + off));
  uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
  if (off + 16 > lead && off < end) {
    const uint8_t* p = (const uint8_t*)(a0 + off);
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      uint64_t o = off + b;
      uint32_t byte = (o >= lead && o < end) ? (uint32_t)p[b] : 0u;
      uint32_t sh = 8 * (b & 3);
      if (b < 4) w0 |= byte << sh;
      else if (b < 8) w1 |= byte << sh;
      else if (b < 12) w2 |= byte << sh;
      else w3 |= byte << sh;
    }
  }
  return make_uint4(w0, w1, w2, w3);
}

// TMA / mbarrier helpers (also used by the bulk copy engine below).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------------------
// CRC advance operators.
//
// Z^512 runs out of a lane-replicated table: entry e of slice k for lane l
// lives at byte (k>>1)*65536 + e*256 + (k&1)*128 + l*4, so every lane hits its
// own bank (conflict-free LDS) and one PRMT builds the address:
// __byte_perm(x, lane*4, 0x55k4) = lane*4 + byte_k(x)*256.

template <int IMM>
__device__ __forceinline__ uint32_t lds_abs(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(IMM));
  return v;
}

// lsel = lane*4 | kRepAbs: __byte_perm(x, lsel, 0x76k4) = kRepAbs + byte_k(x)*256 + lane*4.
__device__ __forceinline__ uint32_t adv512(uint32_t lsel, uint32_t x) {
  uint32_t o0 = __byte_perm(x, lsel, 0x7604);
  uint32_t o1 = __byte_perm(x, lsel, 0x7614);
  uint32_t o2 = __byte_perm(x, lsel, 0x7624);
  uint32_t o3 = __byte_perm(x, lsel, 0x7634);
  return lds_abs<0>(o0) ^ lds_abs<128>(o1) ^ lds_abs<65536>(o2) ^ lds_abs<65536 + 128>(o3);
}

__device__ __forceinline__ uint32_t adv_small(const uint32_t* t, uint32_t x) {
  return t[x & 255] ^ t[256 + ((x >> 8) & 255)] ^ t[512 + ((x >> 16) & 255)] ^ t[768 + (x >> 24)];
}

// ---------------------------------------------------------------------------
// One warp computes crc32 of [src, src+len) (len > 0).  Lane l owns 4
// streams: word j of its 16 B in every 512-B warp step.  A stream's register
// r advances r <- Z^512(r ^ w) from step to step.  In the last step the lane
// merges its 4 streams with Z^4, the warp folds lanes with Z^16..Z^256
// (shuffle tree), and the zero padding up to the step boundary is undone
// with x^(-8 pad).  Leading bytes below the 16-B aligned base read as zero,
// which leaves a register that starts at 0 unchanged.  COPY: every loaded
// vector is also stored at dst (only when src is 16-B aligned).
template <bool COPY, bool D2 = false>
__device__ __forceinline__ uint32_t warp_crc32(const uint32_t* small, const uint32_t* xinv, uint32_t lsel, int lane,
                                               uint64_t src, uint64_t len, uint32_t k_len, uint8_t* dst,
                                               uint32_t q0 = 0, uint32_t* h2 = nullptr) {
  const uint64_t a0 = src & ~15ull;
  const uint64_t lead = src - a0;
  const uint64_t end = lead + len;
  const uint64_t nblk = (end + kStepBytes - 1) / kStepBytes;
  const bool vec_copy = COPY && lead == 0;
  const uint4* base = reinterpret_cast<const uint4*>(a0) + lane;
  uint4* dbase = reinterpret_cast<uint4*>(dst) + lane;

  uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  uint32_t hs = 0;  // D2: this lane's share of the second digest
  const uint32_t qlane = q0 + (uint32_t)lane;
  uint64_t blk = 0;
  if (lead != 0 && nblk > 1) {  // first step straddles the aligned base
    uint4 v = load_masked(a0, 0, lane, lead, end);
    if (D2) hs += d2_mix(v, qlane);
    c0 = adv512(lsel, c0 ^ v.x);
    c1 = adv512(lsel, c1 ^ v.y);
    c2 = adv512(lsel, c2 ^ v.z);
    c3 = adv512(lsel, c3 ^ v.w);
    blk = 1;
  }
  const uint64_t full_end = nblk - 1;  // steps [blk, full_end) are fully inside
  // Software-pipelined batches of kUnroll steps, ping-ponging between two
  // register buffers: the next batch's loads are in flight while this
  // batch's lookups run.  (Measured and dropped: an L2 bulk prefetch ahead of
  // every warp, a rolling ring, a third TMA-filled shared-memory stage -- equal
  // or slower, profiles/r1/tune_sweep1.txt.)
  auto load_batch = [&](uint4 (&buf)[kUnroll], uint64_t at) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) buf[u] = ldg_stream(base + (at + u) * 32);
  };
  auto run_batch = [&](const uint4 (&buf)[kUnroll], uint64_t at) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (vec_copy) stg_stream(dbase + (at + u) * 32, buf[u]);
      if (D2) hs += d2_mix(buf[u], qlane + (uint32_t)(at + u) * 32u);
      c0 = adv512(lsel, c0 ^ buf[u].x);
      c1 = adv512(lsel, c1 ^ buf[u].y);
      c2 = adv512(lsel, c2 ^ buf[u].z);
      c3 = adv512(lsel, c3 ^ buf[u].w);
    }
  };
  if (blk + kUnroll <= full_end) {
    uint4 bufA[kUnroll], bufB[kUnroll];
    load_batch(bufA, blk);
    for (;;) {
      const bool moreB = blk + 2 * kUnroll <= full_end;
      if (moreB) load_batch(bufB, blk + kUnroll);
      run_batch(bufA, blk);
      blk += kUnroll;
      if (!moreB) break;
      const bool moreA = blk + 2 * kUnroll <= full_end;
      if (moreA) load_batch(bufA, blk + kUnroll);
      run_batch(bufB, blk);
      blk += kUnroll;
      if (!moreA) break;
    }
  }
  for (; blk < full_end; ++blk) {
    uint4 v = ldg_stream(base + blk * 32);
    if (vec_copy) stg_stream(dbase + blk * 32, v);
    if (D2) hs += d2_mix(v, qlane + (uint32_t)blk * 32u);
    c0 = adv512(lsel, c0 ^ v.x);
    c1 = adv512(lsel, c1 ^ v.y);
    c2 = adv512(lsel, c2 ^ v.z);
    c3 = adv512(lsel, c3 ^ v.w);
  }
  // Last (partial) step: bytes past `end` read as zero.
  uint4 v = load_masked(a0, full_end, lane, lead, end);
  if (D2) {
    hs += d2_mix(v, qlane + (uint32_t)full_end * 32u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
    *h2 = hs;
  }
  if (vec_copy) {
    uint64_t off = full_end * kStepBytes + (uint64_t)lane * 16;
    if (off < end) stg_stream(dbase + full_end * 32, v);  // zero tail == POSD padding
  }
  const uint32_t* t4 = small;
  uint32_t r = c0;
  r = adv_small(t4, r ^ v.x) ^ c1;
  r = adv_small(t4, r ^ v.y) ^ c2;
  r = adv_small(t4, r ^ v.z) ^ c3;
  r = adv_small(t4, r ^ v.w);  // lane register at step offset 16(l+1)
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    uint32_t t = adv_small(small + 1024 * (k + 1), r);  // Z^(16 << k)
    uint32_t u = __shfl_up_sync(0xffffffffu, t, 1 << k);
    const int m = (2 << k) - 1;
    if ((lane & m) == m) r ^= u;
  }
  // lane 31: register at nblk*512; undo the zero padding.
  uint32_t pad = (uint32_t)(nblk * kStepBytes - end);
  uint32_t raw = pad ? multmodp(__ldg(xinv + pad), r) : r;
  uint32_t crc = raw ^ k_len;
  crc = __shfl_sync(0xffffffffu, crc, 31);
  if (COPY && !vec_copy) {  // unaligned source: plain byte copy, zero padding
    uint64_t padded = (len + 15) & ~15ull;
    for (uint64_t i = lane; i < padded; i += 32)
      dst[i] = i < len ? *reinterpret_cast<const uint8_t*>(src + i) : 0;
  }
  return crc;
}

// Table prologue: one TMA bulk copy brings the 24 KiB of small tables and the
// 4 KiB Z^512 source into shared memory (the per-thread __ldg loop it
// replaces was 27 % of a 100 MB launch's stall samples: 76 dependent L2
// round trips per thread), then the lane-replicated table is built from
// shared memory.  The source sits in the gap between the small tables and
// the replicated table at 0x10000.
constexpr uint32_t kRepSrcOff = kSmallTablesBytes;  // 4 KiB source, after the small tables

// Split in two so that a kernel can overlap its own first global loads with
// the tables' flight: issue (thread 0 starts the bulk copy) ... finish (wait,
// replicate, block barrier).
__device__ __forceinline__ void load_hash_tables_issue(uint8_t* smem, const uint32_t* tables) {
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if (sbase + kSmallTablesBytes + 4096 + 64 > kRepAbs) __trap();  // layout assumption (reserved smem < 36 KiB)
  uint32_t* src = reinterpret_cast<uint32_t*>(smem + kRepSrcOff);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kRepSrcOff + 4096);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, kSmallTablesBytes + 4096);
    bulk_g2s(smem, tables + 1024, kSmallTablesBytes, bar);  // Z^4, Z^16..Z^256
    bulk_g2s(src, tables, 4096, bar);                        // Z^512
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
}

__device__ __forceinline__ void load_hash_tables_finish(uint8_t* smem) {
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  uint32_t* rep = reinterpret_cast<uint32_t*>(smem + (kRepAbs - sbase));
  uint32_t* src = reinterpret_cast<uint32_t*>(smem + kRepSrcOff);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kRepSrcOff + 4096);
  mbar_wait(bar, 0);
  // 4 consecutive lane slots of one entry hold the same word: 16-B stores
  for (int q = threadIdx.x; q < 32768 / 4; q += blockDim.x) {
    const int i = 4 * q;
    const int t2 = (i >> 5) & 1, e = (i >> 6) & 255, pair = i >> 14;
    const uint32_t v = src[(pair * 2 + t2) * 256 + e];
    reinterpret_cast<uint4*>(rep)[q] = make_uint4(v, v, v, v);
  }
  __syncthreads();
}

enum : int { kModeHash = 0, kModeCopy = 1, kModeCached = 2 };

// Phase stamps of k_hash_chunks for tools/hash_micro.cu (compiled there only):
// per (CTA, warp), globaltimer at entry, tables ready, chunk record read,
// CRC done, digest published -- for the warp's first item.
#ifdef POS_HASH_PROF
__device__ unsigned long long g_hash_prof[1024][16][5];
#define POS_PROF(k, first)                                                              \
  do {                                                                                  \
    if ((first) && (threadIdx.x & 31) == 0 && blockIdx.x < 1024) {                      \
      unsigned long long t_;                                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
      g_hash_prof[blockIdx.x][threadIdx.x >> 5][k] = t_;                                \
    }                                                                                   \
  } while (0)
#else
#define POS_PROF(k, first) \
  do {                     \
  } while (0)
#endif

// kModeHash: every chunk -> digest, dirty flag, bitmap bit.
// kModeCopy: every work item -> digest + pack entry + payload (hash while copying).
// kModeCached: every work item's payload, already in the pack -> digest + entry.
// One CTA of kHashThreads per SM (the replicated table takes 192 KiB of
// shared memory).  <= 96 registers (batches of 6 steps) leave a quarter of
// the register file to other CTAs on the same SM -- the application's and
// the dump's own scan / ship / copy kernels.  Measured on a config-5 wave
// (7.5 GB): 8 steps / 120 registers 1.203 ms, 6 / 96 1.22 ms; the
// application's optimizer-tail window launched beside the dump's first
// waves: 17x -> 1.8x slower than alone (profiles/r2/hash_regs.txt).
template <int MODE, bool D2 = false>
__global__ void __maxnreg__(96) k_hash_chunks(HashParams p) {
  constexpr int kThreads = kHashThreads;
  constexpr bool COPY = MODE == kModeCopy;
  constexpr bool WORK = MODE != kModeHash;
  extern __shared__ __align__(128) uint8_t smem[];
  POS_PROF(0, true);
  load_hash_tables_issue(smem, p.tables);
  if (MODE == kModeHash) {
    // Warm this warp's first chunk while the tables fly: its record (chunk
    // map -> buffer: two dependent DRAM loads, ~1.2 us) and its first 4 KiB
    // (one L2 prefetch per lane).  Measured: the record phase was 1.2 us of a
    // 100 MB launch's ~27 us, serial after the 1.9 us prologue.
    constexpr int W0 = kThreads / 32;
    const uint32_t warp0 = threadIdx.x >> 5;
    uint64_t it0;
    if (p.nseg == 1) {
      it0 = (uint64_t)warp0 * gridDim.x + blockIdx.x;
    } else {
      const uint32_t grp = warp0 / p.nseg;
      it0 = ((uint64_t)grp * gridDim.x + blockIdx.x) * p.nseg + warp0 % p.nseg;
    }
    if (it0 < p.n_items * p.nseg && (W0 % p.nseg) == 0) {
      const uint64_t g0 = p.item_base + it0 / p.nseg;
      const uint2 cm0 = p.chunk_map[g0];
      const DevBuf& b0 = p.bufs[cm0.x];
      const uint64_t off0 = (uint64_t)cm0.y * p.chunk_size + (it0 % p.nseg) * p.seg_bytes;
      const uint64_t pf = (threadIdx.x & 31) * 128ull;
      if (off0 + pf < b0.size)  // stays inside the buffer
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b0.ptr + off0 + pf));
    }
  }
  load_hash_tables_finish(smem);
  POS_PROF(1, true);
  const uint32_t* small = reinterpret_cast<const uint32_t*>(smem);
  const int lane = threadIdx.x & 31;
  const uint32_t lsel = (uint32_t)lane * 4 | kRepAbs;
  // nseg == 1: item i goes to CTA i % grid, warp (i / grid) % W, so a short
  // list still spreads over every SM.  nseg > 1: the nseg segments of a chunk
  // go to nseg consecutive warps of ONE CTA (a "group"), which fold their
  // segment registers through shared memory behind a named barrier; groups
  // are dealt round-robin over CTAs.
  constexpr int W = kThreads / 32;
  __shared__ uint32_t s_seg[2][W];
  __shared__ uint32_t s_seg2[D2 ? 2 : 1][D2 ? W : 1];  // D2: the segments' second-digest sums
  const int warp = threadIdx.x >> 5;
  const uint32_t nseg = p.nseg;
  const uint32_t G = W / nseg;                       // groups per CTA
  const uint32_t my_group = warp / nseg, my_seg = warp % nseg;
  const uint64_t n_units = p.n_items * nseg;
  uint64_t it, stride;
  if (nseg == 1) {
    it = (uint64_t)warp * gridDim.x + blockIdx.x;
    stride = (uint64_t)gridDim.x * W;
  } else {
    it = ((uint64_t)my_group * gridDim.x + blockIdx.x) * nseg + my_seg;
    stride = (uint64_t)gridDim.x * G * nseg;
  }
  // kModeHash: the next item's chunk-map entry is loaded one item ahead (its
  // DRAM latency hides under the current chunk instead of heading the next).
  uint2 cm_next = make_uint2(0, 0);
  if (!WORK && it < n_units) cm_next = p.chunk_map[p.item_base + (nseg == 1 ? it : it / nseg)];
  for (uint32_t round = 0; it < n_units; it += stride, ++round) {
    const uint64_t item = nseg == 1 ? it : it / nseg;
    const uint32_t seg = nseg == 1 ? 0u : my_seg;
    uint64_t g, dst_off = 0;
    uint32_t entry = 0;
    uint2 cm;
    if (WORK) {
      uint4 w = p.work[item];
      g = w.x;
      entry = w.y;
      dst_off = (uint64_t)w.z | ((uint64_t)w.w << 32);
      cm = p.chunk_map[g];
    } else {
      g = p.item_base + item;
      cm = cm_next;
      if (it + stride < n_units) cm_next = p.chunk_map[p.item_base + (nseg == 1 ? it + stride : (it + stride) / nseg)];
    }
    const DevBuf& b = p.bufs[cm.x];
    // plan_precopy's O2 branch (cr.hpp:396-401): a buffer nothing wrote since
    // the last checkpoint is captured without a copy -- and, trusting the
    // bit, without a hash: its digests carry over, nothing ships.  (Every
    // warp of a segment group takes the same branch: no barrier is skipped
    // by half a group.)
    if (!WORK && p.skip_clean && p.prev_valid &&
        !(b.flags & (kBufWrittenSinceCkpt | kBufFresh | kBufStaged))) {
      if (lane == 31 && (nseg == 1 || my_seg == 0)) {
        p.digest_cur[g] = p.digest_prev[g];
        if (D2) p.digest2_cur[g] = p.digest2_prev[g];
        if (p.flags) p.flags[g] = 0;
      }
      continue;
    }
    const uint64_t start = (uint64_t)cm.y * p.chunk_size;
    const bool last = cm.y + 1 == b.nchunks;
    const uint64_t len = last ? b.size - start : p.chunk_size;
    const uint32_t k_len = last ? b.k_tail : p.k_full;
    uint8_t* dst = COPY ? p.pack + p.payload_off + dst_off : nullptr;
    // kModeCached reads the gathered copy (16-B aligned) instead of the live buffer.
    const uint64_t src = MODE == kModeCached ? (uint64_t)(p.pack + p.payload_off + dst_off) : b.ptr + start;
    uint32_t crc;
    // Whole chunk (nseg == 1), or this warp's segment: raw register (init 0)
    // at the segment end.
    const uint64_t lo = (uint64_t)seg * p.seg_bytes;
    const uint64_t n = p.nseg == 1 ? len : (lo >= len ? 0 : (len - lo < p.seg_bytes ? len - lo : p.seg_bytes));
    POS_PROF(2, round == 0);
    uint32_t h2 = 0;  // D2: the second digest of this warp's bytes
    const uint32_t q0 = D2 ? (uint32_t)((((src + lo) & ~15ull) - (src & ~15ull)) >> 4) : 0u;
    const uint32_t r = n ? warp_crc32<COPY, D2>(small, p.xinv, lsel, lane, src + lo, n, p.nseg == 1 ? k_len : 0u,
                                                COPY ? dst + lo : nullptr, q0, &h2)
                         : 0u;
    POS_PROF(3, round == 0);
    if (nseg == 1) {
      crc = r;
    } else {
      // raw(chunk) = XOR_s Z^(len - end_s)(raw_s); segments past the tail are empty.
      uint32_t* slot = s_seg[round & 1] + my_group * nseg;
      uint32_t* slot2 = D2 ? s_seg2[round & 1] + my_group * nseg : nullptr;
      if (lane == 31) {
        slot[seg] = r;
        if (D2) slot2[seg] = h2;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + my_group), "r"(nseg * 32) : "memory");
      if (seg != 0) continue;  // the group's first warp folds and publishes
      if (D2) {  // segments past the tail are empty: their sums are 0
        h2 = 0;
        for (uint32_t k = 0; k < nseg; ++k) h2 += slot2[k];
      }
      const uint32_t m = (uint32_t)((len - 1) / p.seg_bytes);  // last non-empty segment
      const uint32_t xl = len == p.chunk_size ? p.xseg[1] : p.lastseg[cm.x];
      uint32_t v = 0;
      if ((uint32_t)lane <= m) {
        v = slot[lane];
        if ((uint32_t)lane < m) v = multmodp(p.xseg[m - 1 - lane], multmodp(xl, v));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
      crc = v ^ k_len;
    }
    if (lane == 31) {
      // a CoW-staged buffer keeps the digest of its staged snapshot (pre-copy hash only)
      const bool staged = !WORK && p.flags && (b.flags & kBufStaged);
      if (!staged) {
        p.digest_cur[g] = crc;
        if (D2) p.digest2_cur[g] = h2;
      }
      if (WORK) {
        uint4* e = reinterpret_cast<uint4*>(p.pack + kPackHeader + (uint64_t)entry * kPackEntry);
        e[0] = make_uint4((uint32_t)b.handle, (uint32_t)(b.handle >> 32), (uint32_t)dst_off,
                          (uint32_t)(dst_off >> 32));
        e[1] = make_uint4(cm.y, (uint32_t)len, crc, 0u);
      } else if (staged) {
        p.flags[g] = 0;  // its snapshot is in the staging pack: nothing to ship
      } else if (p.flags) {
        const bool dirty = !p.prev_valid || (b.flags & kBufFresh) || p.digest_prev[g] != crc ||
                           (D2 && p.d2_prev_valid && p.digest2_prev[g] != h2);
        p.flags[g] = dirty;
        if (dirty && p.bitmap) atomicOr(p.bitmap + (g >> 5), 1u << (g & 31));
      }
    }
    POS_PROF(4, round == 0);
  }
}

// ---------------------------------------------------------------------------
// Whole-buffer CRC by one warp (O1, note_h2d_provenance): lanes fold
// right-aligned runs of `per` full chunks with Z^chunk_size (table tz in
// smem) -- only a prefix of lanes can be short, and a short run's left
// neighbours are empty (crc 0), so every right operand of the lane tree is a
// whole subtree of per * 2^k chunks and is shifted in with x^(8 cs per 2^k)
// (xfold = x^(8 cs per), squared per level).  The last (possibly short)
// chunk is appended with x^(8 tail).  Returns the crc on every lane.
__device__ __forceinline__ uint32_t warp_fold_buffer(const DevBuf& b, const uint32_t* digests,
                                                     const uint32_t* tz, uint32_t xfold, int lane) {
  const uint32_t* d = digests + b.chunk_base;
  const uint32_t nfull = b.nchunks - 1;
  if (nfull == 0) return d[0];
  uint32_t crc = 0;
  if (nfull <= 32) {
    // Short buffer: one coalesced load, then a shuffle-fed Z^cs chain
    // (~40 cycles per chunk; the lane tree's multmodp levels cost more).
    const uint32_t v = (uint32_t)lane < nfull ? d[lane] : 0u;
    for (uint32_t c = 0; c < nfull; ++c) crc = adv_small(tz, crc) ^ __shfl_sync(0xffffffffu, v, c);
  } else {
    const uint32_t per = (nfull + 31) / 32;
    const int64_t hi = (int64_t)nfull - (int64_t)per * (31 - lane);
    const int64_t lo = hi - per;
#pragma unroll 4
    for (int64_t c = lo < 0 ? 0 : lo; c < hi; ++c) crc = adv_small(tz, crc) ^ d[c];
    uint32_t x = xfold;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t o = __shfl_down_sync(0xffffffffu, crc, 1 << k);
      if ((lane & ((2 << k) - 1)) == 0) crc = multmodp(x, crc) ^ o;
      x = multmodp(x, x);
    }
    crc = __shfl_sync(0xffffffffu, crc, 0);
  }
  return multmodp(b.x8_tail, crc) ^ d[nfull];
}

// finalize_image clears written_since_ckpt of every buffer (cr.hpp:745).
__global__ void k_clear_written(DevBuf* bufs, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) bufs[i].flags &= ~kBufWrittenSinceCkpt;
}

// O1: whole-buffer CRC (crc32_combine fold of the chunk digests, one warp
// per buffer), then the scan_dedup verdict (cr.hpp:419-421) and the
// finalize_image gate (!dirty_set_, cr.hpp:720).
__global__ void k_buffer_crc(const DevBuf* bufs, uint32_t nbufs, const uint32_t* digests,
                             const uint32_t* tcs, const uint32_t* xfold, const uint8_t* dag_dirty, int dedup,
                             int all, uint32_t* crc_out, uint8_t* verdict_out) {
  __shared__ uint32_t t[1024];  // Z^chunk_size
  for (int q = threadIdx.x; q < 1024; q += blockDim.x) t[q] = __ldg(tcs + q);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= nbufs) return;
  const DevBuf b = bufs[i];
  const bool candidate = dedup && (b.flags & kBufHasUpstream);
  if (!all && !candidate) {  // verdict only: no provenance, no CRC needed (cr.hpp:390)
    if (lane == 0) verdict_out[i] = 0;
    return;
  }
  const uint32_t crc = warp_fold_buffer(b, digests, t, xfold[i], lane);
  if (lane == 0) {
    crc_out[i] = crc;
    verdict_out[i] = candidate && crc == b.upstream_crc && (b.flags & kBufHostUntouched) && !dag_dirty[i];
  }
}

// note_h2d_provenance (process.hpp:505-522) on the device: after a
// whole-buffer H2D (whole != 0) the buffer's chunk digests (just hashed into
// `digests`) fold into Upstream::crc, which lands in the device buffer table
// and in a mapped host mirror; a partial H2D drops the provenance
// (process.hpp:510-513).  Either way the buffer is written_since_ckpt.
// One warp.
__global__ void k_note_upstream(DevBuf* bufs, uint32_t i, const uint32_t* digests, const uint32_t* tcs,
                                const uint32_t* xfold, int whole, volatile uint32_t* mirror) {
  __shared__ uint32_t tz[1024];
  for (int q = threadIdx.x; q < 1024; q += blockDim.x) tz[q] = __ldg(tcs + q);
  __syncwarp();
  const int lane = threadIdx.x & 31;
  DevBuf& b = bufs[i];
  if (!whole) {
    if (lane == 0) b.flags = (b.flags & ~(kBufHasUpstream | kBufHostUntouched)) | kBufWrittenSinceCkpt;
    return;
  }
  const DevBuf snap = b;
  const uint32_t crc = warp_fold_buffer(snap, digests, tz, xfold[i], lane);
  if (lane == 0) {
    b.upstream_crc = crc;
    b.flags |= kBufHasUpstream | kBufHostUntouched | kBufWrittenSinceCkpt;
    mirror[i] = crc;
    __threadfence_system();
  }
}

// ---------------------------------------------------------------------------
// Pack layout: one CTA scans the eligible-chunk flags of [chunk_lo, chunk_hi)
// in global chunk order (= ascending (handle, chunk), since buffers are
// registered by ascending handle), writes the POSD header + entries and one
// CopyItem per entry.
// eligible = flag && !verdict_ok(buffer) && !(exclude_dag && dag_dirty(buffer)).
//
// Rounds of 32 chunks aligned to bitmap words: lane l of a round holds chunk
// 32k + l, so loads are coalesced, the dirty-bitmap word is one ballot and a
// lane's rank among the round's entries is a popc.  Each warp owns a
// contiguous range of rounds; two block barriers join the warp totals.
// Bitmap word k is written by the launch holding its last existing chunk
// (earlier launches' flags are final by then), so waves need no memset.
// 512 threads x 64 registers: half an SM, so the scan starts beside a
// running hash CTA of the next wave.
constexpr int kScanThreads = 512;
constexpr int kScanWarps = kScanThreads / 32;
constexpr uint32_t kCandSlots = 1024;  // O1 candidate list (the rest is walked)
constexpr int kScanKeep = 4;  // rounds per warp kept in registers between the passes

__global__ void __launch_bounds__(kScanThreads) k_pack_scan(
    const DevBuf* bufs, const uint2* chunk_map, uint64_t chunk_lo, uint64_t chunk_hi,
    uint64_t chunk_size, const uint8_t* flags, const uint8_t* verdict, const uint8_t* dag_dirty,
    int exclude_dag, const uint32_t* digests, uint64_t epoch, uint32_t pack_flags, uint8_t* cache,
    uint64_t cache_capacity, uint64_t* cursor, CopyItem* items,
    uint64_t* result /* [n, total, overflow, n_items, base, -, payload] */,
    volatile uint64_t* result_host /* mapped pinned mirror (no DMA queue in between) */,
    uint64_t seq /* written last into result_host[5] */,
    // fused O1 (whole-buffer CRC + verdict for buffers [vb0, vb1) with upstream provenance):
    uint32_t vb0, uint32_t vb1, const uint32_t* tcs, const uint32_t* xfold, int dedup, uint32_t* crc_out,
    uint8_t* verdict_out, uint64_t fixed_base /* ~0 = at *cursor; cursor (if set) is advanced */,
    uint32_t* bitmap /* dirty bitmap words to (re)build, or null */, uint64_t n_total) {
  __shared__ uint32_t tz[1024];  // Z^chunk_size
  __shared__ uint64_t s_wn[kScanWarps], s_wb[kScanWarps], s_tot[3];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  if (vb1 > vb0) {
    // Candidates (upstream provenance) into a smem list in one parallel pass,
    // then one warp per candidate: no warp walks buffers it has nothing to do for.
    __shared__ uint32_t s_cand[kCandSlots];
    __shared__ uint32_t s_ncand;
    if (t == 0) s_ncand = 0;
    for (int q = t; q < 1024; q += kScanThreads) tz[q] = __ldg(tcs + q);
    __syncthreads();
    for (uint32_t i = vb0 + t; i < vb1; i += kScanThreads) {
      const bool cand = dedup && (bufs[i].flags & kBufHasUpstream);
      if (cand) {
        const uint32_t slot = atomicAdd(&s_ncand, 1u);
        if (slot < kCandSlots) s_cand[slot] = i;
        else verdict_out[i] = 2;  // list full: folded by the walk below
      } else {
        verdict_out[i] = 0;  // no provenance -> no verdict (cr.hpp:390)
      }
    }
    __syncthreads();
    const uint32_t nc = s_ncand < kCandSlots ? s_ncand : kCandSlots;
    for (uint32_t q = warp; q < nc; q += kScanWarps) {
      const uint32_t i = s_cand[q];
      const DevBuf b = bufs[i];
      const uint32_t crc = warp_fold_buffer(b, digests, tz, xfold[i], lane);
      if (lane == 0) {
        crc_out[i] = crc;
        verdict_out[i] = crc == b.upstream_crc && (b.flags & kBufHostUntouched) && !dag_dirty[i];
      }
    }
    if (s_ncand > kCandSlots) {  // more candidates than list slots: walk the rest
      __syncthreads();
      for (uint32_t i = vb0 + warp; i < vb1; i += kScanWarps) {
        if (verdict_out[i] != 2) continue;
        const DevBuf b = bufs[i];
        const uint32_t crc = warp_fold_buffer(b, digests, tz, xfold[i], lane);
        __syncwarp();
        if (lane == 0) {
          crc_out[i] = crc;
          verdict_out[i] = crc == b.upstream_crc && (b.flags & kBufHostUntouched) && !dag_dirty[i];
        }
      }
    }
    __syncthreads();  // verdicts are read below
  }
  const uint64_t base = fixed_base != ~0ull ? fixed_base : *cursor;
  uint8_t* pack = cache + base;
  const uint64_t w0 = chunk_lo >> 5, w1 = (chunk_hi + 31) >> 5;
  const uint64_t per_w = (w1 - w0 + kScanWarps - 1) / kScanWarps;
  const uint64_t r0 = w0 + (uint64_t)warp * per_w < w1 ? w0 + (uint64_t)warp * per_w : w1;
  const uint64_t r1 = r0 + per_w < w1 ? r0 + per_w : w1;

  struct Lane {
    uint2 cm;
    uint32_t mask;   // ballot of eligible lanes
    uint64_t len;    // this lane's chunk length (0 if not eligible)
  };
  auto look = [&](uint64_t k, bool with_bitmap) -> Lane {
    const uint64_t g = 32 * k + lane;
    const bool in = g >= chunk_lo && g < chunk_hi;
    Lane L{make_uint2(0, 0), 0u, 0};
    uint8_t f = 0;
    if (in) {
      L.cm = chunk_map[g];
      f = flags[g];
    }
    bool el = false;
    if (in && f) {
      el = !verdict[L.cm.x] && !(exclude_dag && dag_dirty[L.cm.x]);
      if (el) {
        const DevBuf& b = bufs[L.cm.x];
        L.len = L.cm.y + 1 == b.nchunks ? b.size - (uint64_t)L.cm.y * chunk_size : chunk_size;
      }
    }
    L.mask = __ballot_sync(0xffffffffu, el);
    if (with_bitmap && bitmap) {
      const uint64_t last = (32 * k + 31 < n_total ? 32 * k + 31 : n_total - 1);
      if (last >= chunk_lo && last < chunk_hi) {  // this launch owns word k
        const uint32_t fb = in ? f : (g < n_total ? flags[g] : 0);
        const uint32_t word = __ballot_sync(0xffffffffu, fb != 0);
        if (lane == 0) bitmap[k] = word;
      }
    }
    return L;
  };
  auto warp_sum = [&](uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  // Pass 1: per-warp totals (entries, padded payload bytes).
  Lane keep[kScanKeep];
  uint64_t wn = 0, wb = 0;
  auto count = [&](const Lane& L) {
    wn += __popc(L.mask);
    wb += warp_sum(L.len ? (L.len + 15) & ~15ull : 0);
  };
#pragma unroll
  for (int j = 0; j < kScanKeep; ++j) {  // fixed indices: `keep` stays in registers
    keep[j] = Lane{make_uint2(0, 0), 0u, 0};
    if (r0 + j < r1) {
      keep[j] = look(r0 + j, true);
      count(keep[j]);
    }
  }
  for (uint64_t k = r0 + kScanKeep; k < r1; ++k) count(look(k, true));
  if (lane == 0) {
    s_wn[warp] = wn;
    s_wb[warp] = wb;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the warp totals
    uint64_t n = lane < kScanWarps ? s_wn[lane] : 0, b = lane < kScanWarps ? s_wb[lane] : 0;
    uint64_t in_n = n, in_b = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t an = __shfl_up_sync(0xffffffffu, in_n, o), ab = __shfl_up_sync(0xffffffffu, in_b, o);
      if (lane >= o) {
        in_n += an;
        in_b += ab;
      }
    }
    if (lane < kScanWarps) {
      s_wn[lane] = in_n - n;
      s_wb[lane] = in_b - b;
    }
    const uint64_t N = __shfl_sync(0xffffffffu, in_n, 31), B = __shfl_sync(0xffffffffu, in_b, 31);
    if (lane == 0) {
      const uint64_t payload_off = (kPackHeader + kPackEntry * N + kPackAlign - 1) / kPackAlign * kPackAlign;
      const uint64_t total = payload_off + B;
      const bool overflow = base + total > cache_capacity;
      result[0] = N;
      result[1] = total;
      result[2] = overflow;
      result[3] = overflow ? 0 : N;  // items for the copy kernel
      result[4] = base;
      result[6] = B;
      result[7] = 0;
      if (!overflow && cursor) *cursor = base + (total + kPackAlign - 1) / kPackAlign * kPackAlign;
      if (result_host) {
        result_host[0] = N;
        result_host[1] = total;
        result_host[2] = overflow;
        result_host[3] = overflow ? 0 : N;
        result_host[4] = base;
        result_host[6] = B;
        result_host[7] = 0;
        __threadfence_system();
        result_host[5] = seq;
        __threadfence_system();
      }
      s_tot[0] = N;
      s_tot[1] = B;
      s_tot[2] = overflow;
    }
  }
  __syncthreads();
  const uint64_t N = s_tot[0], B = s_tot[1];
  if (s_tot[2]) return;  // overflow: the host reports StagingExhausted
  const uint64_t payload_off = (kPackHeader + kPackEntry * N + kPackAlign - 1) / kPackAlign * kPackAlign;
  if (t == 0) {
    uint32_t* h = reinterpret_cast<uint32_t*>(pack);
    h[0] = kPackMagic;
    h[1] = 1;
    *reinterpret_cast<uint64_t*>(pack + 8) = chunk_size;
    h[4] = (uint32_t)N;
    h[5] = pack_flags;
    *reinterpret_cast<uint64_t*>(pack + 24) = payload_off;
    *reinterpret_cast<uint64_t*>(pack + 32) = B;
    *reinterpret_cast<uint64_t*>(pack + 40) = epoch;
    *reinterpret_cast<uint64_t*>(pack + 48) = payload_off + B;
    *reinterpret_cast<uint64_t*>(pack + 56) = 0;
  }
  for (uint64_t i = kPackHeader + kPackEntry * N + t; i < payload_off; i += kScanThreads) pack[i] = 0;
  // Pass 2: entries + copy items at the warp's base.
  uint64_t e = s_wn[warp], off = s_wb[warp];
  auto emit = [&](uint64_t k, const Lane& L) {
    const uint64_t pl = L.len ? (L.len + 15) & ~15ull : 0;
    uint64_t incl = pl;  // inclusive prefix of the round's padded lengths
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t a = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += a;
    }
    if (L.mask >> lane & 1) {
      const uint64_t my_e = e + __popc(L.mask & lt);
      const uint64_t my_off = off + incl - pl;
      const DevBuf& b = bufs[L.cm.x];
      const uint64_t g = 32 * k + lane;
      uint4* ent = reinterpret_cast<uint4*>(pack + kPackHeader + my_e * kPackEntry);
      ent[0] = make_uint4((uint32_t)b.handle, (uint32_t)(b.handle >> 32), (uint32_t)my_off,
                          (uint32_t)(my_off >> 32));
      ent[1] = make_uint4(L.cm.y, (uint32_t)L.len, digests[g], 0u);
      CopyItem ci;
      ci.src = b.ptr + (uint64_t)L.cm.y * chunk_size;
      ci.dst = (uint64_t)pack + payload_off + my_off;
      ci.len = L.len;
      ci.padded = pl;
      items[my_e] = ci;
    }
    e += __popc(L.mask);
    off += __shfl_sync(0xffffffffu, incl, 31);
  };
#pragma unroll
  for (int j = 0; j < kScanKeep; ++j)
    if (r0 + j < r1) emit(r0 + j, keep[j]);
  for (uint64_t k = r0 + kScanKeep; k < r1; ++k) emit(k, look(k, false));
}

// ---------------------------------------------------------------------------
// Tiled scan for the copy-engine direct pre-copy (no O1 phase: k_buffer_crc
// ran before it).  Tiles of `wpt` 32-chunk words are taken in order through an
// atomic ticket; each publishes its aggregate {entries, padded bytes, runs},
// looks back over its predecessors (decoupled look-back: an inclusive prefix
// stops the walk, aggregates are summed past) and publishes its inclusive
// prefix.  Status flags carry the launch's sequence number, so nothing is
// cleared between launches; the last ticket resets the ticket counter, and
// the last tile to finish emitting writes the header and the host mirror.
struct TileStatus {
  unsigned long long agg_flag, inc_flag;  // = seq when the values below are valid
  unsigned long long agg[3], inc[3];      // entries, padded payload bytes, runs
};
struct TileCtl {
  unsigned int ticket;     // next tile id
  unsigned int finished;   // tiles done emitting
};

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(
    const DevBuf* bufs, const uint2* chunk_map, uint64_t chunk_lo, uint64_t chunk_hi, uint64_t chunk_size,
    const uint8_t* flags, const uint8_t* verdict, const uint8_t* dag_dirty, int exclude_dag,
    const uint32_t* digests, uint64_t epoch, uint8_t* cache, uint64_t cache_capacity, uint64_t* cursor,
    uint64_t fixed_base, uint64_t* result, volatile uint64_t* result_host, uint64_t seq, uint32_t* bitmap,
    uint64_t n_total, uint64_t* run_src, uint64_t* run_dst, uint64_t* run_len, TileStatus* status,
    TileCtl* ctl, uint32_t wpt) {
  __shared__ uint64_t s_wn[kScanWarps], s_wb[kScanWarps], s_wr[kScanWarps];
  __shared__ uint64_t s_pre[3];
  __shared__ uint32_t s_tile, s_last;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t w0 = chunk_lo >> 5, w1 = (chunk_hi + 31) >> 5;
  const uint32_t ntiles = (uint32_t)((w1 - w0 + wpt - 1) / wpt);
  if (t == 0) s_tile = atomicAdd(&ctl->ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  if (t == 0 && tile == ntiles - 1) ctl->ticket = 0;  // every other ticket is taken
  const uint64_t base = fixed_base != ~0ull ? fixed_base : *cursor;
  uint8_t* pack = cache + base;
  const uint64_t tw0 = w0 + (uint64_t)tile * wpt, tw1 = tw0 + wpt < w1 ? tw0 + wpt : w1;
  const uint64_t per_w = (tw1 - tw0 + kScanWarps - 1) / kScanWarps;
  const uint64_t r0 = tw0 + (uint64_t)warp * per_w < tw1 ? tw0 + (uint64_t)warp * per_w : tw1;
  const uint64_t r1 = r0 + per_w < tw1 ? r0 + per_w : tw1;
  struct Lane {
    uint2 cm;
    uint32_t mask, start;
    uint64_t len;
  };
  auto look = [&](uint64_t k) -> Lane {
    const uint64_t g = 32 * k + lane;
    const bool in = g >= chunk_lo && g < chunk_hi;
    Lane L{make_uint2(0, 0), 0u, 0u, 0};
    uint8_t f = 0;
    if (in) {
      L.cm = chunk_map[g];
      f = flags[g];
    }
    bool el = false;
    if (in && f) {
      el = !verdict[L.cm.x] && !(exclude_dag && dag_dirty[L.cm.x]);
      if (el) {
        const DevBuf& b = bufs[L.cm.x];
        L.len = L.cm.y + 1 == b.nchunks ? b.size - (uint64_t)L.cm.y * chunk_size : chunk_size;
      }
    }
    L.mask = __ballot_sync(0xffffffffu, el);
    const uint32_t prev_buf = __shfl_up_sync(0xffffffffu, L.cm.x, 1);
    const uint32_t same = __ballot_sync(0xffffffffu, lane > 0 && prev_buf == L.cm.x);
    L.start = L.mask & ~(L.mask & (L.mask << 1) & same);
    if (bitmap) {
      const uint64_t last = (32 * k + 31 < n_total ? 32 * k + 31 : n_total - 1);
      if (last >= chunk_lo && last < chunk_hi) {
        const uint32_t fb = in ? f : (g < n_total ? flags[g] : 0);
        const uint32_t word = __ballot_sync(0xffffffffu, fb != 0);
        if (lane == 0) bitmap[k] = word;
      }
    }
    return L;
  };
  auto warp_sum = [&](uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  Lane keep[kScanKeep];
  uint64_t wn = 0, wb = 0, wr = 0;
  auto count = [&](const Lane& L) {
    wn += __popc(L.mask);
    wr += __popc(L.start);
    wb += warp_sum(L.len ? (L.len + 15) & ~15ull : 0);
  };
#pragma unroll
  for (int j = 0; j < kScanKeep; ++j) {
    keep[j] = Lane{make_uint2(0, 0), 0u, 0u, 0};
    if (r0 + j < r1) {
      keep[j] = look(r0 + j);
      count(keep[j]);
    }
  }
  for (uint64_t k = r0 + kScanKeep; k < r1; ++k) count(look(k));
  if (lane == 0) {
    s_wn[warp] = wn;
    s_wb[warp] = wb;
    s_wr[warp] = wr;
  }
  __syncthreads();
  if (warp == 0) {
    uint64_t v[3] = {lane < kScanWarps ? s_wn[lane] : 0, lane < kScanWarps ? s_wb[lane] : 0,
                     lane < kScanWarps ? s_wr[lane] : 0};
    uint64_t in[3] = {v[0], v[1], v[2]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const uint64_t a = __shfl_up_sync(0xffffffffu, in[q], o);
        if (lane >= o) in[q] += a;
      }
    }
    if (lane < kScanWarps) {
      s_wn[lane] = in[0] - v[0];
      s_wb[lane] = in[1] - v[1];
      s_wr[lane] = in[2] - v[2];
    }
    uint64_t agg[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) agg[q] = __shfl_sync(0xffffffffu, in[q], 31);
    if (lane == 0) {
      TileStatus* my = status + tile;
      if (tile == 0) {  // no predecessor: the inclusive prefix is the aggregate
        for (int q = 0; q < 3; ++q) my->inc[q] = agg[q];
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&my->inc_flag), "l"((unsigned long long)seq)
                     : "memory");
        for (int q = 0; q < 3; ++q) s_pre[q] = 0;
      } else {
        for (int q = 0; q < 3; ++q) my->agg[q] = agg[q];
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&my->agg_flag), "l"((unsigned long long)seq)
                     : "memory");
        uint64_t pre[3] = {0, 0, 0};
        for (int p = (int)tile - 1; p >= 0;) {
          TileStatus* st = status + p;
          unsigned long long fi, fa;
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(fi) : "l"(&st->inc_flag) : "memory");
          if (fi == seq) {
            for (int q = 0; q < 3; ++q) pre[q] += st->inc[q];
            break;
          }
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(fa) : "l"(&st->agg_flag) : "memory");
          if (fa == seq) {
            for (int q = 0; q < 3; ++q) pre[q] += st->agg[q];
            --p;
          }
          // else: the predecessor has not published yet -- poll again
        }
        for (int q = 0; q < 3; ++q) my->inc[q] = pre[q] + agg[q];
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&my->inc_flag), "l"((unsigned long long)seq)
                     : "memory");
        for (int q = 0; q < 3; ++q) s_pre[q] = pre[q];
      }
    }
  }
  __syncthreads();
  // Emit: entries at their global index, runs at their global run index.
  uint64_t e = s_pre[0] + s_wn[warp], off = s_pre[1] + s_wb[warp], rb = s_pre[2] + s_wr[warp];
  auto emit = [&](uint64_t k, const Lane& L) {
    const uint32_t cont = L.mask & ~L.start;
    const uint32_t rest = lane < 31 ? cont >> (lane + 1) : 0u;
    const int nrun = __ffs(~rest);
    const int last = lane + nrun - 1 < 31 ? lane + nrun - 1 : 31;
    const uint64_t last_len = __shfl_sync(0xffffffffu, L.len, last);
    const uint64_t pl = L.len ? (L.len + 15) & ~15ull : 0;
    uint64_t incl = pl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t a = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += a;
    }
    if (L.mask >> lane & 1) {
      const DevBuf& b = bufs[L.cm.x];
      const uint64_t g = 32 * k + lane;
      const uint64_t my_e = e + __popc(L.mask & lt), my_off = off + incl - pl;
      if (base + kPackHeader + (my_e + 1) * kPackEntry <= cache_capacity) {  // (host reserves the worst case)
        uint4* ent = reinterpret_cast<uint4*>(pack + kPackHeader + my_e * kPackEntry);
        ent[0] = make_uint4((uint32_t)b.handle, (uint32_t)(b.handle >> 32), (uint32_t)my_off,
                            (uint32_t)(my_off >> 32));
        ent[1] = make_uint4(L.cm.y, (uint32_t)L.len, digests[g], 0u);
      }
      if (L.start >> lane & 1) {
        const uint64_t ri = rb + __popc(L.start & lt);
        run_src[ri] = b.ptr + (uint64_t)L.cm.y * chunk_size;
        run_dst[ri] = b.image + (uint64_t)L.cm.y * chunk_size;
        run_len[ri] = (uint64_t)(nrun - 1) * chunk_size + last_len;
      }
    }
    e += __popc(L.mask);
    off += __shfl_sync(0xffffffffu, incl, 31);
    rb += __popc(L.start);
  };
#pragma unroll
  for (int j = 0; j < kScanKeep; ++j)
    if (r0 + j < r1) emit(r0 + j, keep[j]);
  for (uint64_t k = r0 + kScanKeep; k < r1; ++k) emit(k, look(k));
  // The last tile to finish writes the header and tells the host.
  __syncthreads();
  if (t == 0) {
    __threadfence();
    s_last = atomicAdd(&ctl->finished, 1u) == ntiles - 1;
  }
  __syncthreads();
  if (!s_last || t != 0) return;
  ctl->finished = 0;
  const TileStatus* lastst = status + (ntiles - 1);
  unsigned long long fl;
  do {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(fl) : "l"(&lastst->inc_flag) : "memory");
  } while (fl != seq);
  const uint64_t N = lastst->inc[0], B = lastst->inc[1], R = lastst->inc[2];
  const uint64_t total = kPackHeader + kPackEntry * N;  // index pack: header + entries
  const bool overflow = base + total > cache_capacity;
  uint32_t* h = reinterpret_cast<uint32_t*>(pack);
  if (!overflow) {
    h[0] = kPackMagic;
    h[1] = 1;
    *reinterpret_cast<uint64_t*>(pack + 8) = chunk_size;
    h[4] = (uint32_t)N;
    h[5] = kPackFlagDirect;
    *reinterpret_cast<uint64_t*>(pack + 24) = total;
    *reinterpret_cast<uint64_t*>(pack + 32) = 0;
    *reinterpret_cast<uint64_t*>(pack + 40) = epoch;
    *reinterpret_cast<uint64_t*>(pack + 48) = total;
    *reinterpret_cast<uint64_t*>(pack + 56) = 0;
    if (cursor) *cursor = base + (total + kPackAlign - 1) / kPackAlign * kPackAlign;
  }
  result[0] = N;
  result[1] = total;
  result[2] = overflow;
  result[3] = overflow ? 0 : N;
  result[4] = base;
  result[6] = B;
  result[7] = R;
  result_host[0] = N;
  result_host[1] = total;
  result_host[2] = overflow;
  result_host[3] = overflow ? 0 : N;
  result_host[4] = base;
  result_host[6] = B;
  result_host[7] = R;
  __threadfence_system();
  result_host[5] = seq;
  __threadfence_system();
}

// ---------------------------------------------------------------------------
// Bulk copy engine: each CTA streams its items (grid-stride) through a ring of
// kCopyStages smem slots with cp.async.bulk (TMA bulk) G->S loads completing
// on an mbarrier and S->G bulk stores tracked by bulk groups; one elected
// thread drives the pipeline.  Requires 16-B aligned src/dst (checked by the
// host; otherwise k_copy_simt runs).  The <16-B remainder of an item and its
// zero padding go through one vector store.
constexpr int kCopyStages = 8;
constexpr uint32_t kCopyPiece = 8192;
constexpr uint32_t kCopySmem = kCopyStages * kCopyPiece + 64;


__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

struct PieceIter {  // walks (item, offset) pieces of this CTA's grid-stride items
  uint64_t item, off;
};

// ppi == 0: CTA b copies items b, b + grid, ... piece by piece.  ppi > 0
// (every item <= ppi pieces): the grid strides over the n * ppi PIECES
// instead, so a short list of long items (the STW delta: ~200 chunks of
// 64 KiB at config 2) still puts every CTA's ring to work at once.
__global__ void __launch_bounds__(32) k_copy_bulk(const CopyItem* items, const uint64_t* n_items_dev,
                                                  uint64_t n_items_host, uint32_t ppi) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kCopyStages * kCopyPiece);
  const uint64_t n = n_items_dev ? *n_items_dev : n_items_host;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kCopyStages; ++s) mbar_init(bars + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");

  // Piece = up to kCopyPiece bytes of the 16-B-aligned body of an item.
  auto body = [&](uint64_t i) { return items[i].len & ~15ull; };
  uint64_t gp = blockIdx.x;  // ppi > 0: this CTA's next global piece
  auto advance = [&](PieceIter& it) {
    if (ppi) {  // next non-empty piece of the grid-stride over pieces
      for (gp += gridDim.x; gp < n * ppi; gp += gridDim.x) {
        it.item = gp / ppi;
        it.off = (gp % ppi) * kCopyPiece;
        if (it.off < body(it.item)) return;
      }
      it.item = n;
      return;
    }
    it.off += kCopyPiece;
    while (it.item < n && it.off >= body(it.item)) {
      it.item += gridDim.x;
      it.off = 0;
    }
  };
  auto first = [&]() {
    if (ppi) {
      PieceIter it{n, 0};
      for (; gp < n * ppi; gp += gridDim.x) {
        it.item = gp / ppi;
        it.off = (gp % ppi) * kCopyPiece;
        if (it.off < body(it.item)) return it;
      }
      it.item = n;
      return it;
    }
    PieceIter it{blockIdx.x, 0};
    while (it.item < n && body(it.item) == 0) it.item += gridDim.x;
    return it;
  };
  uint64_t slot_dst[kCopyStages];
  uint32_t slot_bytes[kCopyStages];
  uint32_t phase = 0;  // bit s = parity of slot s
  PieceIter ld = first();
  int issued = 0;
  // Prologue: fill the ring.
  for (; issued < kCopyStages && ld.item < n; ++issued) {
    const CopyItem& c = items[ld.item];
    uint32_t bytes = (uint32_t)umin64((uint64_t)kCopyPiece, body(ld.item) - ld.off);
    slot_dst[issued] = c.dst + ld.off;
    slot_bytes[issued] = bytes;
    mbar_expect_tx(bars + issued, bytes);
    bulk_g2s(smem + issued * kCopyPiece, (const void*)(c.src + ld.off), bytes, bars + issued);
    advance(ld);
  }
  int slot = 0;
  for (int done = 0; done < issued; ++done) {
    mbar_wait(bars + slot, (phase >> slot) & 1);
    phase ^= 1u << slot;
    bulk_s2g((void*)slot_dst[slot], smem + slot * kCopyPiece, slot_bytes[slot]);
    bulk_commit();
    if (ld.item < n) {
      // Reuse this slot once its store has read the smem.
      bulk_wait_read<0>();
      const CopyItem& c = items[ld.item];
      uint32_t bytes = (uint32_t)umin64((uint64_t)kCopyPiece, body(ld.item) - ld.off);
      slot_dst[slot] = c.dst + ld.off;
      slot_bytes[slot] = bytes;
      mbar_expect_tx(bars + slot, bytes);
      bulk_g2s(smem + slot * kCopyPiece, (const void*)(c.src + ld.off), bytes, bars + slot);
      advance(ld);
      ++issued;
    }
    slot = (slot + 1) % kCopyStages;
  }
  bulk_wait_all();
  // Remainders (< 16 B) + zero padding of this CTA's items, byte-exact.
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const CopyItem c = items[i];
    const uint8_t* s = reinterpret_cast<const uint8_t*>(c.src);
    uint8_t* d = reinterpret_cast<uint8_t*>(c.dst);
    for (uint64_t k = c.len & ~15ull; k < c.padded; ++k) d[k] = k < c.len ? s[k] : 0;
  }
}

// Fallback for items whose src or dst is not 16-B aligned: one warp per item,
// byte copy + zero padding to `padded`.
__global__ void k_copy_simt(const CopyItem* items, const uint64_t* n_items_dev, uint64_t n_items_host) {
  const uint64_t n = n_items_dev ? *n_items_dev : n_items_host;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < n; i += nw) {
    const CopyItem c = items[i];
    const uint8_t* s = reinterpret_cast<const uint8_t*>(c.src);
    uint8_t* d = reinterpret_cast<uint8_t*>(c.dst);
    for (uint64_t k = lane; k < c.padded; k += 32) d[k] = k < c.len ? s[k] : 0;
  }
}

// Staging without the copy engine: the STW delta's header, work list and copy
// items travel from mapped pinned memory into device memory by SM loads (the
// copy engines are busy with the pre-copy's host leg; an H2D memcpy queued
// behind it held the ckpt stream -- and so the final stop -- for ~50 us).
struct StageSeg {
  const uint8_t* src;  // mapped pinned host memory (16-B aligned)
  uint8_t* dst;        // device memory (16-B aligned); src == null: zero-fill
  uint64_t len;        // multiple of 16
};
struct StageList {
  StageSeg seg[5];
  uint32_t n;
};

__global__ void k_stage_in(const __grid_constant__ StageList L) {
  for (uint32_t s = 0; s < L.n; ++s) {
    const StageSeg g = L.seg[s];
    const uint64_t n16 = g.len / 16;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (g.src)  // uncached: the host rewrites the staging buffer between launches
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(g.src + 16 * i));
      reinterpret_cast<uint4*>(g.dst)[i] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Host leg for SHORT runs (chunk_copied into captured_, cr.hpp:499-501): SM
// stores straight into the mapped pinned host image.  The copy engine pays
// ~4 us per copy (64 KiB runs: 13.8 GB/s, 448 KiB: 38, one copy at a time
// however many streams), while 4 CTAs of plain 16-B stores hold the link at
// 52.7 GB/s for any run length and cost a concurrent HBM kernel ~1.25x (16
// CTAs: 3.3x) -- tools/runs_micro.cu, profiles/r2/runs_micro.txt.  A batch
// is one slot of the host leg's window: SoA {src, dst, bytes, exclusive
// prefix} in mapped pinned memory, read once into shared memory; CTA g
// copies bytes [g*T/G, (g+1)*T/G) of the batch's concatenation.
constexpr int kShipThreads = 512;
constexpr int kShipCtas = 4;
constexpr uint32_t kShipMaxRuns = 2048;
constexpr uint32_t kShipSmem = 4 * kShipMaxRuns * 8;

__device__ __forceinline__ void cta_copy_to_host(const uint8_t* s, uint8_t* d, uint64_t m) {
  if ((((uintptr_t)s ^ (uintptr_t)d) & 15) == 0) {
    const uint64_t head = umin64(m, (16 - ((uintptr_t)s & 15)) & 15);
    if (threadIdx.x < head) d[threadIdx.x] = s[threadIdx.x];
    s += head;
    d += head;
    m -= head;
    const uint64_t n16 = m >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    uint4* d4 = reinterpret_cast<uint4*>(d);
    // 4 loads in flight per thread before the stores: the HBM reads stay
    // ahead of the link even when a hash wave saturates HBM beside them
    constexpr int U = 4;
    uint64_t i = threadIdx.x;
    for (; i + (U - 1) * blockDim.x < n16; i += U * blockDim.x) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(s4 + i + u * blockDim.x));
#pragma unroll
      for (int u = 0; u < U; ++u) d4[i + u * blockDim.x] = v[u];
    }
    for (; i < n16; i += blockDim.x) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(s4 + i));
      d4[i] = v;
    }
    if (threadIdx.x < (m & 15)) d[16 * n16 + threadIdx.x] = s[16 * n16 + threadIdx.x];
  } else {  // different alignments mod 16 (odd chunk sizes): bytes
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) d[i] = s[i];
  }
}

__global__ void __launch_bounds__(kShipThreads) k_ship_runs(const uint64_t* runs, uint32_t n, uint64_t total) {
  extern __shared__ __align__(16) uint64_t ship_sm[];
  uint64_t* src = ship_sm;
  uint64_t* dst = ship_sm + n;
  uint64_t* len = ship_sm + 2 * n;
  uint64_t* pre = ship_sm + 3 * n;
  // the host rewrites a slot between launches: uncached loads, all in flight at once
  for (uint32_t i = threadIdx.x; i < 4 * n; i += blockDim.x) {
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(runs + i));
    ship_sm[i] = v;
  }
  __syncthreads();
  const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
  uint64_t lo = per * blockIdx.x;
  const uint64_t hi = umin64(total, lo + per);
  if (lo >= hi) return;
  uint32_t a = 0, b = n;  // last run with pre <= lo
  while (b - a > 1) {
    const uint32_t mid = (a + b) / 2;
    if (pre[mid] <= lo) a = mid; else b = mid;
  }
  for (uint32_t r = a; lo < hi && r < n; ++r) {
    const uint64_t from = lo - pre[r], to = umin64(len[r], hi - pre[r]);
    if (to > from)
      cta_copy_to_host(reinterpret_cast<const uint8_t*>(src[r]) + from, reinterpret_cast<uint8_t*>(dst[r]) + from,
                       to - from);
    lo = pre[r] + len[r];
  }
}

// A globaltimer stamp in stream order, written by a one-thread kernel: a
// clock that does not ride the channel's event machinery (timing events on a
// stream queued next to a long copy-engine batch were seen landing ~40 us
// late).
__global__ void k_stamp(unsigned long long* at) { *at = globaltimer_ns(); }

// ---------------------------------------------------------------------------
// Restore: POSD entries -> copy items (pack payload -> buffer chunk).
// Validation mirrors write_content's range check (buffer.hpp:80) and the
// pack's own section checks; errors set bits in *err (1 corrupt, 2 locator).
__global__ void k_pack_items(const uint8_t* pack, uint64_t pack_bytes, const DevBuf* bufs,
                             uint32_t nbufs, uint64_t chunk_size, CopyItem* items, uint32_t* err) {
  const uint32_t n = *reinterpret_cast<const uint32_t*>(pack + 16);
  const uint64_t payload_off = *reinterpret_cast<const uint64_t*>(pack + 24);
  const uint64_t payload = *reinterpret_cast<const uint64_t*>(pack + 32);
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t* ent = pack + kPackHeader + e * kPackEntry;
    uint64_t h = *reinterpret_cast<const uint64_t*>(ent);
    uint64_t off = *reinterpret_cast<const uint64_t*>(ent + 8);
    uint32_t c = *reinterpret_cast<const uint32_t*>(ent + 16);
    uint32_t len = *reinterpret_cast<const uint32_t*>(ent + 20);
    // binary search: buffers are registered by ascending handle
    uint32_t lo = 0, hi = nbufs;
    while (lo < hi) {
      uint32_t mid = (lo + hi) / 2;
      if (bufs[mid].handle < h) lo = mid + 1;
      else hi = mid;
    }
    CopyItem ci{0, 0, 0, 0};
    if ((off | payload_off) & 15) {  // payloads are 16-B padded by format: the bulk copy relies on it
      atomicOr(err, 1u);
    } else if (lo >= nbufs || bufs[lo].handle != h) {
      atomicOr(err, 2u);
    } else if ((uint64_t)c * chunk_size + len > bufs[lo].size || off + len > payload) {
      atomicOr(err, 2u);
    } else {
      ci.src = (uint64_t)pack + payload_off + off;
      ci.dst = bufs[lo].ptr + (uint64_t)c * chunk_size;
      ci.len = len;
      ci.padded = len;  // never write past the chunk on restore
    }
    items[e] = ci;
  }
}

// ---------------------------------------------------------------------------
// fill_bytes(seed) into device memory: word k (8 bytes, little endian) is the
// (k+1)-th SplitMix64 output, state_k = seed + (k+1)*gamma (rng.hpp:15-20,
// 43-54): each thread produces its words independently.
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct FillRange {
  uint64_t ptr, n, seed;
};

constexpr int kFillMaxRanges = 256;  // by-value kernel parameter (6 KiB)
struct FillBatch {
  uint32_t count;
  uint32_t pad;
  FillRange r[kFillMaxRanges];
};

__global__ void k_fill(const __grid_constant__ FillBatch b) {
  for (uint32_t ri = blockIdx.y; ri < b.count; ri += gridDim.y) {
    const FillRange f = b.r[ri];
    const uint64_t words = (f.n + 7) / 8;
    const bool aligned = (f.ptr & 15) == 0;
    for (uint64_t p = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 2; p < words;
         p += (uint64_t)gridDim.x * blockDim.x * 2) {
      uint64_t w0 = splitmix_at(f.seed, p), w1 = splitmix_at(f.seed, p + 1);
      uint64_t byte0 = p * 8;
      if (aligned && byte0 + 16 <= f.n) {
        *reinterpret_cast<uint4*>(f.ptr + byte0) =
            make_uint4((uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32));
      } else {
        uint8_t* d = reinterpret_cast<uint8_t*>(f.ptr);
        for (int k = 0; k < 16 && byte0 + k < f.n; ++k)
          d[byte0 + k] = (uint8_t)((k < 8 ? w0 : w1) >> (8 * (k & 7)));
      }
    }
  }
}

}  // namespace posdump
