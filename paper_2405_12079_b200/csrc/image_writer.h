// image_writer.h -- streaming, zero-copy POSI v1 writer.
//
// Emits exactly the bytes of gpucrsim::write_image (include/gpucrsim/image.hpp:
// 136-207): 64-B header, host pages ascending by index, GPU records ascending
// by handle (Inline u64 len + bytes / DedupRef u64 u32 u32 u32 / Recompute
// u32 n + n x u64), DAG bytes, then the meta section unless it is at its
// defaults (image.hpp:68-71).  Unlike the reference it does not deep-copy the
// image (image.hpp:138) and sorts index arrays instead of records, so the
// Inline payloads stream straight from wherever the dump landed them.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/posdump.h"

namespace posdump {

constexpr uint64_t kDeviceAddrBase = 0x700000000000ull;  // config.hpp:14

inline uint64_t posi_record_bytes(const pos_image_rec& r) {  // image.hpp:103-110
  switch (r.kind) {
    case 0: return 9 + 8 + r.inline_len;
    case 1: return 9 + 20;
    case 2: return 9 + 4 + 8ull * r.n_recompute;
  }
  return 0;
}

inline bool posi_meta_default(const pos_image_desc& d) {  // image.hpp:68-71
  return d.n_streams == 0 && d.n_allocs == 0 && d.cursor == 0 && d.next_handle == 1 &&
         d.next_base == kDeviceAddrBase;
}

// Large payloads (Inline bytes, host pages) are not copied in the cursor's
// pass: their places are known there, so the copies run afterwards on
// several host threads (one thread moves ~14 GB/s; the writer streams tens
// of GB per checkpoint).
struct PosiCopy {
  uint8_t* dst;
  const uint8_t* src;
  uint64_t n;
};

struct PosiCursor {
  uint8_t* p;
  std::vector<PosiCopy>* deferred = nullptr;
  static constexpr uint64_t kDeferMin = 1ull << 20;
  void raw(const void* s, uint64_t n) {
    if (n >= kDeferMin && deferred) deferred->push_back(PosiCopy{p, static_cast<const uint8_t*>(s), n});
    else if (n) std::memcpy(p, s, n);
    p += n;
  }
  void u8(uint8_t v) { raw(&v, 1); }
  void u16(uint16_t v) { raw(&v, 2); }
  void u32(uint32_t v) { raw(&v, 4); }
  void u64(uint64_t v) { raw(&v, 8); }
};

// The deferred copies in kPiece pieces over up to 16 threads.
inline void run_posi_copies(const std::vector<PosiCopy>& cps, uint64_t kPiece = 64ull << 20) {
  std::vector<PosiCopy> pieces;
  uint64_t total = 0;
  for (const PosiCopy& c : cps)
    for (uint64_t o = 0; o < c.n; o += kPiece) {
      pieces.push_back(PosiCopy{c.dst + o, c.src + o, std::min(kPiece, c.n - o)});
      total += pieces.back().n;
    }
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nt = (unsigned)std::min<uint64_t>({(uint64_t)std::min(hw, 16u), pieces.size(), total / kPiece + 1});
  if (nt <= 1) {
    for (const PosiCopy& c : pieces) std::memcpy(c.dst, c.src, c.n);
    return;
  }
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i = next++; i < pieces.size(); i = next++) std::memcpy(pieces[i].dst, pieces[i].src, pieces[i].n);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

inline int write_posi_image(const pos_image_desc& d, uint8_t* out, uint64_t cap, uint64_t* size,
                            std::string* err) {
  if ((d.n_pages && !d.pages) || (d.n_recs && !d.recs) || (d.n_allocs && !d.allocs) ||
      (d.n_streams && !d.stream_ids) || (d.dag_len && !d.dag_bytes)) {
    *err = "null section array";
    return POS_E_INVALID_ARGUMENT;
  }
  for (uint32_t i = 0; i < d.n_recs; ++i) {
    const auto& r = d.recs[i];
    if (r.kind > 2) {
      *err = "bad record kind";
      return POS_E_INVALID_ARGUMENT;
    }
    bool found = false;  // image.hpp:152-154
    for (uint32_t a = 0; a < d.n_allocs && !found; ++a) found = d.allocs[a].handle == r.handle;
    if (!found) {
      *err = "gpu record without allocation entry";
      return POS_E_INVARIANT_VIOLATION;
    }
  }
  // Canonical order (image.hpp:138-145) over index arrays.
  std::vector<uint32_t> pg(d.n_pages), rc(d.n_recs), al(d.n_allocs);
  std::iota(pg.begin(), pg.end(), 0u);
  std::iota(rc.begin(), rc.end(), 0u);
  std::iota(al.begin(), al.end(), 0u);
  std::stable_sort(pg.begin(), pg.end(),
                   [&](uint32_t a, uint32_t b) { return d.pages[a].index < d.pages[b].index; });
  std::stable_sort(rc.begin(), rc.end(),
                   [&](uint32_t a, uint32_t b) { return d.recs[a].handle < d.recs[b].handle; });
  std::stable_sort(al.begin(), al.end(),
                   [&](uint32_t a, uint32_t b) { return d.allocs[a].handle < d.allocs[b].handle; });
  std::vector<uint64_t> streams(d.stream_ids, d.stream_ids + d.n_streams);
  std::sort(streams.begin(), streams.end());

  const uint64_t host_len = (uint64_t)d.n_pages * (8 + d.page_size);
  uint64_t gpu_len = 0;
  for (uint32_t i = 0; i < d.n_recs; ++i) gpu_len += posi_record_bytes(d.recs[i]);
  const bool meta_default = posi_meta_default(d);
  const uint64_t meta_len =
      meta_default ? 0 : 4 + 8ull * d.n_streams + 4 + 24ull * d.n_allocs + 24;
  const uint64_t total = 64 + host_len + gpu_len + d.dag_len + meta_len;
  *size = total;
  if (!out || cap < total) return POS_OK;

  std::vector<PosiCopy> deferred;
  PosiCursor w{out, &deferred};
  w.raw("POSI", 4);
  w.u16(1);
  w.u16(d.dag_len ? 1 : 0);
  w.u32(d.n_pages);
  w.u32(d.n_recs);
  w.u64(d.page_size);
  w.u64(host_len);
  w.u64(gpu_len);
  w.u64(d.dag_len);
  w.u64(meta_len);
  w.u64(0);
  for (uint32_t i : pg) {
    w.u64(d.pages[i].index);
    w.raw(d.pages[i].bytes, d.page_size);
  }
  for (uint32_t i : rc) {
    const auto& r = d.recs[i];
    w.u64(r.handle);
    w.u8((uint8_t)r.kind);
    if (r.kind == 0) {
      w.u64(r.inline_len);
      w.raw(r.inline_bytes, r.inline_len);
    } else if (r.kind == 1) {
      w.u64(r.dedup_first_page);
      w.u32(r.dedup_page_count);
      w.u32(r.dedup_offset);
      w.u32(r.dedup_crc);
    } else {
      w.u32(r.n_recompute);
      for (uint32_t k = 0; k < r.n_recompute; ++k) w.u64(r.recompute[k]);
    }
  }
  w.raw(d.dag_bytes, d.dag_len);
  if (!meta_default) {
    w.u32(d.n_streams);
    for (uint64_t s : streams) w.u64(s);
    w.u32(d.n_allocs);
    for (uint32_t i : al) {
      w.u64(d.allocs[i].handle);
      w.u64(d.allocs[i].base);
      w.u64(d.allocs[i].size);
    }
    w.u64(d.cursor);
    w.u64(d.next_handle);
    w.u64(d.next_base);
  }
  run_posi_copies(deferred);
  return POS_OK;
}

}  // namespace posdump
