// posdump.hpp -- C++ host-side mirror of the reference's dump-path interface
// (gpucrsim, /root/reference/proj/include/gpucrsim) over the C ABI in
// posdump.h.  Header-only; link with -lposdump.
//
// Same names, argument meaning and error behaviour as the reference:
//   crc32 / crc32_update            crc32.hpp:26-34 (over DEVICE memory here)
//   GpuBuffer::chunk_count/bytes    buffer.hpp:44-49
//   SimConfig (path keys)           config.hpp:18-45
//   DumpEngine                      the hot-path members of CrEngine
//                                   (cr.hpp:124-1322): plan_precopy, dedup_verdicts,
//                                   record_dirty, dirty_set, at_final_stop,
//                                   materialize, end of session
//   CheckpointImage / write_image   image.hpp:42-207 (byte-identical)
//   SimError / CorruptImageError    errors.hpp:9-68
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "posdump.h"

namespace posdump {

using BufferHandle = uint64_t;

// errors.hpp:9-25 (same order: code = 1 + index).
enum class Errc {
  PastTime,
  Livelock,
  OutOfDeviceMemory,
  InvalidLocator,
  UseAfterFree,
  FreedBuffer,
  BadState,
  PendingKernels,
  UnknownApi,
  InvalidArgument,
  CorruptDag,
  CorruptImage,
  InvariantViolation,
  StagingExhausted,
  OracleMismatch,
  Cuda,      // runtime failure (not in the reference)
  NoDevice,  // there is no CPU fallback
};

class SimError : public std::runtime_error {  // errors.hpp:48-56
 public:
  SimError(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};

class CorruptImageError : public SimError {  // errors.hpp:59-68
 public:
  explicit CorruptImageError(const std::string& what) : SimError(Errc::CorruptImage, what) {}
  CorruptImageError(uint64_t offset, const std::string& what)
      : SimError(Errc::CorruptImage, what), offset_(offset) {}
  uint64_t offset() const { return offset_; }

 private:
  uint64_t offset_ = 0;
};

inline void check(int rc) {
  if (rc == POS_OK) return;
  std::string what = std::string(pos_strerror(rc)) + ": " + pos_last_error();
  if (rc == POS_E_CORRUPT_IMAGE) throw CorruptImageError(what);
  Errc e = rc == POS_E_CUDA ? Errc::Cuda
         : rc == POS_E_NO_DEVICE ? Errc::NoDevice
                                 : static_cast<Errc>(rc - 1);
  throw SimError(e, what);
}

// ---- crc32 over device memory (crc32.hpp:26-34) ---------------------------
inline uint32_t crc32(const void* dev, size_t n, void* stream = nullptr) {
  uint32_t out = 0;
  check(pos_crc32(reinterpret_cast<uint64_t>(dev), n, &out, stream));
  return out;
}
inline uint32_t crc32_update(uint32_t crc, const void* dev, size_t n, void* stream = nullptr) {
  uint32_t out = 0;
  check(pos_crc32_update(crc, reinterpret_cast<uint64_t>(dev), n, &out, stream));
  return out;
}

// ---- buffers (buffer.hpp:20-49) ------------------------------------------------
struct Upstream {
  uint64_t host_addr = 0;
  uint64_t len = 0;
  uint32_t crc = 0;
  uint64_t host_write_seq = 0;
  bool host_untouched = true;  // range_write_seq(host_addr, len) <= host_write_seq (cr.hpp:420)
};

struct GpuBuffer {
  BufferHandle handle = 0;
  uint64_t dev_ptr = 0;  // device address of the allocation (the reference's `base` is virtual)
  uint64_t size = 0;
  bool written_since_ckpt = true;
  std::optional<Upstream> upstream;

  uint32_t chunk_count(uint64_t chunk_size) const {
    return static_cast<uint32_t>((size + chunk_size - 1) / chunk_size);
  }
  uint64_t chunk_bytes(uint32_t idx, uint64_t chunk_size) const {
    uint64_t start = static_cast<uint64_t>(idx) * chunk_size;
    return std::min(chunk_size, size - start);
  }
  pos_buffer_desc desc() const {
    return pos_buffer_desc{handle,
                           dev_ptr,
                           size,
                           upstream.has_value() ? 1u : 0u,
                           upstream ? upstream->crc : 0u,
                           upstream && upstream->host_untouched ? 1u : 0u,
                           written_since_ckpt ? 1u : 0u};
  }
};

struct SimConfig {  // config.hpp:18-45, the keys of the path
  uint64_t chunk_size = 64 * 1024;
  uint64_t page_size = 4096;
  uint64_t device_capacity = 80'000'000'000ull;
  double staging_fraction = 1.0 / 16.0;
  bool dedup = true;
  uint64_t cache_capacity = 0;  // explicit O3 cache size; 0 => staging_fraction of the GPU
  uint64_t staging_capacity() const {
    return static_cast<uint64_t>(static_cast<double>(device_capacity) * staging_fraction);
  }
};

// ---- POSD packs ------------------------------------------------------------------
struct PackRef {
  uint64_t offset = 0;  // in the O3 cache (and in the host landing buffer)
  uint64_t bytes = 0;
};

// ---- the engine ------------------------------------------------------------------
class DumpEngine {
 public:
  explicit DumpEngine(const SimConfig& cfg, int device = 0) : cfg_(cfg) {
    pos_config c{cfg.chunk_size, cfg.page_size, cfg.cache_capacity, cfg.staging_fraction, device,
                 cfg.dedup ? 1 : 0};
    check(pos_ctx_create(&c, &ctx_));
  }
  ~DumpEngine() { pos_ctx_destroy(ctx_); }
  DumpEngine(const DumpEngine&) = delete;
  DumpEngine& operator=(const DumpEngine&) = delete;

  // at_initial_stop: snapshot_buffers_ = active_handles() (cr.hpp:343-375).
  void snapshot(std::vector<GpuBuffer> bufs) {
    std::sort(bufs.begin(), bufs.end(),
              [](const GpuBuffer& a, const GpuBuffer& b) { return a.handle < b.handle; });
    bufs_ = std::move(bufs);
    std::vector<pos_buffer_desc> d;
    for (const auto& b : bufs_) d.push_back(b.desc());
    check(pos_register_buffers(ctx_, d.data(), static_cast<uint32_t>(d.size())));
    dirty_.clear();
  }
  const std::vector<GpuBuffer>& snapshot_buffers() const { return bufs_; }

  // CheckpointTarget::fresh (cr.hpp:35, 396): the next round ships every chunk.
  void set_target_fresh(bool fresh = true) { check(pos_set_target_fresh(ctx_, fresh ? 1 : 0)); }

  // on_alloc (cr.hpp:298-306) / a buffer gone mid-session (cr.hpp:709-716):
  // the snapshot's list changes; unchanged buffers keep their digest history,
  // a new one joins dirty (recorded in dirty_set_, as on_alloc does).
  void update_snapshot(std::vector<GpuBuffer> bufs, bool new_ones_dirty = true) {
    std::sort(bufs.begin(), bufs.end(),
              [](const GpuBuffer& a, const GpuBuffer& b) { return a.handle < b.handle; });
    std::set<BufferHandle> old;
    for (const auto& b : bufs_) old.insert(b.handle);
    bufs_ = std::move(bufs);
    std::vector<pos_buffer_desc> d;
    for (const auto& b : bufs_) d.push_back(b.desc());
    check(pos_update_buffer_set(ctx_, d.data(), static_cast<uint32_t>(d.size())));
    std::set<BufferHandle> kept;
    for (const auto& b : bufs_)
      if (dirty_.count(b.handle) || (new_ones_dirty && !old.count(b.handle))) kept.insert(b.handle);
    dirty_ = kept;
    std::vector<uint64_t> hs(dirty_.begin(), dirty_.end());
    if (!hs.empty()) check(pos_record_dirty(ctx_, hs.data(), static_cast<uint32_t>(hs.size())));
  }

  // plan_precopy (cr.hpp:377-406): O2 digests + O1 verdicts + O3 pack.
  // Returns the pre-copy pack (at cache offset 0).
  PackRef plan_precopy(void* stream = nullptr) {
    check(pos_precopy(ctx_, 1, stream));
    uint64_t n = 0;
    check(pos_precopy_size(ctx_, &n));
    return PackRef{0, n};
  }

  // Wave-pipelined variant with the D2H into host_dst (same offsets).
  std::vector<PackRef> plan_precopy_pipelined(void* host_dst, uint32_t waves, void* ckpt_stream,
                                              void* copy_stream) {
    uint64_t off[16], sz[16];
    uint32_t n = 0;
    check(pos_precopy_pipelined(ctx_, 1, waves, ckpt_stream, copy_stream, host_dst, 0, off, sz, &n));
    std::vector<PackRef> out;
    for (uint32_t i = 0; i < n; ++i) out.push_back({off[i], sz[i]});
    return out;
  }

  // dedup_verdicts() (cr.hpp:141): buffers with provenance only.
  std::map<BufferHandle, bool> dedup_verdicts(void* stream = nullptr) {
    std::vector<uint32_t> crcs(bufs_.size());
    std::vector<uint8_t> v(bufs_.size());
    check(pos_buffer_crc(ctx_, stream));
    check(pos_read_buffer_crcs(ctx_, crcs.data(), v.data(), static_cast<uint32_t>(v.size()), stream));
    std::map<BufferHandle, bool> out;
    for (size_t i = 0; i < bufs_.size(); ++i)
      if (bufs_[i].upstream) out[bufs_[i].handle] = v[i] != 0;
    return out;
  }

  // record_dirty (cr.hpp:901-931): DAG spec_writes -> dirty_set_.
  void record_dirty(const std::vector<BufferHandle>& writes) {
    check(pos_record_dirty(ctx_, writes.data(), static_cast<uint32_t>(writes.size())));
    for (BufferHandle h : writes)
      for (const auto& b : bufs_)
        if (b.handle == h) dirty_.insert(h);  // handles outside the snapshot are ignored (cr.hpp:904)
  }
  const std::set<BufferHandle>& dirty_set() const { return dirty_; }

  // Eager delta capture: DAG-dirty buffers whose last writer is already on
  // after_stream are gathered into the prepared delta pack now; the stop
  // gathers only the rest (pos_delta_pregather).
  void prepare_final_stop(void* stream = nullptr) { check(pos_delta_prepare(ctx_, stream, nullptr, nullptr)); }
  void pregather(const std::vector<BufferHandle>& done_writing, void* after_stream, void* stream = nullptr) {
    check(pos_delta_pregather(ctx_, done_writing.data(), static_cast<uint32_t>(done_writing.size()), after_stream,
                              stream));
  }

  // at_final_stop (cr.hpp:599-621): the STW delta pack.
  PackRef at_final_stop(void* stream = nullptr) {
    PackRef r;
    check(pos_delta_copy(ctx_, stream, &r.offset, &r.bytes));
    return r;
  }
  // Same, the stop-the-world window delimited by events stw_begin / stw_end
  // and holding only the gather (pos_final_stop).
  PackRef at_final_stop(void* stream, int stw_begin, int stw_end) {
    PackRef r;
    check(pos_final_stop(ctx_, stream, stw_begin, stw_end, &r.offset, &r.bytes));
    return r;
  }

  void d2h(void* pinned_dst, const PackRef& p, void* stream = nullptr) {
    check(pos_d2h_async(ctx_, pinned_dst, p.offset, p.bytes, 0, stream));
  }

  // materialize / load_complete (cr.hpp:1026-1084): scatter a device-resident pack.
  void materialize(const void* pack_dev, uint64_t bytes, void* stream = nullptr) {
    check(pos_scatter(ctx_, reinterpret_cast<uint64_t>(pack_dev), bytes, stream));
  }

  // chunk_copied straight into the target's captured_ (cr.hpp:499-501): the
  // image of each snapshot buffer (ascending handle), then the direct pre-copy.
  void register_image(const std::vector<uint8_t*>& hosts) {
    std::vector<uint64_t> sizes;
    for (const auto& b : bufs_) sizes.push_back(b.size);
    if (hosts.size() != bufs_.size()) throw SimError(Errc::InvalidArgument, "one image per buffer");
    check(pos_register_image(ctx_, hosts.data(), sizes.data(), static_cast<uint32_t>(hosts.size())));
  }
  void plan_precopy_direct(uint32_t waves, void* ckpt_stream, void* drain_stream) {
    check(pos_precopy_direct(ctx_, 1, waves, ckpt_stream, drain_stream));
  }
  // (chunks, payload bytes) the last direct pre-copy shipped.
  std::pair<uint64_t, uint64_t> direct_result() {
    uint64_t n = 0, pay = 0, idx = 0;
    check(pos_precopy_direct_result(ctx_, &n, &pay, &idx));
    return {n, pay};
  }
  void drain_final_stop(void* stream) { check(pos_delta_drain(ctx_, stream)); }

  // note_h2d_provenance (process.hpp:505-522) with the copy itself.
  void h2d(void* dst_dev, const void* host_src, uint64_t bytes, void* stream = nullptr) {
    check(pos_h2d_provenance(ctx_, reinterpret_cast<uint64_t>(dst_dev), host_src, bytes, 1, stream));
  }
  std::optional<uint32_t> upstream_crc(BufferHandle h) {
    uint32_t has = 0, crc = 0;
    check(pos_read_upstream(ctx_, h, &has, &crc));
    return has ? std::optional<uint32_t>(crc) : std::nullopt;
  }

  // gate_cow -> stage_buffers (cr.hpp:806-888): stop-point bytes of the
  // conflicting writers into a staging pack, on the writer's stream.
  PackRef stage_buffers(const std::vector<BufferHandle>& conflicts, void* app_stream) {
    PackRef r;
    check(pos_stage_buffers(ctx_, conflicts.data(), static_cast<uint32_t>(conflicts.size()), app_stream,
                            &r.offset, &r.bytes));
    return r;
  }

  // restore (cr.hpp:167-204) from a flat image: start_loads in `order`,
  // gate_restore per kernel buffer, all_loaded.
  void restore_begin(const std::vector<uint8_t*>& hosts, const std::vector<BufferHandle>& order,
                     void* h2d_stream) {
    std::vector<uint64_t> sizes;
    for (const auto& b : bufs_) sizes.push_back(b.size);
    check(pos_restore_image_begin(ctx_, hosts.data(), sizes.data(), static_cast<uint32_t>(hosts.size()),
                                  order.data(), static_cast<uint32_t>(order.size()), 0, h2d_stream));
  }
  void gate_restore(BufferHandle h, void* stream) { check(pos_restore_gate(ctx_, h, stream)); }
  void restore_wait() { check(pos_restore_image_wait(ctx_)); }

  // read_image + materialize (image.hpp:209-361, cr.hpp:1026-1030): restore a
  // POSI image onto the snapshot's buffers; returns (loaded, recompute).
  std::pair<uint32_t, uint32_t> restore_image(const std::vector<uint8_t>& posi, void* stream = nullptr) {
    uint64_t off = 0;
    uint32_t loaded = 0, recompute = 0;
    int rc = pos_image_restore(ctx_, posi.data(), posi.size(), stream, &off, &loaded, &recompute);
    if (rc == POS_E_CORRUPT_IMAGE) throw CorruptImageError(off, pos_last_error());
    check(rc);
    return {loaded, recompute};
  }

  // NVLink peer-GPU cache for the cache-cycled pre-copy (config 5).
  void attach_peer_cache(int peer_device, uint64_t bytes) {
    check(pos_peer_cache_attach(ctx_, peer_device, bytes));
  }

  // At finalize_image (cr.hpp:745, where the reference clears written_since_ckpt):
  // this epoch's digests become the baseline the next epoch compares with.
  void end_checkpoint_session() {
    check(pos_commit_epoch(ctx_));
    dirty_.clear();
  }

  std::vector<uint32_t> digests(void* stream = nullptr) {
    uint64_t n = 0;
    check(pos_num_chunks(ctx_, &n));
    std::vector<uint32_t> d(n);
    check(pos_read_digests(ctx_, d.data(), n, stream));
    return d;
  }
  std::vector<uint8_t> dirty_flags(void* stream = nullptr) {
    uint64_t n = 0;
    check(pos_num_chunks(ctx_, &n));
    std::vector<uint8_t> f(n);
    check(pos_read_flags(ctx_, f.data(), n, stream));
    return f;
  }
  pos_ctx* raw() { return ctx_; }
  const SimConfig& cfg() const { return cfg_; }

 private:
  SimConfig cfg_;
  pos_ctx* ctx_ = nullptr;
  std::vector<GpuBuffer> bufs_;
  std::set<BufferHandle> dirty_;
};

// Apply a host-resident pack onto host copies of the buffers (captured_,
// cr.hpp:499-501).  `captured` holds a vector per handle, sized to the buffer.
inline void apply_pack(const uint8_t* pack, uint64_t bytes,
                       std::map<BufferHandle, std::vector<uint8_t>>& captured, uint32_t threads = 1) {
  std::vector<uint64_t> handles, sizes;
  std::vector<uint8_t*> hosts;
  for (auto& [h, v] : captured) {
    handles.push_back(h);
    hosts.push_back(v.data());
    sizes.push_back(v.size());
  }
  check(pos_pack_apply_host(pack, bytes, handles.data(), hosts.data(), sizes.data(),
                            static_cast<uint32_t>(handles.size()), threads));
}

// ---- checkpoint image (image.hpp:42-207) --------------------------------------
enum class GpuRecordKind : uint8_t { Inline = 0, DedupRef = 1, Recompute = 2 };

struct HostPageRec {
  uint64_t index = 0;
  std::vector<uint8_t> bytes;
};
struct GpuBufferRec {
  BufferHandle handle = 0;
  GpuRecordKind kind = GpuRecordKind::Inline;
  std::vector<uint8_t> inline_bytes;
  uint64_t dedup_first_page = 0;
  uint32_t dedup_page_count = 0;
  uint32_t dedup_offset = 0;
  uint32_t dedup_crc = 0;
  std::vector<uint64_t> recompute_nodes;
};
struct AllocEntry {
  BufferHandle handle = 0;
  uint64_t base = 0;
  uint64_t size = 0;
};
struct ImageMeta {
  std::vector<uint64_t> stream_ids;
  std::vector<AllocEntry> allocs;
  uint64_t cursor = 0;
  uint64_t next_handle = 1;
  uint64_t next_base = 0x7000'0000'0000ull;  // kDeviceAddrBase (config.hpp:14)
};
struct CheckpointImage {
  uint64_t page_size = 4096;
  std::vector<HostPageRec> host_pages;
  std::vector<GpuBufferRec> gpu_records;
  std::vector<uint8_t> dag_bytes;
  ImageMeta meta;
};

// Byte-identical to gpucrsim::write_image (streaming, no deep copy).
// read_image's validation (image.hpp:209-361): throws CorruptImageError with
// the reference's offset.  (The DAG body is opaque to this reader.)
inline void read_image_check(const std::vector<uint8_t>& posi) {
  uint64_t off = 0;
  int rc = pos_image_check(posi.data(), posi.size(), &off);
  if (rc == POS_E_CORRUPT_IMAGE) throw CorruptImageError(off, pos_last_error());
  check(rc);
}

inline std::vector<uint8_t> write_image(const CheckpointImage& img) {
  std::vector<pos_image_page> pages;
  for (const auto& p : img.host_pages) {
    if (p.bytes.size() != img.page_size) throw SimError(Errc::InvariantViolation, "host page size mismatch");
    pages.push_back({p.index, p.bytes.data()});
  }
  std::vector<pos_image_rec> recs;
  for (const auto& r : img.gpu_records) {
    pos_image_rec x{};
    x.handle = r.handle;
    x.kind = static_cast<uint32_t>(r.kind);
    x.inline_bytes = r.inline_bytes.data();
    x.inline_len = r.inline_bytes.size();
    x.dedup_first_page = r.dedup_first_page;
    x.dedup_page_count = r.dedup_page_count;
    x.dedup_offset = r.dedup_offset;
    x.dedup_crc = r.dedup_crc;
    x.recompute = r.recompute_nodes.data();
    x.n_recompute = static_cast<uint32_t>(r.recompute_nodes.size());
    recs.push_back(x);
  }
  std::vector<pos_image_alloc> allocs;
  for (const auto& a : img.meta.allocs) allocs.push_back({a.handle, a.base, a.size});
  pos_image_desc d{};
  d.page_size = img.page_size;
  d.pages = pages.data();
  d.n_pages = static_cast<uint32_t>(pages.size());
  d.recs = recs.data();
  d.n_recs = static_cast<uint32_t>(recs.size());
  d.allocs = allocs.data();
  d.n_allocs = static_cast<uint32_t>(allocs.size());
  d.stream_ids = img.meta.stream_ids.data();
  d.n_streams = static_cast<uint32_t>(img.meta.stream_ids.size());
  d.cursor = img.meta.cursor;
  d.next_handle = img.meta.next_handle;
  d.next_base = img.meta.next_base;
  d.dag_bytes = img.dag_bytes.data();
  d.dag_len = img.dag_bytes.size();
  uint64_t size = 0;
  check(pos_image_write(&d, nullptr, 0, &size));
  std::vector<uint8_t> out(size);
  check(pos_image_write(&d, out.data(), out.size(), &size));
  return out;
}

}  // namespace posdump
