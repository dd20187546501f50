// ref_shim.cpp -- extern "C" wrappers over the UNMODIFIED reference headers
// (/root/reference/proj/include/gpucrsim), compiled by oracle/Makefile into
// oracle/_ref/libgpucrsim_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (posdump_oracle.c)
// against the reference's own code, to generate tests/golden/, and as the
// reference CPU arm of bench.py.  No reference source is copied here; the
// headers are included from where they lie.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <thread>
#include <vector>

#include <array>
#include <deque>
#include <fstream>
#include <functional>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <unordered_map>
#include <utility>

#include <json.hpp>

// ref_checkpoint_session reads CrEngine session state that finalize_image
// consumes but the class keeps private (final_outstanding_, retention_,
// dedup_snapshot_); every library header is included above, so only the
// reference's own classes see this.
#define private public
#include "gpucrsim/buffer.hpp"
#include "gpucrsim/crc32.hpp"
#include "gpucrsim/image.hpp"
#include "gpucrsim/rng.hpp"
#include "gpucrsim/workload.hpp"
#include "gpucrsim/scenario.hpp"
#undef private

#include <sstream>

using namespace gpucrsim;

extern "C" {

uint32_t ref_crc32(const void* p, uint64_t n) { return crc32(p, n); }
uint32_t ref_crc32_update(uint32_t c, const void* p, uint64_t n) { return crc32_update(c, p, n); }
uint64_t ref_mix64(uint64_t a, uint64_t b) { return mix64(a, b); }
uint64_t ref_fnv1a(const void* p, uint64_t n, uint64_t h) { return fnv1a(p, n, h); }
void ref_make_bytes(uint64_t seed, uint8_t* out, uint64_t n) {
  std::vector<uint8_t> v = make_bytes(seed, n);
  std::memcpy(out, v.data(), n);
}

// Chunk geometry through the reference's own allocator + GpuBuffer
// (buffer.hpp:44-49, :101-124).  Returns chunk count; fills out[] if given.
uint32_t ref_chunk_geometry(uint64_t size, uint64_t chunk_size, uint64_t* out) {
  DeviceMemory dev(size + (1ull << 20), chunk_size);
  BufferHandle h = dev.alloc(size);
  const GpuBuffer& b = dev.at(h);
  if (out)
    for (uint32_t i = 0; i < b.chunk_count(); ++i) out[i] = b.chunk_bytes(i);
  return b.chunk_count();
}

// ---- image encode/decode (image.hpp:136-361) -------------------------------

struct ref_rec_t {
  uint64_t handle;
  uint32_t kind;
  uint32_t n_recompute;
  const uint8_t* inline_bytes;
  uint64_t inline_len;
  uint64_t dedup_first_page;
  uint32_t dedup_page_count, dedup_offset, dedup_crc, pad;
  const uint64_t* recompute;
};
struct ref_alloc_t {
  uint64_t handle, base, size;
};
struct ref_page_t {
  uint64_t index;
  const uint8_t* bytes;
};

uint64_t ref_write_image(uint64_t page_size, const ref_page_t* pages, uint32_t npages,
                         const ref_rec_t* recs, uint32_t nrecs, const ref_alloc_t* allocs,
                         uint32_t nallocs, const uint64_t* streams, uint32_t nstreams,
                         uint64_t cursor, uint64_t next_handle, uint64_t next_base,
                         const uint8_t* dag, uint64_t dag_len, uint8_t* out, uint64_t cap) {
  CheckpointImage img;
  img.page_size = page_size;
  for (uint32_t i = 0; i < npages; ++i)
    img.host_pages.push_back({pages[i].index, {pages[i].bytes, pages[i].bytes + page_size}});
  for (uint32_t i = 0; i < nrecs; ++i) {
    GpuBufferRec r;
    r.handle = recs[i].handle;
    r.kind = static_cast<GpuRecordKind>(recs[i].kind);
    if (r.kind == GpuRecordKind::Inline)
      r.inline_bytes.assign(recs[i].inline_bytes, recs[i].inline_bytes + recs[i].inline_len);
    r.dedup_first_page = recs[i].dedup_first_page;
    r.dedup_page_count = recs[i].dedup_page_count;
    r.dedup_offset = recs[i].dedup_offset;
    r.dedup_crc = recs[i].dedup_crc;
    for (uint32_t k = 0; k < recs[i].n_recompute; ++k) r.recompute_nodes.push_back(recs[i].recompute[k]);
    img.gpu_records.push_back(std::move(r));
  }
  for (uint32_t i = 0; i < nallocs; ++i)
    img.meta.allocs.push_back({allocs[i].handle, allocs[i].base, allocs[i].size});
  for (uint32_t i = 0; i < nstreams; ++i) img.meta.stream_ids.push_back(streams[i]);
  img.meta.cursor = cursor;
  img.meta.next_handle = next_handle;
  img.meta.next_base = next_base;
  if (dag_len) img.dag_bytes.assign(dag, dag + dag_len);
  std::vector<uint8_t> bytes = write_image(img);
  if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
  return bytes.size();
}

// 0 = valid, else 1 + offset of the CorruptImageError (image.hpp:209-361).
uint64_t ref_read_image_check(const uint8_t* p, uint64_t n) {
  try {
    std::vector<uint8_t> v(p, p + n);
    (void)read_image(v);
    return 0;
  } catch (const CorruptImageError& e) {
    return 1 + e.offset();
  }
}

// ---- reference CPU dump path (the --impl reference arm) --------------------
// One "process" worth of GpuBuffers (buffer.hpp:27-97) plus the captured_
// map of CrEngine (cr.hpp:1300).  ref_state_dump runs, per chunk, the
// reference's digest crc32 (crc32.hpp:26-34) and, for dirty chunks, the
// chunk_copied() capture: read_content + std::copy into captured_[h]
// (cr.hpp:488-501).  Chunks are split across `threads` std::threads
// (parallel-for over chunks; the reference itself is single-threaded).
struct RefState {
  DeviceMemory dev;
  std::vector<BufferHandle> handles;
  std::map<BufferHandle, std::vector<uint8_t>> captured;
  uint64_t chunk_size;
  RefState(uint64_t cap, uint64_t cs) : dev(cap, cs), chunk_size(cs) {}
};

void* ref_state_create(uint32_t n, const uint64_t* sizes, const uint8_t* const* contents,
                       uint64_t chunk_size) {
  uint64_t total = 0;
  for (uint32_t i = 0; i < n; ++i) total += sizes[i];
  auto* s = new RefState(total + (1ull << 20), chunk_size);
  for (uint32_t i = 0; i < n; ++i) {
    BufferHandle h = s->dev.alloc(sizes[i]);
    s->dev.at(h).write_content(0, contents[i], sizes[i]);
    s->handles.push_back(h);
    s->captured[h].assign(sizes[i], 0);
  }
  return s;
}

void ref_state_destroy(void* p) { delete static_cast<RefState*>(p); }

// prev/cur are digest tables over global chunk order; flags out.  Returns
// number of dirty chunks.  prev_valid == 0 marks every chunk dirty (fresh).
uint64_t ref_state_dump(void* p, const uint32_t* prev, int prev_valid, uint32_t* cur,
                        uint8_t* flags, uint32_t threads) {
  auto* s = static_cast<RefState*>(p);
  std::vector<uint64_t> first(s->handles.size() + 1, 0);
  for (size_t i = 0; i < s->handles.size(); ++i)
    first[i + 1] = first[i] + s->dev.at(s->handles[i]).chunk_count();
  // Pre-touch captured_ entries so worker threads never mutate the map.
  std::vector<std::vector<uint8_t>*> dst;
  for (BufferHandle h : s->handles) dst.push_back(&s->captured[h]);
  std::vector<uint64_t> dirty(threads ? threads : 1, 0);
  // Thread t takes the contiguous global chunk range [N*t/nt, N*(t+1)/nt):
  // every chunk is independent (its own crc32, its own bytes of captured_),
  // so a state of a few huge buffers still keeps every core busy.
  const uint64_t N = first.back();
  auto work = [&](uint32_t t, uint32_t nt) {
    const uint64_t lo = N * t / nt, hi = N * (t + 1) / nt;
    size_t i = std::upper_bound(first.begin(), first.end(), lo) - first.begin() - 1;
    for (uint64_t g = lo; g < hi; ++g) {
      while (g >= first[i + 1]) ++i;
      const GpuBuffer& b = s->dev.at(s->handles[i]);
      const uint32_t ci = static_cast<uint32_t>(g - first[i]);
      const uint64_t off = static_cast<uint64_t>(ci) * b.chunk_size;
      const uint64_t len = b.chunk_bytes(ci);
      uint32_t d = crc32(b.content().data() + off, len);
      cur[g] = d;
      bool is_dirty = !prev_valid || prev[g] != d;
      flags[g] = is_dirty;
      if (!is_dirty) continue;
      ++dirty[t];
      std::vector<uint8_t> bytes = b.read_content(off, len);
      std::copy(bytes.begin(), bytes.end(), dst[i]->begin() + static_cast<ptrdiff_t>(off));
    }
  };
  uint32_t nt = threads ? threads : 1;
  if (nt == 1) {
    work(0, 1);
  } else {
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < nt; ++t) pool.emplace_back(work, t, nt);
    for (auto& th : pool) th.join();
  }
  uint64_t total = 0;
  for (uint64_t d : dirty) total += d;
  return total;
}

// Overwrite a byte range of buffer i (epoch writes for the baseline).
void ref_state_write(void* p, uint32_t i, uint64_t off, const uint8_t* data, uint64_t len) {
  auto* s = static_cast<RefState*>(p);
  s->dev.at(s->handles[i]).write_content(off, data, len);
}

// Copy out captured_[h] of buffer i.
void ref_state_captured(void* p, uint32_t i, uint8_t* out) {
  auto* s = static_cast<RefState*>(p);
  const auto& v = s->captured[s->handles[i]];
  std::memcpy(out, v.data(), v.size());
}

// gen_workload (workload.hpp:162-410) for a named desk profile
// (workload.hpp:461-529) with total_bytes / kernel durations overridden; the
// trace as JSON lines (api.hpp:125-160).  Returns the byte length.
uint64_t ref_gen_workload(const char* profile, uint64_t total_bytes, uint64_t p50_ns,
                          uint64_t p99_ns, uint64_t seed, char* out, uint64_t cap) {
  WorkloadProfile p = profile_by_name(profile, seed);
  if (total_bytes) p.total_bytes = total_bytes;
  if (p50_ns) p.p50_ns = p50_ns;
  if (p99_ns) p.p99_ns = p99_ns;
  std::ostringstream os;
  write_trace(os, gen_workload(p));
  std::string s = os.str();
  if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
  return s.size();
}

// The reference engine end to end: generate a trace (desk profile with
// total_bytes override, or a fuzz trace when profile == "fuzz"), checkpoint it
// with checkpoint_at (scenario.hpp:63-78) at default_trigger (mid-trace
// iteration boundary), mode 1 = StopTheWorld, 3 = DirtyBitCheckpoint; return the
// POSI bytes of the image (write_image, image.hpp:136-207).
uint64_t ref_checkpoint_image(const char* profile, uint64_t total_bytes, uint64_t seed, int mode,
                              uint8_t* out, uint64_t cap) {
  std::vector<ApiCall> trace;
  if (std::string(profile) == "fuzz") {
    trace = gen_fuzz_trace(seed);
  } else {
    WorkloadProfile p = profile_by_name(profile, seed);
    if (total_bytes) p.total_bytes = total_bytes;
    trace = gen_workload(p);
  }
  SimConfig cfg;
  auto [img, metrics] = checkpoint_at(trace, default_trigger(trace), static_cast<CrMode>(mode), cfg);
  std::vector<uint8_t> bytes = write_image(img);
  if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
  return bytes.size();
}

// The reference engine's finalize_image INPUTS for one checkpoint (the state
// cr.hpp:680-764 reads), so a test can derive the record kinds itself:
// checkpoint_at's flow (scenario.hpp:63-78) with resume_after = false, so the
// process stays exactly as finalize_image saw it when `done` runs.  Blob
// (little endian): "SESS", u32 n, u64 image_len, image bytes, 8 x u64
// metrics {bytes_precopy, bytes_dirty, bytes_dedup_saved,
// bytes_recompute_saved, image_bytes, image_file_bytes, dirty_count,
// retention}, then per allocation of the image: u64 handle, base, size;
// u32 has_upstream; u64 up_host_addr, up_len; u32 up_crc, host_untouched;
// i32 dedup_ok (-1: not scanned); u32 dirty, recompute_eligible, n_pending;
// u64 pending[n_pending]; u64 content_len; content.  Returns the blob size.
static bool shim_recompute_eligible(GpuProcess& p, BufferHandle h) {  // restates cr.hpp:938-951
  auto first = p.dag().first_pending_accessor(h);
  if (!first) return false;
  const KernelNode& n = p.dag().at(*first);
  if (n.kind == ApiKind::LaunchOpaque) return false;
  bool writes = std::find(n.spec_writes.begin(), n.spec_writes.end(), h) != n.spec_writes.end();
  bool reads = std::find(n.spec_reads.begin(), n.spec_reads.end(), h) != n.spec_reads.end();
  if (!writes || reads) return false;
  for (uint64_t id : p.dag().pending_in_order()) {
    if (id == *first) break;
    if (p.dag().at(id).kind == ApiKind::LaunchOpaque) return false;
  }
  return true;
}

static std::vector<ApiCall> shim_trace(const char* profile, uint64_t total_bytes, uint64_t seed) {
  if (std::string(profile) == "fuzz") return gen_fuzz_trace(seed);
  WorkloadProfile p = profile_by_name(profile, seed);
  if (total_bytes) p.total_bytes = total_bytes;
  return gen_workload(p);
}

uint64_t ref_checkpoint_session(const char* profile, uint64_t total_bytes, uint64_t seed, int mode, uint8_t* out,
                                uint64_t cap) {
  std::vector<ApiCall> trace = shim_trace(profile, total_bytes, seed);
  SimConfig cfg;
  SimCell cell(cfg, trace);
  std::vector<uint8_t> blob;
  auto put = [&](const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    blob.insert(blob.end(), b, b + n);
  };
  auto u32 = [&](uint32_t v) { put(&v, 4); };
  auto u64 = [&](uint64_t v) { put(&v, 8); };
  bool fired = false;
  std::set<BufferHandle> recopied;  // final_outstanding_ as at_final_stop left it
  auto fire = [&] {
    cell.cr.checkpoint(static_cast<CrMode>(mode), CheckpointTarget{}, [&](CheckpointImage img) {
      fired = true;
      std::vector<uint8_t> bytes = write_image(img);
      const CrMetrics& m = cell.cr.metrics;
      put("SESS", 4);
      u32(static_cast<uint32_t>(img.meta.allocs.size()));
      u64(bytes.size());
      put(bytes.data(), bytes.size());
      for (uint64_t v : {m.bytes_precopy, m.bytes_dirty, m.bytes_dedup_saved, m.bytes_recompute_saved,
                         m.image_bytes, m.image_file_bytes, m.dirty_count, (uint64_t)m.retention})
        u64(v);
      const CrEngine& cr = cell.cr;
      for (const auto& a : img.meta.allocs) {
        const GpuBuffer& b = cell.proc.device().at(a.handle);
        u64(a.handle);
        u64(a.base);
        u64(a.size);
        // dedup_snapshot_ (cr.hpp:436) when scanned, else the live provenance
        auto ds = cr.dedup_snapshot_.find(a.handle);
        const std::optional<Upstream> up =
            ds != cr.dedup_snapshot_.end() ? std::optional<Upstream>(ds->second) : b.upstream;
        u32(up ? 1 : 0);
        u64(up ? up->host_addr : 0);
        u64(up ? up->len : 0);
        u32(up ? up->crc : 0);
        u32(up ? (cell.proc.host().range_write_seq(up->host_addr, up->len) <= up->host_write_seq) : 0);
        const auto& v = cell.cr.dedup_verdicts();
        auto it = v.find(a.handle);
        u32(static_cast<uint32_t>(it == v.end() ? -1 : (it->second ? 1 : 0)));
        u32(cell.cr.dirty_set().count(a.handle) ? 1 : 0);
        // bit 0: recompute_eligible; bit 1: re-copied at the final stop
        // (final_outstanding_); bit 2: retention_ && fully_copied && not
        // re-copied (its pre-copy survived, cr.hpp:741)
        // (recorded right after at_final_stop ran; retention_ itself is
        // reset before `done`, metrics.retention keeps it)
        const bool outstanding = recopied.count(a.handle) > 0;
        u32((shim_recompute_eligible(cell.proc, a.handle) ? 1u : 0u) | (outstanding ? 2u : 0u) |
            (m.retention && b.fully_copied() ? 4u : 0u));
        std::vector<uint64_t> pw = cell.proc.dag().pending_writers(a.handle);
        u32(static_cast<uint32_t>(pw.size()));
        for (uint64_t id : pw) u64(id);
        u64(b.size);
        put(b.content().data(), b.size);
      }
    }, /*resume_after=*/false);
  };
  if (!trace.empty() && default_trigger(trace) <= trace.back().seq)
    cell.runner->set_trigger(default_trigger(trace), fire);
  else
    cell.runner->on_finished = fire;
  cell.runner->start();
  bool stopped = false;
  while (cell.clk.step())  // event by event: catch the final stop's re-copy set
    if (!stopped && cell.cr.phase_ >= CrEngine::Phase::Final && cell.cr.mode_ != CrMode::None &&
        cell.cr.drained_at_ != 0) {  // at_final_stop has run (it stamps drained_at_)
      stopped = true;
      recopied = cell.cr.final_outstanding_;
    }
  if (!fired) return 0;
  if (out && cap >= blob.size()) std::memcpy(out, blob.data(), blob.size());
  return blob.size();
}

// ---- P5: restore parity (scenario.hpp:51-90, process.hpp:65-90) ----------

uint64_t ref_fnv1a_u64(uint64_t v, uint64_t h) { return fnv1a_u64(v, h); }

// StateSnapshot::hash (process.hpp:76-89) of a state given as arrays:
// buffers (ascending handle) and host pages (only non-zero ones count).
uint64_t ref_snapshot_hash(uint32_t nb, const uint64_t* handles, const uint64_t* bases, const uint64_t* sizes,
                           const uint8_t* const* contents, uint32_t np, const uint64_t* idx,
                           const uint8_t* const* pages, uint64_t page_size) {
  StateSnapshot s;
  for (uint32_t i = 0; i < nb; ++i) {
    StateSnapshot::Buf b;
    b.base = bases[i];
    b.size = sizes[i];
    b.content.assign(contents[i], contents[i] + sizes[i]);
    s.buffers[handles[i]] = std::move(b);
  }
  for (uint32_t i = 0; i < np; ++i) {
    std::vector<uint8_t> v(pages[i], pages[i] + page_size);
    if (std::any_of(v.begin(), v.end(), [](uint8_t x) { return x != 0; })) s.pages[idx[i]] = std::move(v);
  }
  return s.hash();
}

// restore_state(read_image(img), cfg, Full).hash() (scenario.hpp:81-90).
uint64_t ref_restore_hash(const uint8_t* img, uint64_t n) {
  SimConfig cfg;
  return restore_state(read_image(std::vector<uint8_t>(img, img + n)), cfg, RestoreKind::Full).hash();
}

// plain_final_state(trace, cfg, limit).hash() (scenario.hpp:51-58).
uint64_t ref_plain_hash(const char* profile, uint64_t total_bytes, uint64_t seed, uint64_t limit) {
  SimConfig cfg;
  return plain_final_state(shim_trace(profile, total_bytes, seed), cfg, limit).hash();
}

// The delta-restore replay plan of an image (replay_pending, cr.hpp:1099-1101):
// its DAG's pending nodes in order.  Per node: u32 kind (ApiKind), u32
// name_len, name, u64 seq, u64 dst, u64 src, u64 bytes, u32 nr, u64
// true_reads[nr], u32 nw, u64 true_writes[nw].  Returns the blob size.
uint64_t ref_replay_plan(const uint8_t* img, uint64_t n, uint8_t* out, uint64_t cap) {
  CheckpointImage im = read_image(std::vector<uint8_t>(img, img + n));
  std::vector<uint8_t> blob;
  auto put = [&](const void* p, size_t k) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    blob.insert(blob.end(), b, b + k);
  };
  auto u32 = [&](uint32_t v) { put(&v, 4); };
  auto u64 = [&](uint64_t v) { put(&v, 8); };
  if (!im.dag_bytes.empty()) {
    KernelDag dag = KernelDag::deserialize(im.dag_bytes);
    for (uint64_t id : dag.pending_in_order()) {
      const KernelNode& k = dag.at(id);
      u32(static_cast<uint32_t>(k.kind));
      u32(static_cast<uint32_t>(k.name.size()));
      put(k.name.data(), k.name.size());
      u64(k.seq);
      u64(k.args.size() > 0 ? k.args[0].v : 0);
      u64(k.args.size() > 1 ? k.args[1].v : 0);
      u64(k.bytes);
      u32(static_cast<uint32_t>(k.true_reads.size()));
      for (auto h : k.true_reads) u64(h);
      u32(static_cast<uint32_t>(k.true_writes.size()));
      for (auto h : k.true_writes) u64(h);
    }
  }
  if (out && cap >= blob.size()) std::memcpy(out, blob.data(), blob.size());
  return blob.size();
}

}  // extern "C"
