// C++ parity tests over include/posdump.hpp, written like the reference's own
// Catch2 suites (proj/tests/test_memory.cpp, test_cr.cpp, test_image.cpp).
// Names tagged [cpu] need no device; [gpu] cases run on the B200.  Expected
// values come from the reference's known answers and from the C restatement
// (oracle/liboracle.so, test infrastructure).
#include <cstdio>
#include <cstring>
#include <map>
#include <vector>

#include "../../include/posdump.hpp"
#include "../../oracle/posdump_oracle.h"
#include "minicatch.hpp"

using namespace posdump;

namespace {

// A device allocation with a host mirror filled by fill_bytes(seed) (rng.hpp:43-54).
struct DevBuf {
  uint64_t ptr = 0, size = 0;
  std::vector<uint8_t> host;
  DevBuf(uint64_t n, uint64_t seed) : size(n), host(n) {
    check(pos_dev_malloc(n, &ptr));
    check(pos_fill(ptr, n, seed, nullptr));
    or_fill_bytes(seed, host.data(), n);
  }
  ~DevBuf() { pos_dev_free(ptr); }
  void write(uint64_t off, uint64_t n, uint64_t seed) {
    check(pos_fill(ptr + off, n, seed, nullptr));
    or_fill_bytes(seed, host.data() + off, n);
  }
};

std::vector<uint8_t> pinned_d2h(DumpEngine& e, const PackRef& p) {
  void* h = nullptr;
  check(pos_host_malloc_pinned(p.bytes, &h));
  e.d2h(h, p);
  check(pos_device_sync());
  std::vector<uint8_t> out(static_cast<uint8_t*>(h), static_cast<uint8_t*>(h) + p.bytes);
  pos_host_free_pinned(h);
  return out;
}

uint32_t pack_entries(const std::vector<uint8_t>& pack) {
  uint32_t n;
  std::memcpy(&n, pack.data() + 16, 4);
  return n;
}

}  // namespace

// ---------------------------------------------------------------------------- [cpu]

TEST_CASE("[cpu] empty image is exactly the 64-byte header") {  // test_image.cpp:86-95
  CheckpointImage img;
  std::vector<uint8_t> bytes = write_image(img);
  REQUIRE(bytes.size() == 64);
  REQUIRE(std::memcmp(bytes.data(), "POSI", 4) == 0);
}

TEST_CASE("[cpu] write_image is canonical: records and allocations sorted by handle") {
  CheckpointImage a;
  a.gpu_records.push_back({3, GpuRecordKind::Inline, {1, 2, 3}});
  a.gpu_records.push_back({1, GpuRecordKind::Inline, {9}});
  a.meta.allocs = {{3, 0x7000'0000'0100ull, 3}, {1, 0x7000'0000'0000ull, 1}};
  CheckpointImage b = a;
  std::swap(b.gpu_records[0], b.gpu_records[1]);
  std::swap(b.meta.allocs[0], b.meta.allocs[1]);
  REQUIRE(write_image(a) == write_image(b));
}

TEST_CASE("[cpu] a gpu record without an allocation entry is an invariant violation") {
  CheckpointImage img;  // image.hpp:152-154
  img.gpu_records.push_back({7, GpuRecordKind::Inline, {0, 0, 0, 0}});
  REQUIRE_THROWS_AS(write_image(img), SimError);
  try {
    write_image(img);
  } catch (const SimError& e) {
    REQUIRE(e.code() == Errc::InvariantViolation);
  }
}

TEST_CASE("[cpu] chunk_size 0 is rejected like SimConfig::from_json") {  // config.hpp:70-71
  SimConfig cfg;
  cfg.chunk_size = 0;
  try {
    DumpEngine e(cfg);
    REQUIRE(false);
  } catch (const SimError& e) {
    REQUIRE(e.code() == Errc::InvalidArgument);
  }
}

TEST_CASE("[cpu] chunk geometry covers the buffer with a short tail") {  // test_memory.cpp:89-99
  GpuBuffer b;
  b.size = 10000;
  REQUIRE(b.chunk_count(4096) == 3);
  REQUIRE(b.chunk_bytes(0, 4096) == 4096);
  REQUIRE(b.chunk_bytes(2, 4096) == 10000 - 2 * 4096);
}

// ---------------------------------------------------------------------------- [gpu]

TEST_CASE("[gpu] crc32 known vector over device memory") {  // test_memory.cpp:10-17
  uint64_t p = 0;
  check(pos_dev_malloc(16, &p));
  check(pos_memcpy(p, reinterpret_cast<uint64_t>("123456789"), 9, 1, nullptr));
  check(pos_device_sync());
  const void* d = reinterpret_cast<const void*>(p);
  REQUIRE(crc32(d, 9) == 0xCBF43926u);
  uint32_t c = crc32_update(0, d, 4);
  c = crc32_update(c, static_cast<const uint8_t*>(d) + 4, 5);
  REQUIRE(c == 0xCBF43926u);
  pos_dev_free(p);
}

TEST_CASE("[gpu] chunk digests are the reference crc32 of every chunk, tail included") {
  SimConfig cfg;
  cfg.chunk_size = 4096;
  cfg.cache_capacity = 1 << 20;
  DumpEngine e(cfg);
  DevBuf a(10000, 2);  // test_memory.cpp:89-99 geometry; SURVEY App. A digests
  e.snapshot({GpuBuffer{1, a.ptr, a.size}});
  e.plan_precopy();
  std::vector<uint32_t> d = e.digests();
  REQUIRE(d.size() == 3);
  REQUIRE(d[0] == 0x7909527eu && d[1] == 0x6fba4432u && d[2] == 0xf994e5fdu);
  for (uint32_t c = 0; c < 3; ++c)
    REQUIRE(d[c] == or_crc32(a.host.data() + c * 4096ull, GpuBuffer{1, 0, 10000}.chunk_bytes(c, 4096)));
}

TEST_CASE("[gpu] no writes during pre-copy leaves the final transfer empty") {  // test_cr.cpp:225-240
  SimConfig cfg;
  cfg.cache_capacity = 8 << 20;
  DumpEngine e(cfg);
  DevBuf a(65536, 11);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}});
  PackRef first = e.plan_precopy();  // fresh target: everything ships (bytes_precopy == 64 KiB)
  REQUIRE(pack_entries(pinned_d2h(e, first)) == 1);
  e.end_checkpoint_session();
  PackRef again = e.plan_precopy();  // incremental round, nothing written
  REQUIRE(pack_entries(pinned_d2h(e, again)) == 0);
  REQUIRE(e.dirty_set().empty());  // dirty_count == 0
  PackRef fin = e.at_final_stop();   // bytes_dirty == 0
  REQUIRE(pack_entries(pinned_d2h(e, fin)) == 0);
}

TEST_CASE("[gpu] dedup: clean upstream dedups, any rewrite falls back to inline bytes") {
  // test_cr.cpp:375-415: clean -> DedupRef, rewritten -> Inline, host-touched -> Inline
  SimConfig cfg;
  cfg.cache_capacity = 8 << 20;
  DumpEngine e(cfg);
  DevBuf clean(65536, 21), rewritten(65536, 22), touched(65536, 23);
  GpuBuffer b1{1, clean.ptr, clean.size}, b2{2, rewritten.ptr, rewritten.size}, b3{3, touched.ptr, touched.size};
  b1.upstream = Upstream{0x1000, 65536, or_crc32(clean.host.data(), 65536), 1, true};
  b2.upstream = Upstream{0x20000, 65536, or_crc32(rewritten.host.data(), 65536), 1, true};
  b3.upstream = Upstream{0x40000, 65536, or_crc32(touched.host.data(), 65536), 1, false};
  rewritten.write(100, 8, 99);
  check(pos_device_sync());
  e.snapshot({b1, b2, b3});
  PackRef p = e.plan_precopy();
  auto v = e.dedup_verdicts();
  REQUIRE(v.at(1) == true);
  REQUIRE(v.at(2) == false);
  REQUIRE(v.at(3) == false);
  // the dedup-ok buffer is not packed: bytes_dedup_saved == 64 KiB
  std::vector<uint8_t> pack = pinned_d2h(e, p);
  REQUIRE(pack_entries(pack) == 2);
  std::map<BufferHandle, std::vector<uint8_t>> cap{{1, std::vector<uint8_t>(65536)},
                                                   {2, std::vector<uint8_t>(65536)},
                                                   {3, std::vector<uint8_t>(65536)}};
  apply_pack(pack.data(), pack.size(), cap);
  REQUIRE(cap[2] == rewritten.host);
  REQUIRE(cap[3] == touched.host);
}

TEST_CASE("[gpu] dirty-bit checkpoint: pre-copy + final delta rebuild the state byte for byte") {
  SimConfig cfg;
  cfg.chunk_size = 65536;
  cfg.cache_capacity = 16 << 20;
  DumpEngine e(cfg);
  DevBuf a(300000, 31), b(65536 * 3, 32), c(777, 33);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}, GpuBuffer{2, b.ptr, b.size}, GpuBuffer{3, c.ptr, c.size}});
  std::map<BufferHandle, std::vector<uint8_t>> captured{
      {1, std::vector<uint8_t>(a.size)}, {2, std::vector<uint8_t>(b.size)}, {3, std::vector<uint8_t>(c.size)}};
  auto ship = [&](const PackRef& p) {
    std::vector<uint8_t> pk = pinned_d2h(e, p);
    apply_pack(pk.data(), pk.size(), captured, 2);
  };
  ship(e.plan_precopy());
  e.end_checkpoint_session();
  a.write(65536 + 3, 10, 41);  // one chunk of buffer 1 changes before the round
  check(pos_device_sync());
  PackRef pre = e.plan_precopy();
  ship(pre);
  e.record_dirty({2, 999});  // a kernel of the window writes buffer 2; 999 is not in the snapshot
  REQUIRE(e.dirty_set() == std::set<BufferHandle>{2});
  b.write(0, b.size, 42);
  check(pos_device_sync());
  PackRef fin = e.at_final_stop(nullptr, 3, 4);  // STW window = [event 3, gather, event 4]
  REQUIRE(fin.offset >= pre.bytes);
  float stw_ms = 0;
  check(pos_event_elapsed(e.raw(), 3, 4, &stw_ms));
  REQUIRE(stw_ms > 0);
  ship(fin);
  REQUIRE(captured[1] == a.host);
  REQUIRE(captured[2] == b.host);
  REQUIRE(captured[3] == c.host);
  // Inline image of the captured state == image of the live device state
  CheckpointImage img;
  for (auto& [h, bytes] : captured) {
    img.gpu_records.push_back({h, GpuRecordKind::Inline, bytes});
    img.meta.allocs.push_back({h, 0x7000'0000'0000ull + 0x100000 * h, bytes.size()});
  }
  CheckpointImage want = img;
  want.gpu_records[0].inline_bytes = a.host;
  want.gpu_records[1].inline_bytes = b.host;
  want.gpu_records[2].inline_bytes = c.host;
  REQUIRE(write_image(img) == write_image(want));
}

TEST_CASE("[gpu] a buffer allocated mid-session joins dirty, a freed one is dropped") {  // cr.hpp:298-306
  SimConfig cfg;
  cfg.chunk_size = 4096;
  cfg.cache_capacity = 4 << 20;
  DumpEngine e(cfg);
  DevBuf a(3 * 4096 + 5, 61), b(5000, 62), c(100, 63);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}, GpuBuffer{2, b.ptr, b.size}, GpuBuffer{3, c.ptr, c.size}});
  std::map<BufferHandle, std::vector<uint8_t>> captured{
      {1, std::vector<uint8_t>(a.size)}, {2, std::vector<uint8_t>(b.size)}, {3, std::vector<uint8_t>(c.size)}};
  auto ship = [&](const PackRef& p) {
    std::vector<uint8_t> pk = pinned_d2h(e, p);
    apply_pack(pk.data(), pk.size(), captured, 2);
  };
  ship(e.plan_precopy());
  e.end_checkpoint_session();
  DevBuf d(2 * 4096, 64);  // allocated during the next session
  a.write(4096 + 1, 7, 65);
  check(pos_device_sync());
  e.update_snapshot({GpuBuffer{1, a.ptr, a.size}, GpuBuffer{3, c.ptr, c.size}, GpuBuffer{4, d.ptr, d.size}});
  REQUIRE(e.dirty_set() == std::set<BufferHandle>{4});
  captured.erase(2);
  captured[4] = std::vector<uint8_t>(d.size);
  PackRef pre = e.plan_precopy();  // buffer 1's rewritten chunk only (4 is DAG-dirty)
  ship(pre);
  PackRef fin = e.at_final_stop();  // the new buffer, whole
  ship(fin);
  REQUIRE(captured[1] == a.host);
  REQUIRE(captured[3] == c.host);
  REQUIRE(captured[4] == d.host);
}

TEST_CASE("[gpu] restore scatter rejects corrupt packs and unknown handles") {
  SimConfig cfg;
  cfg.chunk_size = 4096;
  cfg.cache_capacity = 1 << 20;
  DumpEngine e(cfg);
  DevBuf a(10000, 51);
  e.snapshot({GpuBuffer{4, a.ptr, a.size}});
  PackRef p = e.plan_precopy();
  std::vector<uint8_t> pk = pinned_d2h(e, p);
  uint64_t dev = 0;
  check(pos_dev_malloc(pk.size(), &dev));
  pk[0] = 'X';
  check(pos_memcpy(dev, reinterpret_cast<uint64_t>(pk.data()), pk.size(), 1, nullptr));
  check(pos_device_sync());
  REQUIRE_THROWS_AS(e.materialize(reinterpret_cast<void*>(dev), pk.size()), CorruptImageError);
  pk[0] = 'P';
  uint64_t bogus = 77;
  std::memcpy(pk.data() + 64, &bogus, 8);  // entry 0 names a handle not in the snapshot
  check(pos_memcpy(dev, reinterpret_cast<uint64_t>(pk.data()), pk.size(), 1, nullptr));
  check(pos_device_sync());
  try {
    e.materialize(reinterpret_cast<void*>(dev), pk.size());
    REQUIRE(false);
  } catch (const SimError& ex) {
    REQUIRE(ex.code() == Errc::InvalidLocator);
  }
  pos_dev_free(dev);
}

TEST_CASE("[gpu] staging exhaustion surfaces as StagingExhausted") {
  SimConfig cfg;
  cfg.chunk_size = 4096;
  cfg.cache_capacity = 16 * 4096;
  DumpEngine e(cfg);
  DevBuf a(64 * 4096, 61);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}});
  try {
    e.plan_precopy();
    REQUIRE(false);
  } catch (const SimError& ex) {
    REQUIRE(ex.code() == Errc::StagingExhausted);
  }
}

TEST_CASE("[gpu] eager delta capture: pregathered buffers land as the stop gather would") {  // cr.hpp:599-621
  SimConfig cfg;
  cfg.chunk_size = 4096;
  cfg.cache_capacity = 4 << 20;
  DumpEngine e(cfg);
  DevBuf a(5 * 4096 + 9, 81), b(6000, 82), c(4096 * 2, 83);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}, GpuBuffer{2, b.ptr, b.size}, GpuBuffer{3, c.ptr, c.size}});
  std::map<BufferHandle, std::vector<uint8_t>> captured{
      {1, std::vector<uint8_t>(a.size)}, {2, std::vector<uint8_t>(b.size)}, {3, std::vector<uint8_t>(c.size)}};
  auto ship = [&](const PackRef& p) {
    std::vector<uint8_t> pk = pinned_d2h(e, p);
    apply_pack(pk.data(), pk.size(), captured, 2);
  };
  ship(e.plan_precopy());
  e.record_dirty({1, 2, 3});
  e.prepare_final_stop();
  a.write(7, 5000, 84);
  b.write(0, b.size, 85);
  e.pregather({1, 2}, nullptr);  // behind their writers on the legacy stream
  c.write(100, 300, 86);
  b.write(10, 20, 87);           // a later writer of buffer 2: recorded, so the stop re-gathers it
  e.record_dirty({2});
  check(pos_device_sync());
  PackRef fin = e.at_final_stop(nullptr, 3, 4);
  ship(fin);
  REQUIRE(captured[1] == a.host);
  REQUIRE(captured[2] == b.host);
  REQUIRE(captured[3] == c.host);
}

int main(int argc, char** argv) { return minicatch::run(argc, argv); }

TEST_CASE("[gpu] direct pre-copy writes chunk_copied's bytes straight into captured_") {
  SimConfig cfg;
  cfg.chunk_size = 65536;
  cfg.cache_capacity = 8 << 20;
  DumpEngine e(cfg);
  DevBuf a(300000, 51), b(65536 * 3, 52);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}, GpuBuffer{2, b.ptr, b.size}});
  void* pin = nullptr;
  check(pos_host_malloc_pinned(a.size + b.size + 256, &pin));
  uint8_t* ia = static_cast<uint8_t*>(pin);
  uint8_t* ib = ia + (a.size + 255) / 256 * 256;
  std::memset(pin, 0, a.size + b.size + 256);
  e.register_image({ia, ib});
  void *s1 = nullptr, *s2 = nullptr;
  check(pos_stream_create(&s1));
  check(pos_stream_create(&s2));
  e.plan_precopy_direct(1, s1, s2);
  check(pos_device_sync());
  REQUIRE(e.direct_result().first == 5u + 3u);  // every chunk of a fresh target
  e.end_checkpoint_session();
  a.write(65536 + 3, 10, 61);
  check(pos_device_sync());
  e.record_dirty({2});  // the window's kernel is in the DAG from submission
  e.plan_precopy_direct(1, s1, s2);
  check(pos_device_sync());
  b.write(100, 50, 62);
  check(pos_device_sync());
  e.at_final_stop(s1);
  check(pos_stream_wait(s2, s1));
  e.drain_final_stop(s2);
  check(pos_device_sync());
  REQUIRE(e.direct_result().first == 1u);  // the one rewritten chunk of buffer 1
  REQUIRE(std::memcmp(ia, a.host.data(), a.size) == 0);
  REQUIRE(std::memcmp(ib, b.host.data(), b.size) == 0);
  pos_stream_destroy(s1);
  pos_stream_destroy(s2);
  pos_host_free_pinned(pin);
}

TEST_CASE("[gpu] CoW staging keeps the pre-write payload of a conflicting writer") {  // test_cr.cpp:106-127
  SimConfig cfg;
  cfg.chunk_size = 4096;
  cfg.cache_capacity = 4 << 20;
  DumpEngine e(cfg);
  DevBuf a(1 << 20, 71);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}});
  std::vector<uint8_t> before = a.host;
  void* app = nullptr;
  check(pos_stream_create(&app));
  PackRef st = e.stage_buffers({1}, app);
  REQUIRE(st.bytes > a.size);
  check(pos_fill(a.ptr, a.size, 72, app));  // the writer, after the gate on its own stream
  check(pos_device_sync());
  PackRef pre = e.plan_precopy();
  std::map<BufferHandle, std::vector<uint8_t>> captured{{1, std::vector<uint8_t>(a.size)}};
  std::vector<uint8_t> p1 = pinned_d2h(e, pre), p2 = pinned_d2h(e, st);
  REQUIRE(pack_entries(p1) == 0u);  // the staged buffer is not in the pre-copy
  apply_pack(p2.data(), p2.size(), captured, 1);
  REQUIRE(captured[1] == before);
  pos_stream_destroy(app);
}

TEST_CASE("[gpu] H2D provenance records crc32 of the payload and dedups the buffer") {  // test_api.cpp:76-98
  SimConfig cfg;
  cfg.chunk_size = 4096;
  cfg.cache_capacity = 1 << 20;
  DumpEngine e(cfg);
  DevBuf a(4096 * 40 + 7, 81);
  e.snapshot({GpuBuffer{1, a.ptr, a.size}});
  std::vector<uint8_t> payload(a.size);
  or_fill_bytes(82, payload.data(), payload.size());
  e.h2d(reinterpret_cast<void*>(a.ptr), payload.data(), payload.size());
  REQUIRE(e.upstream_crc(1).value() == or_crc32(payload.data(), payload.size()));
  PackRef pre = e.plan_precopy();
  REQUIRE(pack_entries(pinned_d2h(e, pre)) == 0u);  // O1: nothing to ship
}

TEST_CASE("[cpu] read_image rejects a truncated image at the reference's offset") {  // image.hpp:209-230
  CheckpointImage img;
  std::vector<uint8_t> bytes = write_image(img);
  read_image_check(bytes);  // the 64-byte empty image is valid
  bytes.resize(10);
  bool threw = false;
  try {
    read_image_check(bytes);
  } catch (const CorruptImageError& e) {
    threw = true;
    REQUIRE(e.offset() == 8u);  // flags u16 read at 6..8 succeeds; n_pages u32 at 8 is truncated
  }
  REQUIRE(threw);
}
