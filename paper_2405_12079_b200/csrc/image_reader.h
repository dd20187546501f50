// image_reader.h -- POSI v1 reader with read_image's validation
// (include/gpucrsim/image.hpp:209-361, ByteReader bytes.hpp:43-98): the same
// checks in the same order, failing with the reader position the reference's
// CorruptImageError carries.  The DAG section's structure is validated as
// KernelDag::deserialize does (posi_check_dag) and recompute nodes must exist
// in it; the DAG itself is not rebuilt (the kernel DAG is out of scope).
// DedupRef checksums are verified when `verify_dedup` is set (host CRC-32,
// crc32.hpp:26-34).
#pragma once
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace posdump {

struct PosiCorrupt {
  uint64_t offset;
  std::string reason;
};

struct PosiRecord {
  uint64_t handle = 0;
  uint8_t kind = 0;  // 0 Inline, 1 DedupRef, 2 Recompute
  const uint8_t* inline_bytes = nullptr;
  uint64_t inline_len = 0;
  uint64_t first_page = 0;
  uint32_t page_count = 0, offset = 0, crc = 0;
  std::vector<uint64_t> nodes;
};

struct PosiImage {
  uint64_t page_size = 0;
  std::vector<uint64_t> page_index;
  std::vector<const uint8_t*> page_bytes;
  std::vector<PosiRecord> recs;
  const uint8_t* dag = nullptr;
  uint64_t dag_len = 0;
  std::vector<uint64_t> streams;
  struct Alloc {
    uint64_t handle, base, size;
  };
  std::vector<Alloc> allocs;
  uint64_t cursor = 0, next_handle = 1, next_base = 0;
};

inline uint32_t posi_crc32(const uint8_t* p, uint64_t n) {  // reflected 0xEDB88320 (crc32.hpp:12-34)
  static uint32_t t[8][256];
  static bool init = [] {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
      t[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int s = 1; s < 8; ++s) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xff];
    return true;
  }();
  (void)init;
  uint32_t c = 0xFFFFFFFFu;
  while (n >= 8) {  // slicing by 8
    uint32_t lo, hi;
    std::memcpy(&lo, p, 4);
    std::memcpy(&hi, p + 4, 4);
    lo ^= c;
    c = t[7][lo & 0xff] ^ t[6][(lo >> 8) & 0xff] ^ t[5][(lo >> 16) & 0xff] ^ t[4][lo >> 24] ^ t[3][hi & 0xff] ^
        t[2][(hi >> 8) & 0xff] ^ t[1][(hi >> 16) & 0xff] ^ t[0][hi >> 24];
    p += 8;
    n -= 8;
  }
  while (n--) c = t[0][(c ^ *p++) & 0xff] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

class PosiReader {
 public:
  PosiReader(const uint8_t* d, uint64_t n) : d_(d), n_(n) {}
  uint64_t pos() const { return pos_; }
  uint64_t remaining() const { return n_ - pos_; }
  [[noreturn]] void fail(const std::string& why) const { throw PosiCorrupt{pos_, why}; }
  const uint8_t* take(uint64_t k) {
    if (k > n_ - pos_) fail("truncated input");
    const uint8_t* p = d_ + pos_;
    pos_ += k;
    return p;
  }
  uint8_t u8() { return *take(1); }
  template <typename T>
  T load() {
    T v;
    std::memcpy(&v, take(sizeof(T)), sizeof(T));
    return v;
  }

 private:
  const uint8_t* d_;
  uint64_t n_, pos_ = 0;
};

// The KDAG section's structure, as read_image checks it through
// KernelDag::deserialize (dag.hpp:322-387; image.hpp:309-319): node records
// (buffer u64 | kernel: id, seq, stream, api kind < 12, name, duration,
// bytes, args x 12 B, four u64 vectors, state <= 2), each exactly its
// declared length, then the edge table (kind <= 2) and nothing after it.
// A bounded read that runs out fails like the reference's ByteReader -- a
// CorruptImageError at the position inside the DAG bytes, rethrown as is;
// a structural error is CorruptDag, which read_image reports at offset 0 as
// "dag: ...".  Returns the kernel node ids (the recompute lists' domain).
inline std::set<uint64_t> posi_check_dag(const uint8_t* d, uint64_t n) {
  PosiReader rd(d, n);
  auto corrupt_dag = [](const std::string& why) -> void { throw PosiCorrupt{0, "dag: " + why}; };
  auto vec = [&rd]() {
    const uint32_t k = rd.load<uint32_t>();
    if ((uint64_t)k * 8 > rd.remaining()) rd.fail("vector length past end");
    rd.take((uint64_t)k * 8);
  };
  if (std::memcmp(rd.take(4), "KDAG", 4) != 0) corrupt_dag("bad magic");
  if (rd.load<uint32_t>() != 1) corrupt_dag("unsupported version");
  const uint32_t count = rd.load<uint32_t>();
  std::set<uint64_t> ids;
  for (uint32_t i = 0; i < count; ++i) {
    const uint32_t len = rd.load<uint32_t>();
    if (len > rd.remaining()) corrupt_dag("node record past end");
    const uint64_t end = rd.pos() + len;
    const uint8_t kind = rd.u8();
    if (kind == 0) {
      rd.load<uint64_t>();
    } else if (kind == 1) {
      const uint64_t id = rd.load<uint64_t>();
      rd.load<uint64_t>();  // seq
      rd.load<uint64_t>();  // stream
      if (rd.u8() >= 12) corrupt_dag("bad api kind");
      const uint32_t name = rd.load<uint32_t>();
      if (name > rd.remaining()) rd.fail("string length past end");
      rd.take(name);
      rd.load<uint64_t>();  // duration
      rd.load<uint64_t>();  // bytes
      const uint32_t na = rd.load<uint32_t>();
      if ((uint64_t)na * 12 > rd.remaining()) corrupt_dag("arg vector past end");
      rd.take((uint64_t)na * 12);
      for (int v = 0; v < 4; ++v) vec();  // spec reads/writes, true reads/writes
      if (rd.u8() > 2) corrupt_dag("bad node state");
      ids.insert(id);
    } else {
      corrupt_dag("bad node kind");
    }
    if (rd.pos() != end) corrupt_dag("node record length mismatch");
  }
  const uint32_t ne = rd.load<uint32_t>();
  if ((uint64_t)ne * 17 > rd.remaining()) corrupt_dag("edge table past end");
  for (uint32_t i = 0; i < ne; ++i) {
    rd.take(16);
    if (rd.u8() > 2) corrupt_dag("bad edge kind");
  }
  if (rd.remaining() != 0) corrupt_dag("trailing bytes");
  return ids;
}

// Dedup content of record r (image.hpp:364-376) into out (size bytes).
inline bool posi_dedup_bytes(const PosiImage& img, const PosiRecord& r, uint64_t size, uint8_t* out) {
  const uint64_t want_begin = r.offset, want_end = r.offset + size;
  uint64_t got = 0;
  for (size_t i = 0; i < img.page_index.size(); ++i) {
    const uint64_t idx = img.page_index[i];
    if (idx < r.first_page || idx >= r.first_page + r.page_count) continue;
    const uint64_t page_off = (idx - r.first_page) * img.page_size;
    const uint64_t lo = want_begin > page_off ? want_begin : page_off;
    const uint64_t hi = want_end < page_off + img.page_size ? want_end : page_off + img.page_size;
    if (hi > lo) {
      std::memcpy(out + (lo - want_begin), img.page_bytes[i] + (lo - page_off), hi - lo);
      got += hi - lo;
    }
  }
  return got == size;
}

// read_image (image.hpp:209-361).  Throws PosiCorrupt.
inline PosiImage posi_read(const uint8_t* bytes, uint64_t size, bool verify_dedup) {
  PosiReader rd(bytes, size);
  const uint8_t* magic = rd.take(4);
  if (std::memcmp(magic, "POSI", 4) != 0) rd.fail("bad magic");
  const uint16_t version = rd.load<uint16_t>();
  if (version != 1) rd.fail("unsupported version " + std::to_string(version));
  const uint16_t flags = rd.load<uint16_t>();
  if (flags > 1) rd.fail("unknown flags");
  const uint32_t n_pages = rd.load<uint32_t>();
  const uint32_t n_records = rd.load<uint32_t>();
  PosiImage img;
  img.page_size = rd.load<uint64_t>();
  if (img.page_size == 0 || img.page_size > (1u << 20)) rd.fail("implausible page size");
  const uint64_t host_len = rd.load<uint64_t>();
  const uint64_t gpu_len = rd.load<uint64_t>();
  const uint64_t dag_len = rd.load<uint64_t>();
  const uint64_t meta_len = rd.load<uint64_t>();
  if (rd.load<uint64_t>() != 0) rd.fail("reserved field not zero");
  if (host_len != (uint64_t)n_pages * (8 + img.page_size)) rd.fail("host section length mismatch");
  const uint64_t declared = 64 + host_len + gpu_len + dag_len + meta_len;  // wraps like the reference's
  if (declared != size) rd.fail("declared sections do not cover file");

  uint64_t last_index = 0;
  for (uint32_t i = 0; i < n_pages; ++i) {
    const uint64_t index = rd.load<uint64_t>();
    if (i > 0 && index <= last_index) rd.fail("host pages not strictly ascending");
    last_index = index;
    img.page_index.push_back(index);
    img.page_bytes.push_back(rd.take(img.page_size));
  }
  const uint64_t gpu_end = rd.pos() + gpu_len;
  uint64_t last_handle = 0;
  for (uint32_t i = 0; i < n_records; ++i) {
    if (rd.pos() >= gpu_end) rd.fail("gpu record past section");
    PosiRecord r;
    r.handle = rd.load<uint64_t>();
    if (i > 0 && r.handle <= last_handle) rd.fail("gpu records not strictly ascending");
    last_handle = r.handle;
    r.kind = rd.u8();
    if (r.kind > 2) rd.fail("bad gpu record kind");
    if (r.kind == 0) {
      const uint64_t len = rd.load<uint64_t>();
      if (len > rd.remaining()) rd.fail("inline length past end");
      r.inline_bytes = rd.take(len);
      r.inline_len = len;
    } else if (r.kind == 1) {
      r.first_page = rd.load<uint64_t>();
      r.page_count = rd.load<uint32_t>();
      r.offset = rd.load<uint32_t>();
      r.crc = rd.load<uint32_t>();
    } else {
      const uint32_t n = rd.load<uint32_t>();
      if ((uint64_t)n * 8 > rd.remaining()) rd.fail("recompute list past end");
      for (uint32_t k = 0; k < n; ++k) r.nodes.push_back(rd.load<uint64_t>());
    }
    img.recs.push_back(std::move(r));
  }
  if (rd.pos() != gpu_end) rd.fail("gpu section length mismatch");
  if (dag_len > rd.remaining()) rd.fail("dag section past end");
  img.dag = rd.take(dag_len);
  img.dag_len = dag_len;
  if ((flags & 1) != (dag_len == 0 ? 0 : 1)) rd.fail("dag flag/section disagree");
  if (meta_len > 0) {
    const uint64_t meta_end = rd.pos() + meta_len;
    const uint32_t ns = rd.load<uint32_t>();
    if ((uint64_t)ns * 8 > rd.remaining()) rd.fail("vector length past end");
    for (uint32_t k = 0; k < ns; ++k) img.streams.push_back(rd.load<uint64_t>());
    const uint32_t na = rd.load<uint32_t>();
    if ((uint64_t)na * 24 > rd.remaining()) rd.fail("alloc table past end");
    for (uint32_t k = 0; k < na; ++k) {
      PosiImage::Alloc a;
      a.handle = rd.load<uint64_t>();
      a.base = rd.load<uint64_t>();
      a.size = rd.load<uint64_t>();
      img.allocs.push_back(a);
    }
    img.cursor = rd.load<uint64_t>();
    img.next_handle = rd.load<uint64_t>();
    img.next_base = rd.load<uint64_t>();
    if (rd.pos() != meta_end) rd.fail("meta section length mismatch");
  }
  if (rd.remaining() != 0) rd.fail("trailing bytes");

  // Cross-section invariants (all reported at the end of the file).
  std::set<uint64_t> page_set(img.page_index.begin(), img.page_index.end());
  std::map<uint64_t, const PosiImage::Alloc*> allocs;
  for (const auto& a : img.allocs) {
    if (a.size == 0) rd.fail("zero-size allocation");
    if (!allocs.emplace(a.handle, &a).second) rd.fail("duplicate allocation entry");
  }
  std::set<uint64_t> dag_nodes;
  if (img.dag_len) {
    dag_nodes = posi_check_dag(img.dag, img.dag_len);
    if (dag_nodes.empty()) rd.fail("dag flag set but dag has no kernels");
  }
  std::vector<uint8_t> scratch;
  for (const auto& r : img.recs) {
    auto it = allocs.find(r.handle);
    if (it == allocs.end()) rd.fail("gpu record without allocation entry");
    const PosiImage::Alloc& a = *it->second;
    if (r.kind == 0) {
      if (r.inline_len != a.size) rd.fail("inline length != buffer size");
    } else if (r.kind == 1) {
      if (r.page_count == 0) rd.fail("empty dedup page range");
      for (uint64_t p = r.first_page; p < r.first_page + r.page_count; ++p)
        if (!page_set.count(p)) rd.fail("dedup page missing from host section");
      const uint64_t span = (uint64_t)r.page_count * img.page_size;
      if ((uint64_t)r.offset + a.size > span) rd.fail("dedup range does not cover buffer");
      if (verify_dedup) {
        scratch.assign(a.size, 0);
        if (!posi_dedup_bytes(img, r, a.size, scratch.data()) || posi_crc32(scratch.data(), a.size) != r.crc)
          rd.fail("dedup checksum mismatch");
      }
    } else {
      if (r.nodes.empty()) rd.fail("empty recompute list");
      for (uint64_t id : r.nodes)
        if (!dag_nodes.count(id)) rd.fail("recompute node missing from dag");
    }
  }
  return img;
}

}  // namespace posdump
