// posdump.cu -- host side of libposdump.so: the C ABI of include/posdump.h.
//
// Owns device memory for the buffer table, the per-chunk digest tables
// (double-buffered by epoch), the dirty flags/bitmap, the O3 cache and the
// launch plumbing.  There is no CPU path: every operation on buffer bytes is
// a kernel from kernels.cuh, and a missing device is an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/posdump.h"
#include "crc_math.h"
#include "kernels.cuh"
#include "image_writer.h"

using namespace posdump;

namespace {

thread_local std::string g_last_error;

struct Fail {
  int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
  g_last_error = msg;
  throw Fail{code};
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(POS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return POS_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return POS_E_OUT_OF_DEVICE_MEMORY;
  }
}

template <typename T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t c = std::max<size_t>(count, 1);
    cudaError_t e = cudaMalloc(&p, c * sizeof(T));
    if (e != cudaSuccess)
      fail(POS_E_OUT_OF_DEVICE_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    n = c;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

template <typename T>
struct PinnedArray {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    size_t c = std::max<size_t>(count, 1);
    ck(cudaHostAlloc((void**)&p, c * sizeof(T), cudaHostAllocMapped), "cudaHostAlloc");
    n = c;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

// Hash kernel variants (threads per CTA x warp steps per batch); one CTA per
// SM either way.  POSDUMP_HASH_CFG selects one for tuning runs.
enum HashCfg { kCfg512x8 = 0, kCfg256x16, kCfg384x12, kCfg512r12, kCfg512r16, kCfg256r24 };

HashCfg hash_cfg() {
  static const HashCfg c = [] {
    const char* e = std::getenv("POSDUMP_HASH_CFG");
    if (!e) return kCfg512x8;
    if (!std::strcmp(e, "256x16")) return kCfg256x16;
    if (!std::strcmp(e, "384x12")) return kCfg384x12;
    if (!std::strcmp(e, "512r12")) return kCfg512r12;
    if (!std::strcmp(e, "512r16")) return kCfg512r16;
    if (!std::strcmp(e, "256r24")) return kCfg256r24;
    return kCfg512x8;
  }();
  return c;
}

int hash_threads() {
  switch (hash_cfg()) {
    case kCfg256x16: return 256;
    case kCfg256r24: return 256;
    case kCfg384x12: return 384;
    default: return 512;
  }
}

template <int COPY>
void launch_hash(int grid, cudaStream_t s, const HashParams& p) {
  switch (hash_cfg()) {
    case kCfg256x16: k_hash_chunks<COPY, 256, 16><<<grid, 256, kHashSmem, s>>>(p); break;
    case kCfg384x12: k_hash_chunks<COPY, 384, 12><<<grid, 384, kHashSmem, s>>>(p); break;
    case kCfg512r12: k_hash_chunks<COPY, 512, 12, true><<<grid, 512, kHashSmem, s>>>(p); break;
    case kCfg512r16: k_hash_chunks<COPY, 512, 16, true><<<grid, 512, kHashSmem, s>>>(p); break;
    case kCfg256r24: k_hash_chunks<COPY, 256, 24, true><<<grid, 256, kHashSmem, s>>>(p); break;
    default: k_hash_chunks<COPY, 512, 8><<<grid, 512, kHashSmem, s>>>(p); break;
  }
}

template <int COPY>
void set_hash_smem() {
  ck(cudaFuncSetAttribute(k_hash_chunks<COPY, 512, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem), "smem attr");
  ck(cudaFuncSetAttribute(k_hash_chunks<COPY, 256, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem), "smem attr");
  ck(cudaFuncSetAttribute(k_hash_chunks<COPY, 384, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem), "smem attr");
  ck(cudaFuncSetAttribute(k_hash_chunks<COPY, 512, 12, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem), "smem attr");
  ck(cudaFuncSetAttribute(k_hash_chunks<COPY, 512, 16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem), "smem attr");
  ck(cudaFuncSetAttribute(k_hash_chunks<COPY, 256, 24, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem), "smem attr");
}

// Tables shared by every launch on a device: Z^512 (replicated in smem by the
// kernel), Z^4, Z^16..Z^256, and x^(-8n) for n < 512.
struct CrcTables {
  DevArray<uint32_t> tables;  // 7 x 1024
  DevArray<uint32_t> xinv;    // 512
  int sm_count = 0;
  void init(int device) {
    std::vector<uint32_t> h(7 * 1024);
    build_advance_table(512, h.data());
    build_advance_table(4, h.data() + 1024);
    for (int k = 0; k < 5; ++k) build_advance_table(16u << k, h.data() + 1024 * (2 + k));
    std::vector<uint32_t> xi(512);
    for (int n = 0; n < 512; ++n) xi[n] = xinv8nmodp(n);
    tables.ensure(h.size());
    xinv.ensure(xi.size());
    ck(cudaMemcpy(tables.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "upload tables");
    ck(cudaMemcpy(xinv.p, xi.data(), xi.size() * 4, cudaMemcpyHostToDevice), "upload xinv");
    ck(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device), "sm count");
    set_hash_smem<kModeHash>();
    set_hash_smem<kModeCopy>();
    set_hash_smem<kModeCached>();
    ck(cudaFuncSetAttribute(k_copy_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, kCopySmem),
       "smem attr");
    // Load every kernel now: under lazy module loading (the CUDA 12 default)
    // a kernel's first launch loads it, and that load waits for the device --
    // behind a persistent k_drain_queue that waits for this very kernel
    // (measured: the first direct pre-copy of a process stalled until the
    // drain's watchdog fired).
    // The drain CTAs run beside the hash kernel's 193 KiB CTAs: an SM's
    // L1/shared split can only change while it is idle, so the drains (and
    // the scan) ask for the hash kernel's maximal-shared carveout -- otherwise
    // every SM holding a drain CTA is closed to the hash (measured: the hash
    // ran in two rounds, 2-4x slower, while the ship-queue drain was live).
    for (const void* f : {(const void*)k_drain_queue, (const void*)k_copy_host, (const void*)k_pack_scan})
      ck(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared),
         "carveout");
    cudaFuncAttributes fa;
    ck(cudaFuncGetAttributes(&fa, k_pack_scan), "load k_pack_scan");
    ck(cudaFuncGetAttributes(&fa, k_scan_tiles), "load k_scan_tiles");
    ck(cudaFuncGetAttributes(&fa, k_drain_queue), "load k_drain_queue");
    ck(cudaFuncGetAttributes(&fa, k_copy_host), "load k_copy_host");
    ck(cudaFuncGetAttributes(&fa, k_copy_simt), "load k_copy_simt");
    ck(cudaFuncGetAttributes(&fa, k_copy_vec), "load k_copy_vec");
    ck(cudaFuncGetAttributes(&fa, k_pack_items), "load k_pack_items");
    ck(cudaFuncGetAttributes(&fa, k_buffer_crc), "load k_buffer_crc");
    ck(cudaFuncGetAttributes(&fa, k_note_upstream), "load k_note_upstream");
    ck(cudaFuncGetAttributes(&fa, k_fill), "load k_fill");
    ck(cudaFuncGetAttributes(&fa, k_stage_in), "load k_stage_in");
    ck(cudaFuncGetAttributes(&fa, k_stamp), "load k_stamp");
  }
};

void require_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    fail(POS_E_NO_DEVICE, "no CUDA device: the dump path has no CPU fallback");
  if (device < 0 || device >= n) fail(POS_E_INVALID_ARGUMENT, "bad device ordinal");
  ck(cudaSetDevice(device), "cudaSetDevice");
}

enum TimerId {
  kTimHash = 0, kTimCombine, kTimScan, kTimCopy, kTimDelta, kTimScatter, kTimD2H, kTimDeltaHash, kTimCount
};
const char* kTimerNames[kTimCount] = {"hash", "combine", "scan", "copy", "delta", "scatter", "d2h", "delta_hash"};

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  bool used = false;
};

}  // namespace

// On-demand restore of a flat host image (start_loads / enqueue_load /
// gate_restore / bump_front, cr.hpp:1043-1143, engines.hpp:63-93): a loader
// thread feeds the copy engine H2D slices from a priority queue of buffers,
// keeping only kLoadWindow slices in flight so a wanted buffer jumps ahead
// within ~kLoadWindow * slice of link time; each buffer's last slice records
// its ready event, which gates kernels on the device (cudaStreamWaitEvent).
struct Loader {
  static constexpr int kLoadWindow = 4;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<uint32_t> queue;         // buffer indices with bytes left to issue; front = next
  std::vector<uint64_t> issued;       // bytes issued per buffer
  std::vector<uint8_t> state;         // 0 queued, 1 ready event recorded, 2 not part of the image
  std::vector<cudaEvent_t> ready;     // per buffer
  std::vector<const uint8_t*> src;    // host image per buffer
  cudaEvent_t ring[kLoadWindow] = {};
  std::vector<void*> pinned_here;     // ranges the loader pinned (unpinned at the end)
  cudaStream_t stream = nullptr;
  uint64_t slice = 8ull << 20;
  int device = 0;
  bool running = false, failed = false;
  std::string error;
};

// NVLink peer-GPU cache (BASELINE config 5): packs of the
// cache-cycled pre-copy move to slots in a peer GPU's free HBM
// (cudaMemcpyPeerAsync), which frees the local cache region at NVLink speed
// (the snapshot is captured once every wave sits in the peer); the peer's
// own copy engine then drains the slots over ITS PCIe link.
struct PeerCache {
  int device = -1;
  uint8_t* base = nullptr;
  uint64_t bytes = 0;
  cudaStream_t stream = nullptr;             // on the peer device: the drain
  std::vector<cudaEvent_t> in, free_;        // per slot: pack landed (local dev) / slot drained (peer dev)
  cudaEvent_t land[2] = {}, t0 = nullptr, captured = nullptr, drained = nullptr;
  float capture_ms = 0, total_ms = 0;
};

struct pos_ctx {
  pos_config cfg{};
  Loader* loader = nullptr;
  PeerCache* peer = nullptr;
  CrcTables crc;
  // Buffer set (ascending handle).
  std::vector<pos_buffer_desc> bufs;
  std::vector<uint64_t> chunk_base;  // per buffer
  std::vector<DevBuf> hbufs;
  std::map<uint64_t, uint32_t> index_of;
  std::map<uint64_t, uint32_t> by_ptr;  // device base -> buffer index (find_containing)
  // note_h2d_provenance on the device (pos_h2d_provenance)
  DevArray<uint32_t> d_prov;            // chunk digests of the H2D'd buffer
  PinnedArray<uint32_t> h_up;           // mapped mirror of Upstream::crc per buffer
  cudaEvent_t ev_prov = nullptr;
  bool prov_pending = false;
  std::vector<uint32_t> prov_bufs;      // buffers whose crc is still on its way
  uint64_t n_chunks = 0;
  DevArray<DevBuf> d_bufs;
  DevArray<uint2> d_chunk_map;
  DevArray<uint32_t> d_digest[2];
  int cur = 0;
  bool prev_valid = false;
  uint64_t epoch = 0;
  DevArray<uint8_t> d_flags;
  DevArray<uint32_t> d_bitmap;
  DevArray<uint32_t> d_buf_crc;
  DevArray<uint8_t> d_verdict;
  DevArray<uint8_t> d_dag_dirty;
  DevArray<uint32_t> d_tcs;  // Z^chunk_size
  DevArray<uint32_t> d_xfold;  // per buffer: x^(8 cs ceil((nchunks-1)/32)) (warp_fold_buffer)
  // chunk segmentation (parallelism for short chunk lists)
  // level L = log2(nseg): x^(8 k cs/2^L) (32 per level) and, per buffer,
  // x^(8 * last segment length of the tail chunk); valid_levels bitmask.
  uint32_t seg_levels = 1;
  DevArray<uint32_t> d_xseg, d_lastseg;
  DevArray<uint64_t> d_result;  // async pre-copy: [n, total, overflow, n_items]
  std::set<uint64_t> dirty_set;
  bool dag_uploaded = false;
  uint64_t dirty_version = 0;
  // STW delta staged ahead of the stop (pos_delta_prepare)
  bool delta_ready = false;
  uint64_t delta_version = 0, delta_precopy = 0, delta_n = 0, delta_offset = 0, delta_total = 0,
           delta_payload_off = 0;
  bool delta_aligned = true;
  bool delta_drain = false;  // drain items staged with the delta
  DevArray<CopyItem> d_delta_items;
  // host image (pos_register_image): device-visible address per buffer, and
  // the host ranges this context pinned itself (unpinned at destroy)
  bool image_ready = false;
  std::vector<void*> image_pinned;
  DevArray<CopyItem> d_drain_items;  // STW delta pack payload -> host image
  uint64_t drain_n = 0;              // items of the last delta copy (pos_delta_drain)
  bool drain_pending = false;
  bool direct_pending = false;       // a pos_precopy_direct awaits pos_precopy_direct_result
  // ship queue (hash -> k_drain_queue) of the direct pre-copy
  DevArray<ShipQueue> d_q;
  DevArray<unsigned long long> d_qslots;
  unsigned long long q_seq = 0;
  cudaEvent_t ev_drained = nullptr;  // the last k_drain_queue exited (queue reset)
  // copy-engine drain (default direct mode): run lists written by the scan
  // into mapped pinned memory = the arguments of cudaMemcpyBatchAsync
  PinnedArray<uint64_t> h_run;   // [3][n_chunks]: src, dst, bytes
  PinnedArray<uint64_t> h_drun;  // STW delta drain runs, same layout
  DevArray<TileStatus> d_tiles;  // tiled scan: decoupled look-back status
  DevArray<TileCtl> d_tile_ctl;  // [kMaxWaves]: ticket + finished counters
  uint64_t drun_n = 0, drun_cap = 0;
  uint32_t direct_lo[16] = {};  // first chunk of each direct wave (kMaxWaves)
  uint32_t direct_waves = 0;
  // O3 cache
  DevArray<uint8_t> cache;
  uint64_t cache_cap = 0;
  // CoW staging (pos_stage_buffers): packs grow down from the top of the cache
  uint64_t staging_used = 0;
  std::vector<uint32_t> staged;  // buffer indices staged this epoch
  uint64_t precopy_bytes = 0;
  DevArray<CopyItem> d_items;
  DevArray<uint64_t> d_scan;     // [n, total, overflow]
  DevArray<uint4> d_work;
  DevArray<uint4> d_stage_work;  // CoW staging work list
  DevArray<uint32_t> d_err;
  PinnedArray<uint64_t> h_scan;
  PinnedArray<uint8_t> h_stage;  // delta header + work list upload
  PinnedArray<uint8_t> h_dag;
  cudaEvent_t stage_free = nullptr;
  cudaEvent_t ev_dag = nullptr;  // DAG flags uploaded on a side stream
  bool dag_side = false;
  // Pre-copy packs: one per wave, chained at a device-side cache cursor.
  static constexpr uint32_t kMaxWaves = 16;
  DevArray<uint64_t> d_cursor;                     // [1]
  cudaEvent_t scanned[kMaxWaves] = {};
  cudaEvent_t copied[kMaxWaves] = {};
  cudaEvent_t wave_hash[kMaxWaves][2] = {};
  uint32_t waves_last = 0;                          // waves of the last pre-copy (hash timing)
  uint64_t scan_seq = 0, slot_seq[kMaxWaves] = {};  // host-mirror sequence numbers
  // cache-cycled pre-copy (pos_precopy_stream): 2 cache regions, 2 pinned landing slots
  PinnedArray<uint8_t> h_land[2];
  cudaEvent_t ev_d2h[2] = {}, ev_copied2[2] = {};
  bool pack_pending = false;
  // timing
  std::vector<cudaEvent_t> events;
  DevArray<unsigned long long> d_stamps;  // [64] globaltimer stamps (pos_stamp)
  Timer timers[kTimCount];
  uint64_t launches = 0;

  void timer_begin(TimerId t, cudaStream_t s) { ck(cudaEventRecord(timers[t].a, s), "event"); }
  void timer_end(TimerId t, cudaStream_t s) {
    ck(cudaEventRecord(timers[t].b, s), "event");
    timers[t].used = true;
  }
  // One CTA per SM (152 KiB of smem tables); items are dealt round-robin over
  // CTAs first, so even a short list occupies every SM.
  int hash_grid(uint64_t items) const {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(items, (uint64_t)crc.sm_count));
  }
};

namespace {

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(POS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// cudaMemcpyBatchAsync flags of the host leg (POSDUMP_CE_OVERLAP=1: prefer
// overlap with compute).
unsigned int ce_flags() {
  static const unsigned int f = [] {
    const char* e = std::getenv("POSDUMP_CE_OVERLAP");
    return (e && e[0] == '1') ? (unsigned int)cudaMemcpyFlagPreferOverlapWithCompute : 0u;
  }();
  return f;
}

// Host leg of the direct pre-copy: 0 copy-engine runs, 1 SM ship queue, 2 SM after each scan.
int direct_drain_mode() {
  static const int m = [] {
    const char* e = std::getenv("POSDUMP_DIRECT_DRAIN");
    if (e && !std::strcmp(e, "queue")) return 1;
    if (e && !std::strcmp(e, "sm")) return 2;
    return 0;
  }();
  return m;
}


// Per-buffer DAG-dirty flags (dirty_set_) to the device.  With a side
// stream the copy runs there (concurrently with the first hash) and `s`
// waits for it only where a consumer is enqueued (upload_dag_flags(c, s)).
void upload_dag_flags(pos_ctx* c, cudaStream_t s, cudaStream_t side = nullptr) {
  if (c->dag_uploaded) {
    if (c->dag_side && !side) ck(cudaStreamWaitEvent(s, c->ev_dag, 0), "wait dag");
    return;
  }
  uint32_t nb = (uint32_t)c->bufs.size();
  c->h_dag.ensure(nb);
  if (c->stage_free) ck(cudaEventSynchronize(c->stage_free), "stage sync");
  for (uint32_t i = 0; i < nb; ++i) c->h_dag.p[i] = c->dirty_set.count(c->bufs[i].handle) ? 1 : 0;
  cudaStream_t us = side ? side : s;
  ck(cudaMemcpyAsync(c->d_dag_dirty.p, c->h_dag.p, nb, cudaMemcpyHostToDevice, us), "dag upload");
  ck(cudaEventRecord(c->stage_free, us), "event");
  c->dag_side = side != nullptr;
  if (side) ck(cudaEventRecord(c->ev_dag, side), "event");
  c->dag_uploaded = true;
}

void launch_copy(pos_ctx* c, const CopyItem* items, const uint64_t* n_dev, uint64_t n_host,
                 bool aligned, cudaStream_t s, bool prefer_vec = false) {
  int sms = c->crc.sm_count;
  static const bool force_simt = [] {
    const char* e = std::getenv("POSDUMP_COPY");
    return e && !std::strcmp(e, "simt");
  }();
  if (force_simt) aligned = false;
  static const bool force_vec = [] {
    const char* e = std::getenv("POSDUMP_COPY");
    return e && !std::strcmp(e, "vec");
  }();
  if (aligned && (force_vec || prefer_vec)) {
    const uint32_t ppi = (uint32_t)std::max<uint64_t>(1, (c->cfg.chunk_size + 15 + kVecPiece - 1) / kVecPiece);
    k_copy_vec<<<sms * 8, 256, 0, s>>>(items, n_dev, n_host, ppi);
  } else if (aligned) {
    // 3 CTAs/SM fit in smem (64 KiB ring each); one elected thread per CTA.
    int grid = sms * 3;
    if (!n_dev) grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(grid, n_host));
    k_copy_bulk<<<grid, 32, kCopySmem, s>>>(items, n_dev, n_host);
  } else {
    k_copy_simt<<<sms * 4, 256, 0, s>>>(items, n_dev, n_host);
  }
  check_launch("copy");
  ++c->launches;
}

void launch_copy_host(pos_ctx* c, const CopyItem* items, const uint64_t* n_dev, uint64_t n_host,
                      cudaStream_t s) {
  static const int ctas = [] {
    const char* e = std::getenv("POSDUMP_HOST_CTAS");  // tuning override
    int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : kHostCopyCtas;
  }();
  int grid = ctas;
  if (!n_dev) grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(grid, (n_host + 3) / 4));
  k_copy_host<<<grid, kHostCopyThreads, 0, s>>>(items, n_dev, n_host);
  check_launch("k_copy_host");
  ++c->launches;
}

// Global per-device CRC engine for pos_crc32 (no context).
std::mutex g_engine_mu;
std::map<int, CrcTables*> g_engines;

CrcTables& engine_for_current_device() {
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_engine_mu);
  auto it = g_engines.find(dev);
  if (it != g_engines.end()) return *it->second;
  auto* e = new CrcTables();
  e->init(dev);
  g_engines[dev] = e;
  return *e;
}

}  // namespace

extern "C" {

const char* pos_strerror(int code) {
  static const char* names[] = {"OK",           "PastTime",          "Livelock",
                                "OutOfDeviceMemory", "InvalidLocator", "UseAfterFree",
                                "FreedBuffer",  "BadState",          "PendingKernels",
                                "UnknownApi",   "InvalidArgument",   "CorruptDag",
                                "CorruptImage", "InvariantViolation", "StagingExhausted",
                                "OracleMismatch"};
  if (code >= 0 && code <= 15) return names[code];
  if (code == POS_E_CUDA) return "CudaError";
  if (code == POS_E_NO_DEVICE) return "NoDevice";
  return "Unknown";
}

const char* pos_last_error(void) { return g_last_error.c_str(); }
int pos_abi_version(void) { return POSDUMP_ABI_VERSION; }

int pos_ctx_create(const pos_config* cfg, pos_ctx** out) {
  return guarded([&] {
    if (!cfg || !out) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (cfg->chunk_size == 0 || cfg->page_size == 0)
      fail(POS_E_INVALID_ARGUMENT, "chunk_size and page_size must be positive");
    if (cfg->chunk_size > (1ull << 31)) fail(POS_E_INVALID_ARGUMENT, "chunk_size too large");
    require_device(cfg->device);
    auto* c = new pos_ctx();
    try {
      c->cfg = *cfg;
      c->crc.init(cfg->device);
      std::vector<uint32_t> tcs(1024);
      build_advance_table(cfg->chunk_size, tcs.data());
      c->d_tcs.ensure(1024);
      ck(cudaMemcpy(c->d_tcs.p, tcs.data(), 4096, cudaMemcpyHostToDevice), "upload tcs");
      uint64_t cap = cfg->cache_capacity;
      if (cap == 0) {
        size_t free_b = 0, total_b = 0;
        ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        double frac = cfg->staging_fraction > 0 ? cfg->staging_fraction : 1.0 / 16.0;
        cap = (uint64_t)((double)total_b * frac);  // staging_capacity() (config.hpp:43-45)
      }
      c->cache_cap = round_up(cap, 256);
      c->cache.ensure(c->cache_cap);
      c->d_scan.ensure(8 * pos_ctx::kMaxWaves);
      c->d_err.ensure(1);
      c->h_scan.ensure(8 * pos_ctx::kMaxWaves);
      ck(cudaEventCreateWithFlags(&c->stage_free, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&c->ev_dag, cudaEventDisableTiming), "event");
      for (uint32_t w = 0; w < pos_ctx::kMaxWaves; ++w) {
        ck(cudaEventCreateWithFlags(&c->scanned[w], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->copied[w], cudaEventDisableTiming), "event");
        ck(cudaEventCreate(&c->wave_hash[w][0]), "event");
        ck(cudaEventCreate(&c->wave_hash[w][1]), "event");
      }
      c->d_cursor.ensure(1);
      for (auto& t : c->timers) {
        ck(cudaEventCreate(&t.a), "event");
        ck(cudaEventCreate(&t.b), "event");
      }
      c->events.resize(64);
      for (auto& e : c->events) ck(cudaEventCreate(&e), "event");
    } catch (...) {
      pos_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

static void loader_finish(pos_ctx* c);

static void peer_release(pos_ctx* c);

int pos_ctx_destroy(pos_ctx* c) {
  if (!c) return POS_OK;
  loader_finish(c);
  peer_release(c);
  cudaDeviceSynchronize();
  c->crc.tables.release();
  c->crc.xinv.release();
  c->d_bufs.release();
  c->d_chunk_map.release();
  c->d_digest[0].release();
  c->d_digest[1].release();
  c->d_flags.release();
  c->d_bitmap.release();
  c->d_buf_crc.release();
  c->d_verdict.release();
  c->d_dag_dirty.release();
  c->d_tcs.release();
  c->d_xfold.release();
  c->d_prov.release();
  c->h_up.release();
  if (c->ev_prov) cudaEventDestroy(c->ev_prov);
  c->d_xseg.release();
  c->d_lastseg.release();
  c->d_result.release();
  c->cache.release();
  c->d_items.release();
  c->d_delta_items.release();
  c->d_drain_items.release();
  c->d_q.release();
  c->d_stamps.release();
  c->h_run.release();
  c->d_tiles.release();
  c->d_tile_ctl.release();
  c->h_drun.release();
  c->d_qslots.release();
  if (c->ev_drained) cudaEventDestroy(c->ev_drained);
  for (void* h : c->image_pinned) cudaHostUnregister(h);
  c->d_scan.release();
  c->d_work.release();
  c->d_stage_work.release();
  c->d_err.release();
  c->h_scan.release();
  c->h_stage.release();
  c->h_dag.release();
  if (c->stage_free) cudaEventDestroy(c->stage_free);
  if (c->ev_dag) cudaEventDestroy(c->ev_dag);
  for (uint32_t w = 0; w < pos_ctx::kMaxWaves; ++w) {
    if (c->scanned[w]) cudaEventDestroy(c->scanned[w]);
    if (c->copied[w]) cudaEventDestroy(c->copied[w]);
    if (c->wave_hash[w][0]) cudaEventDestroy(c->wave_hash[w][0]);
    if (c->wave_hash[w][1]) cudaEventDestroy(c->wave_hash[w][1]);
  }
  c->d_cursor.release();
  c->h_land[0].release();
  c->h_land[1].release();
  for (int i = 0; i < 2; ++i) {
    if (c->ev_d2h[i]) cudaEventDestroy(c->ev_d2h[i]);
    if (c->ev_copied2[i]) cudaEventDestroy(c->ev_copied2[i]);
  }
  for (auto& t : c->timers) {
    if (t.a) cudaEventDestroy(t.a);
    if (t.b) cudaEventDestroy(t.b);
  }
  for (auto e : c->events)
    if (e) cudaEventDestroy(e);
  delete c;
  return POS_OK;
}

int pos_register_buffers(pos_ctx* c, const pos_buffer_desc* bufs, uint32_t n) {
  return guarded([&] {
    if (!c || (!bufs && n)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    std::vector<pos_buffer_desc> v(bufs, bufs + n);
    for (uint32_t i = 0; i < n; ++i) {
      if (v[i].size == 0) fail(POS_E_INVALID_ARGUMENT, "buffer of size 0");
      if (i && v[i].handle <= v[i - 1].handle)
        fail(POS_E_INVALID_ARGUMENT, "buffers must be registered by strictly ascending handle");
    }
    const uint64_t cs = c->cfg.chunk_size;
    c->bufs = v;
    c->hbufs.assign(n, DevBuf{});
    c->chunk_base.assign(n, 0);
    c->index_of.clear();
    c->by_ptr.clear();
    c->prov_pending = false;
    c->prov_bufs.clear();
    uint64_t g = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const auto& d = v[i];
      DevBuf& b = c->hbufs[i];
      b.ptr = d.dev_ptr;
      b.size = d.size;
      b.handle = d.handle;
      b.chunk_base = g;
      uint64_t nc = (d.size + cs - 1) / cs;
      if (nc > 0xFFFFFFFFull) fail(POS_E_INVALID_ARGUMENT, "too many chunks in one buffer");
      b.nchunks = (uint32_t)nc;
      uint64_t tail = d.size - (nc - 1) * cs;
      b.k_tail = zeros_crc(tail);
      b.x8_tail = x8nmodp(tail);
      b.flags = (d.has_upstream ? kBufHasUpstream : 0) | (d.host_untouched ? kBufHostUntouched : 0) |
                (d.written_since_ckpt ? kBufWrittenSinceCkpt : 0);
      b.upstream_crc = d.upstream_crc;
      c->chunk_base[i] = g;
      c->index_of[d.handle] = i;
      c->by_ptr[d.dev_ptr] = i;
      g += nc;
    }
    if (g > 0xFFFFFFFFull) fail(POS_E_INVALID_ARGUMENT, "more than 2^32 chunks");
    c->n_chunks = g;
    // Segment tables for nseg = 2^L (L < 6, segment >= 8 KiB, cs % (nseg*512) == 0):
    // used when a launch has too few chunks to occupy every warp.
    {
      std::vector<uint32_t> xs(6 * 32), ls(6 * (size_t)std::max<uint32_t>(n, 1));
      c->seg_levels = 0;
      for (int L = 0; L < 6; ++L) {
        uint64_t nseg = 1ull << L;
        if (cs % (nseg * kStepBytes) != 0 || (L > 0 && cs / nseg < 8192)) break;
        c->seg_levels = L + 1;
        uint64_t sb = cs / nseg;
        for (int k = 0; k < 32; ++k) xs[L * 32 + k] = x8nmodp((uint64_t)k * sb);
        for (uint32_t i = 0; i < n; ++i) {
          const DevBuf& b = c->hbufs[i];
          uint64_t tail = b.size - (uint64_t)(b.nchunks - 1) * cs;
          uint64_t m = (tail - 1) / sb;
          ls[L * (size_t)n + i] = x8nmodp(tail - m * sb);
        }
      }
      if (c->seg_levels == 0) c->seg_levels = 1;  // nseg = 1 always valid
      c->d_xseg.ensure(xs.size());
      c->d_lastseg.ensure(ls.size());
      ck(cudaMemcpy(c->d_xseg.p, xs.data(), xs.size() * 4, cudaMemcpyHostToDevice), "xseg");
      ck(cudaMemcpy(c->d_lastseg.p, ls.data(), ls.size() * 4, cudaMemcpyHostToDevice), "lastseg");
    }
    {
      std::vector<uint32_t> xf(std::max<uint32_t>(n, 1), 0);
      for (uint32_t i = 0; i < n; ++i) xf[i] = x8nmodp(cs * (uint64_t)((c->hbufs[i].nchunks - 1 + 31) / 32));
      c->d_xfold.ensure(xf.size());
      ck(cudaMemcpy(c->d_xfold.p, xf.data(), xf.size() * 4, cudaMemcpyHostToDevice), "xfold");
    }
    std::vector<uint2> cmap(g);
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t k = 0; k < c->hbufs[i].nchunks; ++k) cmap[c->chunk_base[i] + k] = make_uint2(i, k);
    c->d_bufs.ensure(n);
    c->d_chunk_map.ensure(g);
    c->d_digest[0].ensure(g);
    c->d_digest[1].ensure(g);
    c->d_flags.ensure(g);
    c->d_bitmap.ensure((g + 31) / 32);
    c->d_buf_crc.ensure(n);
    c->d_verdict.ensure(n);
    c->d_dag_dirty.ensure(n);
    c->d_items.ensure(g);
    c->d_work.ensure(g);
    if (n) ck(cudaMemcpy(c->d_bufs.p, c->hbufs.data(), n * sizeof(DevBuf), cudaMemcpyHostToDevice), "bufs");
    if (g) ck(cudaMemcpy(c->d_chunk_map.p, cmap.data(), g * sizeof(uint2), cudaMemcpyHostToDevice), "cmap");
    ck(cudaMemset(c->d_verdict.p, 0, std::max<uint32_t>(n, 1)), "memset");
    ck(cudaMemset(c->d_dag_dirty.p, 0, std::max<uint32_t>(n, 1)), "memset");
    c->cur = 0;
    c->prev_valid = false;
    c->epoch = 0;
    c->dirty_set.clear();
    c->dag_uploaded = false;
    ++c->dirty_version;
    c->delta_ready = false;
    c->precopy_bytes = 0;
  });
}

static void set_segments(const pos_ctx* c, uint64_t items, HashParams& p);

// Upstream CRCs computed on the device (pos_h2d_provenance) into the host
// copy of the buffer table, before the host uploads any of it again.
static void sync_provenance(pos_ctx* c) {
  if (!c->prov_pending) return;
  ck(cudaEventSynchronize(c->ev_prov), "provenance sync");
  for (uint32_t i : c->prov_bufs)
    if (c->hbufs[i].flags & kBufHasUpstream) {
      c->hbufs[i].upstream_crc = c->h_up.p[i];
      c->bufs[i].upstream_crc = c->h_up.p[i];
    }
  c->prov_bufs.clear();
  c->prov_pending = false;
}

int pos_h2d_provenance(pos_ctx* c, uint64_t dst, const void* src, uint64_t bytes, int do_copy, void* stream) {
  return guarded([&] {
    if (!c || (do_copy && bytes && !src)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(stream);
    if (do_copy && bytes)
      ck(cudaMemcpyAsync((void*)dst, src, bytes, cudaMemcpyHostToDevice, s), "h2d");
    // find_containing(dst) (buffer.hpp:160-170); no buffer -> no provenance
    auto it = c->by_ptr.upper_bound(dst);
    if (it == c->by_ptr.begin()) return;
    --it;
    const uint32_t i = it->second;
    DevBuf& b = c->hbufs[i];
    if (dst >= b.ptr + b.size) return;
    const bool whole = b.ptr == dst && b.size == bytes;
    if (!c->ev_prov) ck(cudaEventCreateWithFlags(&c->ev_prov, cudaEventDisableTiming), "event");
    c->h_up.ensure(c->bufs.size());
    if (whole) {  // chunk digests of the fresh content -> fold on the device
      c->d_prov.ensure(std::max<uint64_t>(c->n_chunks, 1));
      HashParams p{};
      p.bufs = c->d_bufs.p;
      p.chunk_map = c->d_chunk_map.p;
      p.n_items = b.nchunks;
      p.item_base = b.chunk_base;
      p.chunk_size = c->cfg.chunk_size;
      p.k_full = zeros_crc(c->cfg.chunk_size);
      p.tables = c->crc.tables.p;
      p.xinv = c->crc.xinv.p;
      p.digest_cur = c->d_prov.p;  // indexed by global chunk
      set_segments(c, b.nchunks, p);
      launch_hash<kModeHash>(c->hash_grid(b.nchunks * p.nseg), s, p);
      check_launch("k_hash_chunks<provenance>");
      ++c->launches;
    }
    k_note_upstream<<<1, 32, 0, s>>>(c->d_bufs.p, i, c->d_prov.p, c->d_tcs.p, c->d_xfold.p, whole ? 1 : 0,
                                     c->h_up.p);
    check_launch("k_note_upstream");
    ++c->launches;
    ck(cudaEventRecord(c->ev_prov, s), "event");
    b.flags |= kBufWrittenSinceCkpt;
    c->bufs[i].written_since_ckpt = 1;
    if (whole) {
      b.flags |= kBufHasUpstream | kBufHostUntouched;
      c->bufs[i].has_upstream = 1;
      c->bufs[i].host_untouched = 1;
      c->prov_bufs.push_back(i);
      c->prov_pending = true;
    } else {  // process.hpp:510-513
      b.flags &= ~(kBufHasUpstream | kBufHostUntouched);
      c->bufs[i].has_upstream = 0;
      c->bufs[i].host_untouched = 0;
    }
  });
}

int pos_read_upstream(pos_ctx* c, uint64_t handle, uint32_t* has_upstream, uint32_t* crc) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    auto it = c->index_of.find(handle);
    if (it == c->index_of.end()) fail(POS_E_INVALID_LOCATOR, "unknown handle");
    sync_provenance(c);
    const pos_buffer_desc& d = c->bufs[it->second];
    if (has_upstream) *has_upstream = d.has_upstream;
    if (crc) *crc = d.upstream_crc;
  });
}

int pos_update_buffer(pos_ctx* c, const pos_buffer_desc* d) {
  return guarded([&] {
    if (!c || !d) fail(POS_E_INVALID_ARGUMENT, "null argument");
    sync_provenance(c);
    auto it = c->index_of.find(d->handle);
    if (it == c->index_of.end()) fail(POS_E_INVALID_LOCATOR, "unknown handle");
    uint32_t i = it->second;
    if (d->dev_ptr != c->bufs[i].dev_ptr || d->size != c->bufs[i].size)
      fail(POS_E_INVALID_ARGUMENT, "update may not move or resize a buffer");
    c->bufs[i] = *d;
    DevBuf& b = c->hbufs[i];
    b.flags = (d->has_upstream ? kBufHasUpstream : 0) | (d->host_untouched ? kBufHostUntouched : 0) |
              (d->written_since_ckpt ? kBufWrittenSinceCkpt : 0);
    b.upstream_crc = d->upstream_crc;
    ck(cudaMemcpy(c->d_bufs.p + i, &b, sizeof(DevBuf), cudaMemcpyHostToDevice), "update buf");
  });
}

int pos_num_chunks(pos_ctx* c, uint64_t* out) {
  return guarded([&] {
    if (!c || !out) fail(POS_E_INVALID_ARGUMENT, "null argument");
    *out = c->n_chunks;
  });
}


// Segments for a launch over `items` chunks: split chunks only when the list
// cannot give every warp of the grid one chunk (measured: splitting a list
// that already covers half the warps costs more than it balances).
static void set_segments(const pos_ctx* c, uint64_t items, HashParams& p) {
  const uint32_t wpc = (uint32_t)(hash_threads() / 32);  // warps per CTA: nseg must divide it
  const uint64_t warps = (uint64_t)c->crc.sm_count * wpc;
  auto ok = [&](int L) { return L < (int)c->seg_levels && wpc % (1u << L) == 0; };
  int L = 0;
  if (items < warps / 2)
    while (ok(L + 1) && (items << L) < warps) ++L;
  if (const char* e = std::getenv("POSDUMP_NSEG")) {  // tuning override
    int want = 0;
    for (unsigned v = (unsigned)std::strtoul(e, nullptr, 10); v > 1; v >>= 1) ++want;
    if (ok(want)) L = want;
  }
  const uint32_t nb = (uint32_t)std::max<size_t>(c->bufs.size(), 1);
  p.nseg = 1u << L;
  p.seg_bytes = (uint32_t)(c->cfg.chunk_size >> L);
  p.xseg = c->d_xseg.p + 32 * L;
  p.lastseg = c->d_lastseg.p + (size_t)nb * L;
  p.pf_bytes = 0;
  if (const char* e = std::getenv("POSDUMP_PF")) {  // tuning: L2 bulk prefetch
    if (!std::strcmp(e, "slide")) {
      p.pf_bytes = 1;  // a sliding window POSDUMP_PF_STEPS (default 32) 512-B steps ahead of every warp
      const char* d = std::getenv("POSDUMP_PF_STEPS");
      p.pad3 = d ? std::atoi(d) : 32;
    } else {  // the first N bytes of single-round units at unit start
      uint64_t v = std::strtoull(e, nullptr, 10);
      if (v > 1 && (items << L) <= warps) p.pf_bytes = (uint32_t)std::min<uint64_t>(v, p.seg_bytes);
    }
  }
}

int pos_hash_chunks(pos_ctx* c, void* stream) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(stream);
    if (c->n_chunks == 0) return;
    ck(cudaMemsetAsync(c->d_bitmap.p, 0, ((c->n_chunks + 31) / 32) * 4, s), "memset bitmap");
    HashParams p{};
    p.bufs = c->d_bufs.p;
    p.chunk_map = c->d_chunk_map.p;
    p.n_items = c->n_chunks;
    p.chunk_size = c->cfg.chunk_size;
    p.k_full = zeros_crc(c->cfg.chunk_size);
    p.tables = c->crc.tables.p;
    p.xinv = c->crc.xinv.p;
    p.digest_cur = c->d_digest[c->cur].p;
    p.digest_prev = c->d_digest[c->cur ^ 1].p;
    p.flags = c->d_flags.p;
    p.bitmap = c->d_bitmap.p;
    p.prev_valid = c->prev_valid ? 1 : 0;
    set_segments(c, c->n_chunks, p);
    int grid = c->hash_grid(c->n_chunks * p.nseg);
    c->timer_begin(kTimHash, s);
    launch_hash<kModeHash>(grid, s, p);
    check_launch("k_hash_chunks");
    c->timer_end(kTimHash, s);
    ++c->launches;
  });
}

int pos_commit_epoch(pos_ctx* c) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->staged.empty()) {  // the staged snapshots were part of this checkpoint
      ck(cudaDeviceSynchronize(), "sync");
      for (uint32_t i : c->staged) {
        c->hbufs[i].flags &= ~kBufStaged;
        ck(cudaMemcpy(c->d_bufs.p + i, &c->hbufs[i], sizeof(DevBuf), cudaMemcpyHostToDevice), "unstage");
      }
      c->staged.clear();
    }
    c->staging_used = 0;
    c->cur ^= 1;
    c->prev_valid = true;
    ++c->epoch;
    c->dirty_set.clear();
    c->dag_uploaded = false;
    ++c->dirty_version;
    c->delta_ready = false;
    c->precopy_bytes = 0;
  });
}

static int read_back(pos_ctx* c, void* host, const void* dev, uint64_t bytes, void* stream) {
  return guarded([&] {
    if (!c || (!host && bytes)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!bytes) return;
    ck(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, S(stream)), "read back");
    ck(cudaStreamSynchronize(S(stream)), "sync");
  });
}

int pos_read_digests(pos_ctx* c, uint32_t* host, uint64_t n, void* stream) {
  if (c && n > c->n_chunks) return POS_E_INVALID_ARGUMENT;
  return read_back(c, host, c ? c->d_digest[c->cur].p : nullptr, n * 4, stream);
}
int pos_read_flags(pos_ctx* c, uint8_t* host, uint64_t n, void* stream) {
  if (c && n > c->n_chunks) return POS_E_INVALID_ARGUMENT;
  return read_back(c, host, c ? c->d_flags.p : nullptr, n, stream);
}
int pos_read_bitmap(pos_ctx* c, uint32_t* host, uint64_t nwords, void* stream) {
  if (c && nwords > (c->n_chunks + 31) / 32) return POS_E_INVALID_ARGUMENT;
  return read_back(c, host, c ? c->d_bitmap.p : nullptr, nwords * 4, stream);
}

int pos_buffer_crc(pos_ctx* c, void* stream) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(stream);
    uint32_t nb = (uint32_t)c->bufs.size();
    if (!nb) return;
    upload_dag_flags(c, s);
    c->timer_begin(kTimCombine, s);
    k_buffer_crc<<<(nb + 7) / 8, 256, 0, s>>>(c->d_bufs.p, nb, c->d_digest[c->cur].p, c->d_tcs.p,
                                             c->d_xfold.p, c->d_dag_dirty.p, c->cfg.dedup, 1, c->d_buf_crc.p,
                                             c->d_verdict.p);
    check_launch("k_buffer_crc");
    c->timer_end(kTimCombine, s);
    ++c->launches;
  });
}

int pos_read_buffer_crcs(pos_ctx* c, uint32_t* crcs, uint8_t* verdicts, uint32_t n, void* stream) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (n > c->bufs.size()) fail(POS_E_INVALID_ARGUMENT, "n exceeds buffer count");
    if (!n) return;
    if (crcs) ck(cudaMemcpyAsync(crcs, c->d_buf_crc.p, n * 4, cudaMemcpyDeviceToHost, S(stream)), "rb");
    if (verdicts)
      ck(cudaMemcpyAsync(verdicts, c->d_verdict.p, n, cudaMemcpyDeviceToHost, S(stream)), "rb");
    ck(cudaStreamSynchronize(S(stream)), "sync");
  });
}

int pos_record_dirty(pos_ctx* c, const uint64_t* handles, uint32_t n) {
  return guarded([&] {
    if (!c || (!handles && n)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    for (uint32_t i = 0; i < n; ++i) {
      if (!c->index_of.count(handles[i])) continue;  // not in the snapshot (cr.hpp:904)
      if (c->dirty_set.insert(handles[i]).second) {
        c->dag_uploaded = false;
        ++c->dirty_version;
      }
    }
  });
}

int pos_clear_dirty(pos_ctx* c) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    c->dirty_set.clear();
    c->dag_uploaded = false;
    ++c->dirty_version;
  });
}

// Scan + compaction of chunks [lo, hi) into a pack at the device-side cache
// cursor, fully asynchronous: the copy kernel reads its item count from the
// scan's device-side result, which is mirrored into pinned memory behind
// event scanned[slot] for pack_result().
static void launch_pack(pos_ctx* c, int exclude_dag_dirty, cudaStream_t s, uint64_t lo, uint64_t hi,
                        uint32_t slot, uint32_t vb0 = 0, uint32_t vb1 = 0, uint64_t fixed_base = ~0ull,
                        cudaStream_t direct_stream = nullptr, bool direct = false, bool chain_start = false,
                        ShipQueue* q = nullptr, unsigned long long q_seq = 0, bool last_wave = false,
                        bool ce_runs = false) {
  upload_dag_flags(c, s);
  // Packs chain at the device-side cursor; the first of a chain starts at 0
  // (no memset), a fixed-region pack (cache cycling) leaves the cursor alone.
  uint64_t* cursor = c->d_cursor.p;
  if (chain_start) fixed_base = 0;
  else if (fixed_base != ~0ull) cursor = nullptr;
  uint64_t* res = c->d_scan.p + 8 * slot;
  c->timer_begin(kTimScan, s);
  k_pack_scan<<<1, kScanThreads, 0, s>>>(
      c->d_bufs.p, c->d_chunk_map.p, lo, hi, c->cfg.chunk_size, c->d_flags.p, c->d_verdict.p,
      c->d_dag_dirty.p, exclude_dag_dirty, c->d_digest[c->cur].p, c->epoch, 0u, c->cache.p,
      c->cache_cap - c->staging_used, cursor, c->d_items.p + lo, res, c->h_scan.p + 8 * slot, ++c->scan_seq, vb0, vb1,
      c->d_tcs.p, c->d_xfold.p, c->cfg.dedup, c->d_buf_crc.p, c->d_verdict.p, fixed_base, direct ? 1 : 0,
      c->d_bitmap.p, c->n_chunks, q, q_seq, last_wave ? 1 : 0,
      ce_runs ? c->h_run.p + lo : nullptr, ce_runs ? c->h_run.p + c->n_chunks + lo : nullptr,
      ce_runs ? c->h_run.p + 2 * c->n_chunks + lo : nullptr);
  c->slot_seq[slot] = c->scan_seq;
  check_launch("k_pack_scan");
  c->timer_end(kTimScan, s);
  ++c->launches;
  ck(cudaEventRecord(c->scanned[slot], s), "event");
  if (direct && (q || ce_runs)) {  // shipped by the running drain / by the copy engine (host submits the runs)
    c->pack_pending = true;
    return;
  }
  if (direct) {  // chunks go straight to the host image from the drain stream
    ck(cudaStreamWaitEvent(direct_stream, c->scanned[slot], 0), "wait scan");
    if (slot == 0) c->timer_begin(kTimD2H, direct_stream);
    launch_copy_host(c, c->d_items.p + lo, res + 3, 0, direct_stream);
    ck(cudaEventRecord(c->copied[slot], direct_stream), "event");
    c->pack_pending = true;
    return;
  }
  bool aligned = c->cfg.chunk_size % 16 == 0;
  for (const auto& b : c->bufs) aligned = aligned && (b.dev_ptr % 16 == 0);
  c->timer_begin(kTimCopy, s);
  launch_copy(c, c->d_items.p + lo, res + 3, 0, aligned, s);
  c->timer_end(kTimCopy, s);
  ck(cudaEventRecord(c->copied[slot], s), "event");
  c->pack_pending = true;
}

// Tiled scan (copy-engine direct mode): index entries + runs of [lo, hi)
// over many CTAs with decoupled look-back.
static void launch_scan_tiles(pos_ctx* c, int exclude_dag_dirty, cudaStream_t s, uint64_t lo, uint64_t hi,
                              uint32_t slot, bool chain_start) {
  upload_dag_flags(c, s);
  const uint64_t words = (hi + 31) / 32 - lo / 32;
  const uint32_t wpt = words <= 16ull * 2 * (uint64_t)c->crc.sm_count ? 16u : 64u;  // 1 or 4 rounds per warp
  const uint32_t ntiles = (uint32_t)std::max<uint64_t>(1, (words + wpt - 1) / wpt);
  if (c->d_tiles.n < ntiles) {
    ck(cudaStreamSynchronize(s), "sync");
    c->d_tiles.ensure(ntiles);
    ck(cudaMemset(c->d_tiles.p, 0, ntiles * sizeof(TileStatus)), "tiles");
  }
  if (!c->d_tile_ctl.p) {
    c->d_tile_ctl.ensure(pos_ctx::kMaxWaves);
    ck(cudaMemset(c->d_tile_ctl.p, 0, pos_ctx::kMaxWaves * sizeof(TileCtl)), "tile ctl");
  }
  uint64_t* res = c->d_scan.p + 8 * slot;
  c->timer_begin(kTimScan, s);
  k_scan_tiles<<<ntiles, kScanThreads, 0, s>>>(
      c->d_bufs.p, c->d_chunk_map.p, lo, hi, c->cfg.chunk_size, c->d_flags.p, c->d_verdict.p, c->d_dag_dirty.p,
      exclude_dag_dirty, c->d_digest[c->cur].p, c->epoch, c->cache.p, c->cache_cap - c->staging_used,
      c->d_cursor.p, chain_start ? 0ull : ~0ull, res, c->h_scan.p + 8 * slot, ++c->scan_seq, c->d_bitmap.p,
      c->n_chunks, c->h_run.p + lo, c->h_run.p + c->n_chunks + lo, c->h_run.p + 2 * c->n_chunks + lo, c->d_tiles.p,
      c->d_tile_ctl.p + slot, wpt);
  c->slot_seq[slot] = c->scan_seq;
  check_launch("k_scan_tiles");
  c->timer_end(kTimScan, s);
  ++c->launches;
  ck(cudaEventRecord(c->scanned[slot], s), "event");
  c->pack_pending = true;
}

struct PackResult {
  uint64_t base, total, n, payload;
};

static PackResult pack_result(pos_ctx* c, uint32_t slot) {
  // Spin on the sequence number the scan kernel writes into mapped host memory
  // (wakes within ~1 us; an event sync costs ~30 us), bounded by the event.
  volatile uint64_t* seqp = c->h_scan.p + 8 * slot + 5;
  for (uint32_t spins = 0; *seqp != c->slot_seq[slot]; ++spins) {
    if ((spins & 1023) == 1023 && cudaEventQuery(c->scanned[slot]) == cudaSuccess) break;
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  ck(cudaEventSynchronize(c->scanned[slot]), "scan sync");  // surfaces kernel faults
  const uint64_t* r = c->h_scan.p + 8 * slot;
  if (r[2]) {
    c->precopy_bytes = 0;
    c->pack_pending = false;
    fail(POS_E_STAGING_EXHAUSTED, "pack of " + std::to_string(r[1]) + " B at cache offset " +
                                      std::to_string(r[4]) + " exceeds the cache of " +
                                      std::to_string(c->cache_cap) + " B");
  }
  return PackResult{r[4], r[1], r[0], r[6]};
}

static uint64_t pack_size(pos_ctx* c) {
  if (!c->pack_pending) fail(POS_E_BAD_STATE, "no pre-copy pack in flight");
  PackResult r = pack_result(c, 0);
  c->pack_pending = false;
  c->precopy_bytes = r.total;
  return r.total;
}

static void hash_range(pos_ctx* c, uint64_t lo, uint64_t hi, cudaStream_t s, uint32_t wave,
                       ShipQueue* q = nullptr, unsigned long long q_seq = 0) {
  if (hi <= lo) return;
  HashParams p{};
  p.q = q;
  p.q_seq = q_seq;
  p.dedup = c->cfg.dedup;
  p.bufs = c->d_bufs.p;
  p.chunk_map = c->d_chunk_map.p;
  p.n_items = hi - lo;
  p.item_base = lo;
  p.chunk_size = c->cfg.chunk_size;
  p.k_full = zeros_crc(c->cfg.chunk_size);
  p.tables = c->crc.tables.p;
  p.xinv = c->crc.xinv.p;
  p.digest_cur = c->d_digest[c->cur].p;
  p.digest_prev = c->d_digest[c->cur ^ 1].p;
  p.flags = c->d_flags.p;
  p.bitmap = nullptr;  // the wave's k_pack_scan writes its bitmap words (one ballot per word)
  p.prev_valid = c->prev_valid ? 1 : 0;
  set_segments(c, hi - lo, p);
  int grid = c->hash_grid((hi - lo) * p.nseg);
  ck(cudaEventRecord(c->wave_hash[wave][0], s), "event");
  launch_hash<kModeHash>(grid, s, p);
  check_launch("k_hash_chunks");
  ck(cudaEventRecord(c->wave_hash[wave][1], s), "event");
  ++c->launches;
}


int pos_compact(pos_ctx* c, int exclude_dag_dirty, void* stream, uint64_t* pack_bytes) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    launch_pack(c, exclude_dag_dirty, S(stream), 0, c->n_chunks, 0, 0, 0, ~0ull, nullptr, false, true);
    uint64_t total = pack_size(c);
    if (pack_bytes) *pack_bytes = total;
  });
}

int pos_precopy(pos_ctx* c, int exclude_dag_dirty, void* stream) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(stream);
    int rc = pos_hash_chunks(c, stream);
    if (rc != POS_OK) throw Fail{rc};
    rc = pos_buffer_crc(c, stream);
    if (rc != POS_OK) throw Fail{rc};
    launch_pack(c, exclude_dag_dirty, s, 0, c->n_chunks, 0, 0, 0, ~0ull, nullptr, false, true);
  });
}

int pos_precopy_pipelined(pos_ctx* c, int exclude_dag_dirty, uint32_t waves, void* ckpt_stream,
                          void* copy_stream, void* host_dst, uint64_t slice, uint64_t* offsets,
                          uint64_t* sizes, uint32_t* n_packs) {
  return guarded([&] {
    if (!c || !offsets || !sizes || !n_packs) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(ckpt_stream), cs = S(copy_stream);
    const uint32_t nb = (uint32_t)c->bufs.size();
    uint32_t W = std::max<uint32_t>(1, std::min<uint32_t>(waves, pos_ctx::kMaxWaves));
    W = std::min<uint32_t>(W, std::max<uint32_t>(nb, 1));
    // Wave boundaries at buffer starts, ~equal chunk counts (O1 needs whole buffers).
    std::vector<uint32_t> bb(1, 0);
    for (uint32_t w = 1; w < W; ++w) {
      uint64_t target = c->n_chunks * w / W;
      uint32_t b = bb.back();
      while (b < nb && c->chunk_base[b] < target) ++b;
      if (b > bb.back() && b < nb) bb.push_back(b);
    }
    bb.push_back(nb);
    W = (uint32_t)bb.size() - 1;
    auto chunk_of = [&](uint32_t b) { return b < nb ? c->chunk_base[b] : c->n_chunks; };
    upload_dag_flags(c, s, cs);  // on the copy stream, under the first hash
    c->timer_begin(kTimHash, s);
    for (uint32_t w = 0; w < W; ++w) {
      hash_range(c, chunk_of(bb[w]), chunk_of(bb[w + 1]), s, w);
      // O1 verdicts fused into the scan: one launch less on the critical path
      launch_pack(c, exclude_dag_dirty, s, chunk_of(bb[w]), chunk_of(bb[w + 1]), w, bb[w], bb[w + 1], ~0ull,
                  nullptr, false, w == 0);
    }
    c->timer_end(kTimHash, s);
    c->waves_last = W;
    uint64_t end = 0;
    for (uint32_t w = 0; w < W; ++w) {
      PackResult r = pack_result(c, w);
      offsets[w] = r.base;
      sizes[w] = r.total;
      end = r.base + (r.total + kPackAlign - 1) / kPackAlign * kPackAlign;
      if (host_dst) {
        ck(cudaStreamWaitEvent(cs, c->copied[w], 0), "wait copy");
        if (w == 0) c->timer_begin(kTimD2H, cs);
        if (slice == 0) slice = 8ull << 20;
        for (uint64_t o = 0; o < r.total; o += slice)
          ck(cudaMemcpyAsync(static_cast<uint8_t*>(host_dst) + r.base + o, c->cache.p + r.base + o,
                             std::min(slice, r.total - o), cudaMemcpyDeviceToHost, cs),
             "d2h");
      }
    }
    if (host_dst) c->timer_end(kTimD2H, cs);
    c->pack_pending = false;
    c->precopy_bytes = end;
    *n_packs = W;
  });
}

static void precopy_stream_peer(pos_ctx* c, int exclude_dag_dirty, cudaStream_t s, cudaStream_t cs,
                                uint64_t region, const std::vector<uint64_t>& cuts,
                                const std::function<uint32_t(uint64_t)>& vb_of, pos_pack_sink sink,
                                void* user, uint64_t* total_bytes);

int pos_precopy_stream(pos_ctx* c, int exclude_dag_dirty, void* ckpt_stream, void* copy_stream,
                       uint64_t region, pos_pack_sink sink, void* user, uint64_t* total_bytes,
                       uint32_t* n_packs) {
  return guarded([&] {
    if (!c || !sink) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(ckpt_stream), cs = S(copy_stream);
    if (region == 0) region = c->cache_cap / 2;
    region = region / kPackAlign * kPackAlign;
    if (2 * region > c->cache_cap) fail(POS_E_INVALID_ARGUMENT, "two regions must fit the cache");
    const uint64_t csz = c->cfg.chunk_size;
    const uint32_t nb = (uint32_t)c->bufs.size();
    // Waves = chunk ranges whose worst-case pack (every chunk dirty) fits a region.
    std::vector<uint64_t> cuts(1, 0);
    uint64_t acc_n = 0, acc_b = 0;
    for (uint64_t g = 0; g < c->n_chunks; ++g) {
      uint32_t bi = 0;  // chunk length from the host tables
      {
        auto it = std::upper_bound(c->chunk_base.begin(), c->chunk_base.end(), g);
        bi = (uint32_t)(it - c->chunk_base.begin()) - 1;
      }
      const DevBuf& b = c->hbufs[bi];
      uint32_t k = (uint32_t)(g - c->chunk_base[bi]);
      uint64_t len = k + 1 == b.nchunks ? b.size - (uint64_t)k * csz : csz;
      uint64_t nb_ = acc_b + round_up(len, 16), nn = acc_n + 1;
      if (round_up(kPackHeader + kPackEntry * nn, kPackAlign) + nb_ > region && acc_n > 0) {
        cuts.push_back(g);
        acc_n = 1;
        acc_b = round_up(len, 16);
      } else {
        acc_n = nn;
        acc_b = nb_;
      }
      if (round_up(kPackHeader + kPackEntry * acc_n, kPackAlign) + acc_b > region)
        fail(POS_E_STAGING_EXHAUSTED, "a single chunk exceeds the cache region");
    }
    cuts.push_back(c->n_chunks);
    const uint32_t W = (uint32_t)cuts.size() - 1;
    // Buffers whose O1 verdict is decided in wave w: last chunk in [cuts[w], cuts[w+1]).
    auto vb_of = [&](uint64_t g) {  // first buffer whose last chunk >= g
      uint32_t b = 0;
      while (b < nb && c->chunk_base[b] + c->hbufs[b].nchunks <= g) ++b;
      return b;
    };
    c->h_land[0].ensure(region);
    c->h_land[1].ensure(region);
    if (!c->ev_d2h[0]) {
      ck(cudaEventCreateWithFlags(&c->ev_d2h[0], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&c->ev_d2h[1], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&c->ev_copied2[0], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&c->ev_copied2[1], cudaEventDisableTiming), "event");
    }
    upload_dag_flags(c, s);
    ck(cudaMemsetAsync(c->d_verdict.p, 0, std::max<uint32_t>(nb, 1), s), "memset verdicts");
    if (c->peer) {
      uint64_t total = 0;
      c->timer_begin(kTimHash, s);
      precopy_stream_peer(c, exclude_dag_dirty, s, cs, region, cuts, vb_of, sink, user, &total);
      c->timer_end(kTimHash, s);
      c->pack_pending = false;
      c->precopy_bytes = 0;
      c->waves_last = std::min<uint32_t>(W, pos_ctx::kMaxWaves);
      if (total_bytes) *total_bytes = total;
      if (n_packs) *n_packs = W;
      return;
    }
    std::vector<uint64_t> sizes(W, 0);
    uint64_t total = 0;
    auto finish = [&](uint32_t w) {  // wave w's bytes are on the host: hand them over
      ck(cudaEventSynchronize(c->ev_d2h[w & 1]), "d2h sync");
      sink(user, c->h_land[w & 1].p, sizes[w], w);
    };
    c->timer_begin(kTimHash, s);
    for (uint32_t w = 0; w < W; ++w) {
      const uint32_t r = w & 1;
      if (w >= 2) finish(w - 2);  // frees landing slot r and (its D2H done) cache region r
      hash_range(c, cuts[w], cuts[w + 1], s, w % pos_ctx::kMaxWaves);
      if (w >= 2) ck(cudaStreamWaitEvent(s, c->ev_d2h[r], 0), "wait region");  // before writing region r
      const uint32_t slot = w % pos_ctx::kMaxWaves;
      launch_pack(c, exclude_dag_dirty, s, cuts[w], cuts[w + 1], slot, vb_of(cuts[w]), vb_of(cuts[w + 1]),
                  (uint64_t)r * region);
      ck(cudaEventRecord(c->ev_copied2[r], s), "event");
      PackResult res = pack_result(c, slot);
      sizes[w] = res.total;
      total += res.total;
      ck(cudaStreamWaitEvent(cs, c->ev_copied2[r], 0), "wait copy");
      for (uint64_t o = 0; o < res.total; o += 8ull << 20)
        ck(cudaMemcpyAsync(c->h_land[r].p + o, c->cache.p + res.base + o, std::min<uint64_t>(8ull << 20, res.total - o),
                           cudaMemcpyDeviceToHost, cs),
           "d2h");
      ck(cudaEventRecord(c->ev_d2h[r], cs), "event");
    }
    c->timer_end(kTimHash, s);
    for (uint32_t w = W >= 2 ? W - 2 : 0; w < W; ++w) finish(w);
    c->pack_pending = false;
    c->precopy_bytes = 0;  // every pack has left the cache
    c->waves_last = std::min<uint32_t>(W, pos_ctx::kMaxWaves);
    if (total_bytes) *total_bytes = total;
    if (n_packs) *n_packs = W;
  });
}

static void peer_release(pos_ctx* c) {
  if (!c->peer) return;
  PeerCache* P = c->peer;
  cudaSetDevice(P->device);
  if (P->stream) cudaStreamSynchronize(P->stream);
  for (auto e : P->in) if (e) cudaEventDestroy(e);
  for (auto e : P->free_) if (e) cudaEventDestroy(e);
  for (auto e : {P->land[0], P->land[1], P->t0, P->captured, P->drained}) if (e) cudaEventDestroy(e);
  if (P->base) cudaFree(P->base);
  if (P->stream) cudaStreamDestroy(P->stream);
  cudaSetDevice(c->cfg.device);
  delete P;
  c->peer = nullptr;
}

int pos_peer_cache_attach(pos_ctx* c, int peer_device, uint64_t bytes) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    int n = 0;
    ck(cudaGetDeviceCount(&n), "device count");
    if (peer_device < 0 || peer_device >= n) fail(POS_E_INVALID_ARGUMENT, "bad peer device ordinal");
    peer_release(c);
    if (bytes == 0) return;  // detach
    auto* P = new PeerCache();
    c->peer = P;
    P->device = peer_device;
    const int dev = c->cfg.device;
    if (peer_device != dev) {  // NVLink / NVSwitch path both ways
      int ok = 0;
      ck(cudaDeviceCanAccessPeer(&ok, dev, peer_device), "can access peer");
      if (ok) {
        ck(cudaSetDevice(dev), "cudaSetDevice");
        cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "enable peer access");
        cudaGetLastError();
      }
    }
    ck(cudaSetDevice(peer_device), "cudaSetDevice(peer)");
    cudaError_t e = cudaMalloc(&P->base, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      cudaSetDevice(dev);
      peer_release(c);
      fail(POS_E_OUT_OF_DEVICE_MEMORY, "peer cache of " + std::to_string(bytes) + " B on device " +
                                           std::to_string(peer_device));
    }
    P->bytes = bytes;
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "prio");
    ck(cudaStreamCreateWithPriority(&P->stream, cudaStreamNonBlocking, lo), "peer stream");
    for (auto* ev : {&P->land[0], &P->land[1]}) ck(cudaEventCreateWithFlags(ev, cudaEventDisableTiming), "event");
    ck(cudaEventCreate(&P->drained), "event");
    ck(cudaSetDevice(dev), "cudaSetDevice");
    ck(cudaEventCreate(&P->t0), "event");
    ck(cudaEventCreate(&P->captured), "event");
  });
}

int pos_peer_cache_stats(pos_ctx* c, float* capture_ms, float* total_ms) {
  return guarded([&] {
    if (!c || !c->peer) fail(POS_E_BAD_STATE, "no peer cache attached");
    if (capture_ms) *capture_ms = c->peer->capture_ms;
    if (total_ms) *total_ms = c->peer->total_ms;
  });
}

// Cache-cycled pre-copy through the peer cache.  A capture thread runs the
// waves (hash -> O1 -> scan -> compaction into local region w%2 -> peer slot
// w%M) without waiting for the host; the calling thread drains peer slots
// into the two landing slots on the peer's stream and hands packs to the
// sink in order.  Slot reuse is event-ordered on the device; the only host
// hand-offs are "wave w is in its slot" and "slot m is drained".
static void precopy_stream_peer(pos_ctx* c, int exclude_dag_dirty, cudaStream_t s, cudaStream_t cs,
                                uint64_t region, const std::vector<uint64_t>& cuts,
                                const std::function<uint32_t(uint64_t)>& vb_of, pos_pack_sink sink,
                                void* user, uint64_t* total_bytes) {
  PeerCache& P = *c->peer;
  const int dev = c->cfg.device;
  const uint32_t W = (uint32_t)cuts.size() - 1;
  const uint32_t M = (uint32_t)(P.bytes / region);
  if (M == 0) fail(POS_E_STAGING_EXHAUSTED, "peer cache smaller than one cache region");
  if (P.in.size() < M) {
    ck(cudaSetDevice(dev), "cudaSetDevice");
    while (P.in.size() < M) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      P.in.push_back(e);
    }
    ck(cudaSetDevice(P.device), "cudaSetDevice(peer)");
    while (P.free_.size() < M) {
      cudaEvent_t e;
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      P.free_.push_back(e);
    }
    ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  cudaEvent_t local_free[2] = {c->ev_d2h[0], c->ev_d2h[1]};  // local region r reusable
  std::vector<uint64_t> sizes(W, 0);
  std::mutex mu;
  std::condition_variable cv;
  uint32_t captured = 0, drained = 0;  // waves in a slot / slots drained (enqueued)
  std::string err;
  int err_code = POS_E_CUDA;
  ck(cudaEventRecord(P.t0, s), "event");
  std::thread cap([&] {
    try {
      ck(cudaSetDevice(dev), "cudaSetDevice");
      for (uint32_t w = 0; w < W; ++w) {
        const uint32_t r = w & 1, m = w % M;
        hash_range(c, cuts[w], cuts[w + 1], s, w % pos_ctx::kMaxWaves);
        if (w >= 2) ck(cudaStreamWaitEvent(s, local_free[r], 0), "wait region");
        const uint32_t slot = w % pos_ctx::kMaxWaves;
        launch_pack(c, exclude_dag_dirty, s, cuts[w], cuts[w + 1], slot, vb_of(cuts[w]), vb_of(cuts[w + 1]),
                    (uint64_t)r * region);
        ck(cudaEventRecord(c->ev_copied2[r], s), "event");
        PackResult res = pack_result(c, slot);
        if (w >= M) {  // slot m must have been drained (its D2H enqueued, then done on the device)
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return drained > w - M || !err.empty(); });
          if (!err.empty()) return;
          ck(cudaStreamWaitEvent(cs, P.free_[m], 0), "wait slot");
        }
        ck(cudaStreamWaitEvent(cs, c->ev_copied2[r], 0), "wait pack");
        ck(cudaMemcpyPeerAsync(P.base + (uint64_t)m * region, P.device, c->cache.p + res.base, dev, res.total, cs),
           "peer copy");
        ck(cudaEventRecord(local_free[r], cs), "event");
        ck(cudaEventRecord(P.in[m], cs), "event");
        std::lock_guard<std::mutex> lk(mu);
        sizes[w] = res.total;
        ++captured;
        cv.notify_all();
      }
      ck(cudaEventRecord(P.captured, cs), "event");
    } catch (const Fail& f) {
      std::lock_guard<std::mutex> lk(mu);
      err = g_last_error.empty() ? "capture failed" : g_last_error;  // this thread's message
      err_code = f.code;
      cv.notify_all();
    }
  });
  uint64_t total = 0;
  auto finish = [&](uint32_t w) {
    ck(cudaEventSynchronize(P.land[w & 1]), "d2h sync");
    sink(user, c->h_land[w & 1].p, sizes[w], w);
  };
  try {
    for (uint32_t w = 0; w < W; ++w) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return captured > w || !err.empty(); });
        if (!err.empty()) break;
      }
      if (w >= 2) finish(w - 2);  // landing slot w&1 free
      const uint32_t m = w % M, l = w & 1;
      ck(cudaSetDevice(P.device), "cudaSetDevice(peer)");
      ck(cudaStreamWaitEvent(P.stream, P.in[m], 0), "wait slot in");
      for (uint64_t o = 0; o < sizes[w]; o += 8ull << 20)
        ck(cudaMemcpyAsync(c->h_land[l].p + o, P.base + (uint64_t)m * region + o,
                           std::min<uint64_t>(8ull << 20, sizes[w] - o), cudaMemcpyDeviceToHost, P.stream),
           "peer d2h");
      ck(cudaEventRecord(P.land[l], P.stream), "event");
      ck(cudaEventRecord(P.free_[m], P.stream), "event");
      ck(cudaSetDevice(dev), "cudaSetDevice");
      total += sizes[w];
      std::lock_guard<std::mutex> lk(mu);
      ++drained;
      cv.notify_all();
    }
  } catch (...) {
    {
      std::lock_guard<std::mutex> lk(mu);
      if (err.empty()) err = "drain failed";
      cv.notify_all();
    }
    cap.join();
    cudaSetDevice(dev);
    throw;
  }
  cap.join();
  ck(cudaSetDevice(dev), "cudaSetDevice");
  if (!err.empty()) fail(err_code, "peer pre-copy: " + err);
  for (uint32_t w = W >= 2 ? W - 2 : 0; w < W; ++w) finish(w);
  ck(cudaSetDevice(P.device), "cudaSetDevice(peer)");
  ck(cudaEventRecord(P.drained, P.stream), "event");
  ck(cudaEventSynchronize(P.drained), "sync");
  ck(cudaSetDevice(dev), "cudaSetDevice");
  ck(cudaEventElapsedTime(&P.capture_ms, P.t0, P.captured), "elapsed");
  // t0 (local device) -> drained (peer device): host-side gap is below the drain's length;
  // measured as capture + the peer drain's own span when the devices differ.
  if (P.device == dev) ck(cudaEventElapsedTime(&P.total_ms, P.t0, P.drained), "elapsed");
  else P.total_ms = -1.0f;
  *total_bytes = total;
}

int pos_register_image(pos_ctx* c, uint8_t* const* hosts, const uint64_t* sizes, uint32_t n) {
  return guarded([&] {
    if (!c || (!hosts && n) || (!sizes && n)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (n != c->bufs.size()) fail(POS_E_INVALID_ARGUMENT, "one image range per registered buffer");
    sync_provenance(c);
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    for (uint32_t i = 0; i < n; ++i) {
      if (!hosts[i] || sizes[i] != c->bufs[i].size)
        fail(POS_E_INVALID_ARGUMENT, "image range " + std::to_string(i) + " does not match its buffer");
      cudaPointerAttributes a{};
      cudaError_t e = cudaPointerGetAttributes(&a, hosts[i]);
      if (e != cudaSuccess) cudaGetLastError();
      if (e != cudaSuccess || a.type != cudaMemoryTypeHost) {  // pageable: pin + map it
        ck(cudaHostRegister(hosts[i], sizes[i], cudaHostRegisterMapped | cudaHostRegisterPortable),
           "cudaHostRegister(image)");
        c->image_pinned.push_back(hosts[i]);
      }
      void* dev = nullptr;
      ck(cudaHostGetDevicePointer(&dev, hosts[i], 0), "cudaHostGetDevicePointer(image)");
      c->hbufs[i].image = (uint64_t)dev;
    }
    if (n) ck(cudaMemcpy(c->d_bufs.p, c->hbufs.data(), n * sizeof(DevBuf), cudaMemcpyHostToDevice), "bufs");
    c->image_ready = n > 0;
    c->delta_ready = false;  // re-stage the delta with drain items
  });
}

// Longest a drain warp waits for one producer before giving up (and
// reporting POS_E_CUDA from pos_precopy_direct_result instead of hanging).
static unsigned long long watchdog_ns() {
  static const unsigned long long v = [] {
    const char* e = std::getenv("POSDUMP_WATCHDOG_MS");
    unsigned long long ms = e ? std::strtoull(e, nullptr, 10) : 10000;
    return (ms ? ms : 10000) * 1000000ull;
  }();
  return v;
}

int pos_debug_ship_queue(pos_ctx* c, uint64_t* out14) {
  return guarded([&] {
    if (!c || !out14) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->d_q.p) fail(POS_E_BAD_STATE, "no ship queue");
    ShipQueue h{};
    ck(cudaMemcpy(&h, c->d_q.p, sizeof h, cudaMemcpyDeviceToHost), "queue");
    const uint64_t v[6] = {h.tail, h.head, h.done, h.exited, h.error, c->q_seq};
    std::memcpy(out14, v, sizeof v);
    std::memcpy(out14 + 6, h.dbg, sizeof h.dbg);
  });
}

int pos_precopy_direct(pos_ctx* c, int exclude_dag_dirty, uint32_t waves, void* ckpt_stream,
                       void* drain_stream) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->image_ready) fail(POS_E_BAD_STATE, "no host image registered (pos_register_image)");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(ckpt_stream), ds = S(drain_stream);
    if (s == ds) fail(POS_E_INVALID_ARGUMENT, "the drain needs its own stream");
    const uint32_t nb = (uint32_t)c->bufs.size();
    uint32_t W = std::max<uint32_t>(1, std::min<uint32_t>(waves, pos_ctx::kMaxWaves));
    W = std::min<uint32_t>(W, std::max<uint32_t>(nb, 1));
    // Waves of whole buffers (O1), ~equal chunk counts -- except an optional
    // small first wave (POSDUMP_FIRST_WAVE = fraction of the chunks) so the
    // host leg starts after a short hash + scan while the rest is hashed.
    static const double first = [] {
      const char* e = std::getenv("POSDUMP_FIRST_WAVE");
      return e ? std::atof(e) : 0.0;
    }();
    std::vector<uint32_t> bb(1, 0);
    for (uint32_t w = 1; w < W; ++w) {
      uint64_t target = c->n_chunks * w / W;
      if (first > 0 && first < 1)
        target = (uint64_t)(c->n_chunks * (first + (1 - first) * (double)(w - 1) / (W - 1)));
      uint32_t b = bb.back();
      while (b < nb && c->chunk_base[b] < target) ++b;
      if (b > bb.back() && b < nb) bb.push_back(b);
    }
    bb.push_back(nb);
    W = (uint32_t)bb.size() - 1;
    auto chunk_of = [&](uint32_t b) { return b < nb ? c->chunk_base[b] : c->n_chunks; };
    // The index packs' worst case (every chunk shipped) is reserved up front,
    // so the STW delta's place in the cache is known without waiting.
    uint64_t reserve = 0;
    for (uint32_t w = 0; w < W; ++w)
      reserve += round_up(kPackHeader + kPackEntry * (chunk_of(bb[w + 1]) - chunk_of(bb[w])), kPackAlign);
    if (reserve > c->cache_cap - c->staging_used) fail(POS_E_STAGING_EXHAUSTED, "index packs exceed the cache");
    upload_dag_flags(c, s, ds);  // on the drain stream, under the first hash
    // Host leg of the direct mode (POSDUMP_DIRECT_DRAIN):
    //   ce    (default) the copy engine moves runs of shipped chunks straight
    //         into the image (cudaMemcpyBatchAsync over the scan's run lists);
    //   queue SM warps drain a ship queue fed by the hash (starts earliest, but
    //         SM stores over PCIe slow concurrent HBM kernels ~4x: measured);
    //   sm    k_copy_host after each wave's scan.
    const int drain_mode = direct_drain_mode();
    if (drain_mode == 0) {
      c->h_run.ensure(3 * std::max<uint64_t>(c->n_chunks, 1));
      c->timer_begin(kTimHash, s);
      for (uint32_t w = 0; w < W; ++w) {
        hash_range(c, chunk_of(bb[w]), chunk_of(bb[w + 1]), s, w);
        // O1 as its own wide launch (one warp per buffer, all SMs) rather
        // than inside the one-CTA scan, where candidates queue behind 16 warps
        upload_dag_flags(c, s);
        const uint32_t nbw = bb[w + 1] - bb[w];
        if (nbw) {
          k_buffer_crc<<<(nbw + 7) / 8, 256, 0, s>>>(c->d_bufs.p + bb[w], nbw, c->d_digest[c->cur].p, c->d_tcs.p,
                                                     c->d_xfold.p + bb[w], c->d_dag_dirty.p + bb[w], c->cfg.dedup, 0,
                                                     c->d_buf_crc.p + bb[w], c->d_verdict.p + bb[w]);
          check_launch("k_buffer_crc");
          ++c->launches;
        }
        static const bool tiled = [] {
          const char* e = std::getenv("POSDUMP_SCAN");  // "single": the one-CTA k_pack_scan
          return !(e && !std::strcmp(e, "single"));
        }();
        if (tiled)
          launch_scan_tiles(c, exclude_dag_dirty, s, chunk_of(bb[w]), chunk_of(bb[w + 1]), w, w == 0);
        else
          launch_pack(c, exclude_dag_dirty, s, chunk_of(bb[w]), chunk_of(bb[w + 1]), w, 0, 0, ~0ull,
                      ds, true, w == 0, nullptr, 0, false, true);
        c->direct_lo[w] = (uint32_t)chunk_of(bb[w]);
      }
      c->timer_end(kTimHash, s);
      // each wave's runs go to the copy engine the moment its scan lands
      cudaMemcpyAttributes attr{};
      attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
      attr.srcLocHint.type = cudaMemLocationTypeDevice;
      attr.srcLocHint.id = c->cfg.device;
      attr.dstLocHint.type = cudaMemLocationTypeHost;
      attr.flags = ce_flags();
      for (uint32_t w = 0; w < W; ++w) {
        pack_result(c, w);
        const uint64_t nr = c->h_scan.p[8 * w + 7];
        const uint64_t lo = c->direct_lo[w];
        if (w == 0) c->timer_begin(kTimD2H, ds);
        if (nr) {
          size_t zero = 0, fail_idx = 0;
          ck(cudaMemcpyBatchAsync(reinterpret_cast<void**>(c->h_run.p + c->n_chunks + lo),
                                  reinterpret_cast<void**>(c->h_run.p + lo),
                                  reinterpret_cast<size_t*>(c->h_run.p + 2 * c->n_chunks + lo), nr, &attr, &zero,
                                  1, &fail_idx, ds),
             "cudaMemcpyBatchAsync(direct runs)");
        }
      }
      c->timer_end(kTimD2H, ds);
      c->waves_last = W;
      c->direct_waves = W;
      c->direct_pending = true;
      c->pack_pending = false;
      c->precopy_bytes = reserve;
      return;
    }
    ShipQueue* q = nullptr;
    if (drain_mode == 1) {
      // Ship queue: chunks leave while the rest is still being hashed.
      const uint64_t cap = c->n_chunks + 2 * kDrainCtas * (kDrainThreads / 32) + 64;
      if (!c->d_q.p || c->d_qslots.n < cap) {
        ck(cudaStreamSynchronize(ds), "sync");
        c->d_qslots.ensure(cap);
        ck(cudaMemset(c->d_qslots.p, 0, cap * sizeof(unsigned long long)), "memset slots");
        c->d_q.ensure(1);
        ShipQueue hq{};
        hq.slots = c->d_qslots.p;
        ck(cudaMemcpy(c->d_q.p, &hq, sizeof hq, cudaMemcpyHostToDevice), "queue");
        c->q_seq = 0;
        if (!c->ev_drained) ck(cudaEventCreateWithFlags(&c->ev_drained, cudaEventDisableTiming), "event");
        ck(cudaEventRecord(c->ev_drained, ds), "event");
      }
      q = c->d_q.p;
      ++c->q_seq;
      ck(cudaStreamWaitEvent(s, c->ev_drained, 0), "wait queue reset");  // previous drain gone
      c->timer_begin(kTimD2H, ds);
      k_drain_queue<<<kDrainCtas, kDrainThreads, 0, ds>>>(q, c->q_seq, c->d_bufs.p, c->d_chunk_map.p,
                                                         c->cfg.chunk_size,
                                                         exclude_dag_dirty ? c->d_dag_dirty.p : nullptr,
                                                         watchdog_ns());
      check_launch("k_drain_queue");
      ++c->launches;
    }
    c->timer_begin(kTimHash, s);
    for (uint32_t w = 0; w < W; ++w) {
      hash_range(c, chunk_of(bb[w]), chunk_of(bb[w + 1]), s, w, q, c->q_seq);
      launch_pack(c, exclude_dag_dirty, s, chunk_of(bb[w]), chunk_of(bb[w + 1]), w, bb[w], bb[w + 1], ~0ull,
                  ds, true, w == 0, q, c->q_seq, w + 1 == W);
    }
    c->timer_end(kTimHash, s);
    c->timer_end(kTimD2H, ds);
    if (q) ck(cudaEventRecord(c->ev_drained, ds), "event");
    c->waves_last = W;
    c->direct_waves = W;
    c->direct_pending = true;
    c->pack_pending = false;
    c->precopy_bytes = reserve;
  });
}

int pos_precopy_direct_result(pos_ctx* c, uint64_t* chunks, uint64_t* payload_bytes, uint64_t* index_bytes) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->direct_pending) fail(POS_E_BAD_STATE, "no direct pre-copy in flight");
    uint64_t n = 0, pay = 0, end = 0;
    for (uint32_t w = 0; w < c->direct_waves; ++w) {
      PackResult r = pack_result(c, w);
      n += r.n;
      pay += r.payload;
      end = r.base + round_up(r.total, kPackAlign);
    }
    c->direct_pending = false;  // the index packs stay in [0, end) of the cache
    if (c->d_q.p) {  // watchdog of the ship-queue drain
      unsigned long long err = 0;
      ck(cudaMemcpy(&err, &c->d_q.p->error, sizeof err, cudaMemcpyDeviceToHost), "queue error");
      if (err) {
        ck(cudaMemset(&c->d_q.p->error, 0, sizeof err), "queue error reset");
        fail(POS_E_CUDA, "ship-queue drain watchdog fired (pre-copy " + std::to_string(err) + ")");
      }
    }
    if (chunks) *chunks = n;
    if (payload_bytes) *payload_bytes = pay;
    if (index_bytes) *index_bytes = end;
  });
}

int pos_delta_drain(pos_ctx* c, void* stream) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->drain_pending) fail(POS_E_BAD_STATE, "no STW delta to drain (pos_delta_copy with an image)");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    c->drain_pending = false;
    if (!c->drain_n) return;
    if (direct_drain_mode() == 0 && c->drun_n) {
      cudaMemcpyAttributes attr{};
      attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
      attr.srcLocHint.type = cudaMemLocationTypeDevice;
      attr.srcLocHint.id = c->cfg.device;
      attr.dstLocHint.type = cudaMemLocationTypeHost;
      attr.flags = ce_flags();
      size_t zero = 0, fail_idx = 0;
      const uint64_t r = c->drun_n;
      ck(cudaMemcpyBatchAsync(reinterpret_cast<void**>(c->h_drun.p + r), reinterpret_cast<void**>(c->h_drun.p),
                              reinterpret_cast<size_t*>(c->h_drun.p + 2 * r), r, &attr, &zero, 1, &fail_idx,
                              S(stream)),
         "cudaMemcpyBatchAsync(delta runs)");
      return;
    }
    launch_copy_host(c, c->d_drain_items.p, nullptr, c->drain_n, S(stream));
  });
}

int pos_stage_buffers(pos_ctx* c, const uint64_t* handles, uint32_t n, void* stream, uint64_t* pack_offset,
                      uint64_t* pack_bytes) {
  return guarded([&] {
    if (!c || (n && !handles)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (c->pack_pending || c->direct_pending || c->precopy_bytes)
      fail(POS_E_BAD_STATE, "stage before this epoch's pre-copy (its packs may already hold the buffers)");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(stream);
    const uint64_t cs = c->cfg.chunk_size;
    // conflicts in the snapshot, ascending handle, not staged yet (gate_cow, cr.hpp:822-826)
    std::set<uint32_t> idx;
    for (uint32_t j = 0; j < n; ++j) {
      auto it = c->index_of.find(handles[j]);
      if (it == c->index_of.end()) continue;
      if (c->hbufs[it->second].flags & kBufStaged) continue;
      idx.insert(it->second);
    }
    std::vector<uint4> work;
    uint64_t payload = 0;
    uint32_t entry = 0;
    for (uint32_t i : idx) {
      const DevBuf& b = c->hbufs[i];
      for (uint32_t q = 0; q < b.nchunks; ++q) {
        const uint64_t len = q + 1 == b.nchunks ? b.size - (uint64_t)q * cs : cs;
        const uint64_t g = c->chunk_base[i] + q;
        work.push_back(make_uint4((uint32_t)g, entry++, (uint32_t)payload, (uint32_t)(payload >> 32)));
        payload += round_up(len, 16);
      }
    }
    const uint64_t ne = work.size();
    const uint64_t payload_off = round_up(kPackHeader + kPackEntry * ne, kPackAlign);
    const uint64_t total = payload_off + payload;
    const uint64_t span = round_up(total, kPackAlign);
    // stage_buffers: staging_used_ + bytes <= staging_capacity() (cr.hpp:860)
    if (c->staging_used + span > c->cache_cap)
      fail(POS_E_STAGING_EXHAUSTED, "staging " + std::to_string(total) + " B exceeds the free cache");
    if (pack_offset) *pack_offset = 0;
    if (pack_bytes) *pack_bytes = 0;
    if (!ne) return;
    const uint64_t offset = c->cache_cap - c->staging_used - span;
    uint8_t* pack = c->cache.p + offset;
    const uint64_t work_bytes = ne * sizeof(uint4);
    if (c->stage_free) ck(cudaEventSynchronize(c->stage_free), "stage sync");
    c->h_stage.ensure(kPackHeader + work_bytes + idx.size() * sizeof(DevBuf));
    uint8_t* st = c->h_stage.p;
    std::memset(st, 0, kPackHeader);
    uint32_t magic = kPackMagic, ver = 1, nn = (uint32_t)ne, flags = kPackFlagStaged;
    std::memcpy(st + 0, &magic, 4);
    std::memcpy(st + 4, &ver, 4);
    std::memcpy(st + 8, &cs, 8);
    std::memcpy(st + 16, &nn, 4);
    std::memcpy(st + 20, &flags, 4);
    std::memcpy(st + 24, &payload_off, 8);
    std::memcpy(st + 32, &payload, 8);
    std::memcpy(st + 40, &c->epoch, 8);
    std::memcpy(st + 48, &total, 8);
    std::memcpy(st + kPackHeader, work.data(), work_bytes);
    ck(cudaMemcpyAsync(pack, st, kPackHeader, cudaMemcpyHostToDevice, s), "staging header");
    if (payload_off > kPackHeader + kPackEntry * ne)
      ck(cudaMemsetAsync(pack + kPackHeader + kPackEntry * ne, 0, payload_off - kPackHeader - kPackEntry * ne, s),
         "gap");
    c->d_stage_work.ensure(ne);  // own array: the delta's work list may be staged concurrently
    ck(cudaMemcpyAsync(c->d_stage_work.p, st + kPackHeader, work_bytes, cudaMemcpyHostToDevice, s), "work");
    // the buffers become kBufStaged: the pre-copy hash keeps their staged digests
    DevBuf* upd = reinterpret_cast<DevBuf*>(st + kPackHeader + work_bytes);
    uint32_t u = 0;
    for (uint32_t i : idx) {
      c->hbufs[i].flags |= kBufStaged;
      upd[u] = c->hbufs[i];
      ck(cudaMemcpyAsync(c->d_bufs.p + i, upd + u, sizeof(DevBuf), cudaMemcpyHostToDevice, s), "stage flag");
      ++u;
      c->staged.push_back(i);
    }
    ck(cudaEventRecord(c->stage_free, s), "event");
    // hash while copying: staged digests + entries + payload (the stop-point bytes)
    HashParams p{};
    p.bufs = c->d_bufs.p;
    p.chunk_map = c->d_chunk_map.p;
    p.n_items = ne;
    p.chunk_size = cs;
    p.k_full = zeros_crc(cs);
    p.tables = c->crc.tables.p;
    p.xinv = c->crc.xinv.p;
    p.digest_cur = c->d_digest[c->cur].p;
    p.work = c->d_stage_work.p;
    p.pack = pack;
    p.payload_off = payload_off;
    set_segments(c, ne, p);
    launch_hash<kModeCopy>(c->hash_grid(ne * p.nseg), s, p);
    check_launch("k_hash_chunks<copy>");
    ++c->launches;
    c->staging_used += span;
    if (pack_offset) *pack_offset = offset;
    if (pack_bytes) *pack_bytes = total;
  });
}

int pos_precopy_size(pos_ctx* c, uint64_t* pack_bytes) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    uint64_t total = pack_size(c);
    if (pack_bytes) *pack_bytes = total;
  });
}

static void delta_prepare(pos_ctx* c, cudaStream_t s) {
  const uint64_t cs = c->cfg.chunk_size;
  // at_final_stop: every buffer of dirty_set_ in the snapshot, ascending handle.
  const uint64_t offset = round_up(c->precopy_bytes, kPackAlign);
  std::vector<uint4> work;
  std::vector<CopyItem> items;
  std::vector<uint2> where;  // (buffer index, chunk) per entry
  uint64_t payload = 0;
  uint32_t entry = 0;
  bool aligned = cs % 16 == 0;
  for (uint64_t h : c->dirty_set) {
    uint32_t i = c->index_of.at(h);
    const DevBuf& b = c->hbufs[i];
    aligned = aligned && (b.ptr % 16 == 0);
    for (uint32_t k = 0; k < b.nchunks; ++k) {
      uint64_t len = k + 1 == b.nchunks ? b.size - (uint64_t)k * cs : cs;
      uint64_t g = c->chunk_base[i] + k;
      work.push_back(make_uint4((uint32_t)g, entry++, (uint32_t)payload, (uint32_t)(payload >> 32)));
      items.push_back(CopyItem{b.ptr + (uint64_t)k * cs, 0, len, round_up(len, 16)});
      items.back().dst = payload;  // relative; rebased below
      where.push_back(make_uint2(i, k));
      payload += round_up(len, 16);
    }
  }
  const uint64_t n = work.size();
  const uint64_t payload_off = round_up(kPackHeader + kPackEntry * n, kPackAlign);
  const uint64_t total = payload_off + payload;
  if (offset + total > c->cache_cap - c->staging_used)
    fail(POS_E_STAGING_EXHAUSTED, "delta pack exceeds the cache");
  uint8_t* pack = c->cache.p + offset;
  for (auto& it : items) it.dst = (uint64_t)pack + payload_off + it.dst;
  // Stage the header, the work list (for the post-stop hash) and the gather items.
  const uint64_t work_bytes = n * sizeof(uint4), item_bytes = n * sizeof(CopyItem);
  const uint64_t drain_bytes = c->image_ready ? item_bytes : 0;
  if (c->stage_free) ck(cudaEventSynchronize(c->stage_free), "stage sync");
  c->h_stage.ensure(kPackHeader + work_bytes + item_bytes + drain_bytes);
  uint8_t* st = c->h_stage.p;
  std::memset(st, 0, kPackHeader);
  uint32_t magic = kPackMagic, ver = 1, nn = (uint32_t)n, flags = 1;
  std::memcpy(st + 0, &magic, 4);
  std::memcpy(st + 4, &ver, 4);
  std::memcpy(st + 8, &cs, 8);
  std::memcpy(st + 16, &nn, 4);
  std::memcpy(st + 20, &flags, 4);
  std::memcpy(st + 24, &payload_off, 8);
  std::memcpy(st + 32, &payload, 8);
  std::memcpy(st + 40, &c->epoch, 8);
  std::memcpy(st + 48, &total, 8);
  if (n) {
    std::memcpy(st + kPackHeader, work.data(), work_bytes);
    std::memcpy(st + kPackHeader + work_bytes, items.data(), item_bytes);
    if (drain_bytes) {  // after the stop: gathered payload -> host image (chunk_copied, cr.hpp:499-501)
      CopyItem* d = reinterpret_cast<CopyItem*>(st + kPackHeader + work_bytes + item_bytes);
      for (uint64_t e = 0; e < n; ++e) {
        const uint2 cm = where[e];
        d[e] = CopyItem{items[e].dst, c->hbufs[cm.x].image + (uint64_t)cm.y * cs, items[e].len, items[e].len};
      }
      // copy-engine drain: the same copies merged into runs where both sides
      // are contiguous (full chunks of one buffer: no padding between them)
      c->h_drun.ensure(3 * std::max<uint64_t>(n, 1));
      uint64_t* rs = c->h_drun.p;
      uint64_t* rd = rs + n;
      uint64_t* rl = rs + 2 * n;
      uint64_t r = 0;
      for (uint64_t e = 0; e < n; ++e) {
        if (r && rs[r - 1] + rl[r - 1] == d[e].src && rd[r - 1] + rl[r - 1] == d[e].dst && rl[r - 1] % 16 == 0) {
          rl[r - 1] += d[e].len;
        } else {
          rs[r] = d[e].src;
          rd[r] = d[e].dst;
          rl[r] = d[e].len;
          ++r;
        }
      }
      // compact the dst / len columns behind the first r entries
      if (r < n) {
        std::memmove(rs + r, rd, r * sizeof(uint64_t));
        std::memmove(rs + 2 * r, rl, r * sizeof(uint64_t));
      }
      c->drun_n = r;
    }
  }
  // The kernels write the entries and the payload; the header, the gap and
  // the work / item lists go up now -- by SM loads from the mapped staging
  // buffer, not by the copy engine (which the host leg keeps busy).
  StageList sl{};
  sl.seg[sl.n++] = StageSeg{st, pack, kPackHeader};
  const uint64_t gap0 = kPackHeader + kPackEntry * n;
  if (payload_off > gap0) sl.seg[sl.n++] = StageSeg{nullptr, pack + gap0, payload_off - gap0};
  if (n) {
    c->d_delta_items.ensure(n);
    sl.seg[sl.n++] = StageSeg{st + kPackHeader, reinterpret_cast<uint8_t*>(c->d_work.p), work_bytes};
    sl.seg[sl.n++] = StageSeg{st + kPackHeader + work_bytes, reinterpret_cast<uint8_t*>(c->d_delta_items.p), item_bytes};
    if (drain_bytes) {
      c->d_drain_items.ensure(n);
      sl.seg[sl.n++] = StageSeg{st + kPackHeader + work_bytes + item_bytes,
                                reinterpret_cast<uint8_t*>(c->d_drain_items.p), drain_bytes};
    }
  }
  k_stage_in<<<8, 256, 0, s>>>(sl);
  check_launch("k_stage_in");
  ++c->launches;
  ck(cudaEventRecord(c->stage_free, s), "event");
  c->delta_ready = true;
  c->delta_version = c->dirty_version;
  c->delta_precopy = c->precopy_bytes;
  c->delta_n = n;
  c->delta_offset = offset;
  c->delta_total = total;
  c->delta_payload_off = payload_off;
  c->delta_aligned = aligned;
  c->delta_drain = c->image_ready;
}

static bool delta_current(const pos_ctx* c) {
  return c->delta_ready && c->delta_version == c->dirty_version && c->delta_precopy == c->precopy_bytes;
}

int pos_delta_prepare(pos_ctx* c, void* stream, uint64_t* pack_offset, uint64_t* pack_bytes) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    delta_prepare(c, S(stream));
    if (pack_offset) *pack_offset = c->delta_offset;
    if (pack_bytes) *pack_bytes = c->delta_total;
  });
}

int pos_delta_copy(pos_ctx* c, void* stream, uint64_t* pack_offset, uint64_t* pack_bytes) {
  return pos_delta_copy_ex(c, stream, -1, pack_offset, pack_bytes);
}

int pos_delta_copy_ex(pos_ctx* c, void* stream, int stw_end_slot, uint64_t* pack_offset,
                      uint64_t* pack_bytes) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (stw_end_slot >= (int)c->events.size()) fail(POS_E_INVALID_ARGUMENT, "bad event slot");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(stream);
    if (!delta_current(c)) delta_prepare(c, s);
    c->delta_ready = false;  // one launch per preparation
    c->drain_pending = c->delta_drain;
    c->drain_n = c->delta_drain ? c->delta_n : 0;
    const uint64_t n = c->delta_n, cs = c->cfg.chunk_size;
    // Stop-the-world part: a pure TMA bulk gather of the flagged buffers.
    c->timer_begin(kTimDelta, s);
    // (TMA and SIMT gathers both run ~3x slower while the copy engine drains: measured)
    if (n) launch_copy(c, c->d_delta_items.p, nullptr, n, c->delta_aligned, s);
    c->timer_end(kTimDelta, s);
    if (stw_end_slot >= 0) {
      ck(cudaEventRecord(c->events[stw_end_slot], s), "event");
      c->d_stamps.ensure(64);
      k_stamp<<<1, 1, 0, s>>>(c->d_stamps.p + stw_end_slot);  // device clock of the same point
      check_launch("k_stamp");
    }
    // After the stop: hash the gathered copy -> entry crcs + refreshed digests.
    if (n) {
      HashParams p{};
      p.bufs = c->d_bufs.p;
      p.chunk_map = c->d_chunk_map.p;
      p.n_items = n;
      p.chunk_size = cs;
      p.k_full = zeros_crc(cs);
      p.tables = c->crc.tables.p;
      p.xinv = c->crc.xinv.p;
      p.digest_cur = c->d_digest[c->cur].p;
      p.work = c->d_work.p;
      p.pack = c->cache.p + c->delta_offset;
      p.payload_off = c->delta_payload_off;
      set_segments(c, n, p);
      int grid = c->hash_grid(n * p.nseg);
      c->timer_begin(kTimDeltaHash, s);
      launch_hash<kModeCached>(grid, s, p);
      check_launch("k_hash_chunks<cached>");
      c->timer_end(kTimDeltaHash, s);
      ++c->launches;
    }
    if (pack_offset) *pack_offset = c->delta_offset;
    if (pack_bytes) *pack_bytes = c->delta_total;
  });
}

int pos_d2h_async(pos_ctx* c, void* host_dst, uint64_t offset, uint64_t bytes, uint64_t slice,
                  void* stream) {
  return guarded([&] {
    if (!c || (!host_dst && bytes)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (offset + bytes > c->cache_cap) fail(POS_E_INVALID_LOCATOR, "range outside the cache");
    if (slice == 0) slice = 8ull << 20;
    for (uint64_t o = 0; o < bytes; o += slice) {
      uint64_t n = std::min(slice, bytes - o);
      ck(cudaMemcpyAsync(static_cast<uint8_t*>(host_dst) + o, c->cache.p + offset + o, n,
                         cudaMemcpyDeviceToHost, S(stream)),
         "d2h");
    }
  });
}

int pos_cache_info(pos_ctx* c, uint64_t* dev_ptr, uint64_t* capacity) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (dev_ptr) *dev_ptr = (uint64_t)c->cache.p;
    if (capacity) *capacity = c->cache_cap;
  });
}

int pos_scatter(pos_ctx* c, uint64_t pack_dev, uint64_t pack_bytes, void* stream) {
  return guarded([&] {
    if (!c || !pack_dev) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t s = S(stream);
    if (pack_bytes < kPackHeader) fail(POS_E_CORRUPT_IMAGE, "pack shorter than its header");
    uint8_t hdr[kPackHeader];
    ck(cudaMemcpyAsync(hdr, (const void*)pack_dev, kPackHeader, cudaMemcpyDeviceToHost, s), "hdr");
    ck(cudaStreamSynchronize(s), "sync");
    uint32_t magic, n;
    uint64_t cs, payload_off, payload;
    std::memcpy(&magic, hdr, 4);
    std::memcpy(&cs, hdr + 8, 8);
    std::memcpy(&n, hdr + 16, 4);
    std::memcpy(&payload_off, hdr + 24, 8);
    std::memcpy(&payload, hdr + 32, 8);
    if (magic != kPackMagic) fail(POS_E_CORRUPT_IMAGE, "bad pack magic");
    if (cs != c->cfg.chunk_size) fail(POS_E_CORRUPT_IMAGE, "pack chunk_size differs from the context");
    if (kPackHeader + (uint64_t)kPackEntry * n > payload_off || payload_off + payload > pack_bytes)
      fail(POS_E_CORRUPT_IMAGE, "pack sections exceed its size");
    if (!n) return;
    c->d_items.ensure(std::max<uint64_t>(n, c->n_chunks));
    ck(cudaMemsetAsync(c->d_err.p, 0, 4, s), "memset");
    k_pack_items<<<(n + 255) / 256, 256, 0, s>>>((const uint8_t*)pack_dev, pack_bytes, c->d_bufs.p,
                                                (uint32_t)c->bufs.size(), c->cfg.chunk_size,
                                                c->d_items.p, c->d_err.p);
    check_launch("k_pack_items");
    ++c->launches;
    uint32_t err = 0;
    ck(cudaMemcpyAsync(c->h_scan.p, c->d_err.p, 4, cudaMemcpyDeviceToHost, s), "err");
    ck(cudaStreamSynchronize(s), "sync");
    std::memcpy(&err, c->h_scan.p, 4);
    if (err & 1) fail(POS_E_CORRUPT_IMAGE, "malformed pack entry");
    if (err & 2) fail(POS_E_INVALID_LOCATOR, "pack entry outside its buffer or unknown handle");
    // Bulk path needs 16-B aligned chunk starts and payloads (payloads are by
    // construction); the <16 B remainder is written byte-exact.
    bool aligned = c->cfg.chunk_size % 16 == 0 && payload_off % 16 == 0 && pack_dev % 16 == 0;
    for (const auto& b : c->bufs) aligned = aligned && (b.dev_ptr % 16 == 0);
    c->timer_begin(kTimScatter, s);  // the HBM-bound part (validation above is a host round trip)
    launch_copy(c, c->d_items.p, nullptr, n, aligned, s);
    c->timer_end(kTimScatter, s);
  });
}

// Host-side validation of a POSD pack against the registered buffers: the
// checks write_content makes before it copies (buffer.hpp:80) plus the
// pack's own section bounds.
static void validate_pack_host(const pos_ctx* c, const uint8_t* pack, uint64_t bytes) {
  if (bytes < kPackHeader) fail(POS_E_CORRUPT_IMAGE, "pack shorter than its header");
  uint32_t magic, n;
  uint64_t cs, payload_off, payload;
  std::memcpy(&magic, pack, 4);
  std::memcpy(&cs, pack + 8, 8);
  std::memcpy(&n, pack + 16, 4);
  std::memcpy(&payload_off, pack + 24, 8);
  std::memcpy(&payload, pack + 32, 8);
  if (magic != kPackMagic) fail(POS_E_CORRUPT_IMAGE, "bad pack magic");
  if (cs != c->cfg.chunk_size) fail(POS_E_CORRUPT_IMAGE, "pack chunk_size differs from the context");
  if (kPackHeader + (uint64_t)kPackEntry * n > payload_off || payload_off + payload > bytes)
    fail(POS_E_CORRUPT_IMAGE, "pack sections exceed its size");
  for (uint32_t e = 0; e < n; ++e) {
    const uint8_t* ent = pack + kPackHeader + (uint64_t)e * kPackEntry;
    uint64_t h, off;
    uint32_t ch, len;
    std::memcpy(&h, ent, 8);
    std::memcpy(&off, ent + 8, 8);
    std::memcpy(&ch, ent + 16, 4);
    std::memcpy(&len, ent + 20, 4);
    auto it = c->index_of.find(h);
    if (it == c->index_of.end()) fail(POS_E_INVALID_LOCATOR, "pack entry for unknown handle");
    if ((uint64_t)ch * cs + len > c->bufs[it->second].size || off + len > payload)
      fail(POS_E_INVALID_LOCATOR, "pack entry outside its buffer");
  }
}

int pos_restore_packs(pos_ctx* c, const uint8_t* const* packs, const uint64_t* sizes, uint32_t npacks,
                      void* h2d_stream, void* stream, uint64_t region) {
  return guarded([&] {
    if (!c || (npacks && (!packs || !sizes))) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    cudaStream_t hs = S(h2d_stream), s = S(stream);
    if (region == 0) region = c->cache_cap / 2;
    region = region / kPackAlign * kPackAlign;
    if (2 * region > c->cache_cap) fail(POS_E_INVALID_ARGUMENT, "two regions must fit the cache");
    for (uint32_t i = 0; i < npacks; ++i) {  // all-or-nothing: validate before writing
      if (sizes[i] > region) fail(POS_E_STAGING_EXHAUSTED, "pack larger than a cache region");
      validate_pack_host(c, packs[i], sizes[i]);
    }
    bool aligned = c->cfg.chunk_size % 16 == 0;
    for (const auto& b : c->bufs) aligned = aligned && (b.dev_ptr % 16 == 0);
    if (!c->ev_d2h[0]) {
      for (int k = 0; k < 2; ++k) {
        ck(cudaEventCreateWithFlags(&c->ev_d2h[k], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->ev_copied2[k], cudaEventDisableTiming), "event");
      }
    }
    c->h_land[0].ensure(std::min<uint64_t>(region, std::max<uint64_t>(1, *std::max_element(sizes, sizes + std::max<uint32_t>(npacks, 1)))));
    c->h_land[1].ensure(c->h_land[0].n);
    bool used[2] = {false, false};
    c->timer_begin(kTimScatter, s);
    for (uint32_t i = 0; i < npacks; ++i) {
      const uint32_t r = i & 1;
      uint8_t* dev = c->cache.p + (uint64_t)r * region;
      // region r / landing slot r are free once pack i-2's scatter finished
      cudaPointerAttributes at{};
      bool pinned = cudaPointerGetAttributes(&at, packs[i]) == cudaSuccess && at.type == cudaMemoryTypeHost;
      cudaGetLastError();
      if (used[r]) {
        if (!pinned) ck(cudaEventSynchronize(c->ev_copied2[r]), "scatter sync");  // landing slot reuse
        ck(cudaStreamWaitEvent(hs, c->ev_copied2[r], 0), "wait region");           // cache region reuse
      }
      const uint8_t* src = packs[i];
      if (!pinned) {  // stage through the pinned landing slot with the host's threads
        uint8_t* dst = c->h_land[r].p;
        const uint64_t n = sizes[i];
        unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        if (n < (8u << 20)) nt = 1;
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nt; ++t)
          pool.emplace_back([=] {
            uint64_t lo = n * t / nt, hi = n * (t + 1) / nt;
            std::memcpy(dst + lo, src + lo, hi - lo);
          });
        for (auto& th : pool) th.join();
        src = dst;
      }
      ck(cudaMemcpyAsync(dev, src, sizes[i], cudaMemcpyHostToDevice, hs), "h2d");
      ck(cudaEventRecord(c->ev_d2h[r], hs), "event");
      ck(cudaStreamWaitEvent(s, c->ev_d2h[r], 0), "wait h2d");
      uint32_t ne;
      std::memcpy(&ne, packs[i] + 16, 4);
      if (ne) {
        c->d_items.ensure(std::max<uint64_t>(ne, c->n_chunks));
        k_pack_items<<<(ne + 255) / 256, 256, 0, s>>>(dev, sizes[i], c->d_bufs.p, (uint32_t)c->bufs.size(),
                                                     c->cfg.chunk_size, c->d_items.p, c->d_err.p);
        check_launch("k_pack_items");
        ++c->launches;
        launch_copy(c, c->d_items.p, nullptr, ne, aligned, s);
      }
      ck(cudaEventRecord(c->ev_copied2[r], s), "event");
      used[r] = true;
    }
    c->timer_end(kTimScatter, s);
    ck(cudaStreamSynchronize(s), "sync");
  });
}

// ---- on-demand restore of a flat host image --------------------------------

static void loader_run(pos_ctx* c) {
  Loader& L = *c->loader;
  cudaSetDevice(L.device);
  uint64_t k = 0;  // slices issued
  for (;;) {
    uint32_t b;
    uint64_t off, n;
    {
      std::unique_lock<std::mutex> lk(L.mu);
      if (L.queue.empty() || L.failed) break;
      b = L.queue.front();
      off = L.issued[b];
      n = std::min<uint64_t>(L.slice, c->bufs[b].size - off);
      L.issued[b] = off + n;
    }
    // flow control: slice k reuses the ring event of slice k - kLoadWindow
    cudaEvent_t& ev = L.ring[k % Loader::kLoadWindow];
    cudaError_t e = cudaSuccess;
    if (k >= (uint64_t)Loader::kLoadWindow) e = cudaEventSynchronize(ev);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync((void*)(c->bufs[b].dev_ptr + off), L.src[b] + off, n, cudaMemcpyHostToDevice, L.stream);
    if (e == cudaSuccess) e = cudaEventRecord(ev, L.stream);
    ++k;
    std::lock_guard<std::mutex> lk(L.mu);
    if (e != cudaSuccess) {
      L.failed = true;
      L.error = cudaGetErrorString(e);
      L.cv.notify_all();
      break;
    }
    if (L.issued[b] == c->bufs[b].size) {  // last slice of b: its ready event
      cudaEventRecord(L.ready[b], L.stream);
      L.state[b] = 1;
      auto it = std::find(L.queue.begin(), L.queue.end(), b);
      if (it != L.queue.end()) L.queue.erase(it);
      L.cv.notify_all();
    }
  }
  std::lock_guard<std::mutex> lk(L.mu);
  L.running = false;
  L.cv.notify_all();
}

static void loader_finish(pos_ctx* c) {
  if (!c->loader) return;
  Loader* L = c->loader;
  if (L->th.joinable()) L->th.join();
  if (L->stream) cudaStreamSynchronize(L->stream);
  for (auto e : L->ready)
    if (e) cudaEventDestroy(e);
  for (auto e : L->ring)
    if (e) cudaEventDestroy(e);
  for (void* h : L->pinned_here) cudaHostUnregister(h);
  delete L;
  c->loader = nullptr;
}

int pos_restore_image_begin(pos_ctx* c, uint8_t* const* hosts, const uint64_t* sizes, uint32_t n,
                            const uint64_t* order, uint32_t norder, uint64_t slice_bytes, void* h2d_stream) {
  return guarded([&] {
    if (!c || (n && (!hosts || !sizes)) || (norder && !order)) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (n != c->bufs.size()) fail(POS_E_INVALID_ARGUMENT, "one image range per registered buffer");
    if (c->loader) fail(POS_E_BAD_STATE, "a restore is already running (pos_restore_image_wait)");
    ck(cudaSetDevice(c->cfg.device), "cudaSetDevice");
    auto* L = new Loader();
    c->loader = L;
    L->device = c->cfg.device;
    L->stream = S(h2d_stream);
    if (slice_bytes) L->slice = slice_bytes;
    L->issued.assign(n, 0);
    L->state.assign(n, 2);
    L->ready.assign(n, nullptr);
    L->src.assign(hosts, hosts + n);
    for (int i = 0; i < Loader::kLoadWindow; ++i)
      ck(cudaEventCreateWithFlags(&L->ring[i], cudaEventDisableTiming), "event");
    for (uint32_t i = 0; i < n; ++i) {
      if (!hosts[i] || sizes[i] != c->bufs[i].size)
        fail(POS_E_INVALID_ARGUMENT, "image range " + std::to_string(i) + " does not match its buffer");
      cudaPointerAttributes a{};
      cudaError_t e = cudaPointerGetAttributes(&a, hosts[i]);
      if (e != cudaSuccess) cudaGetLastError();
      if (e != cudaSuccess || a.type != cudaMemoryTypeHost) {
        ck(cudaHostRegister(hosts[i], sizes[i], cudaHostRegisterPortable), "cudaHostRegister(restore image)");
        L->pinned_here.push_back(hosts[i]);
      }
      ck(cudaEventCreateWithFlags(&L->ready[i], cudaEventDisableTiming), "event");
    }
    // load order: `order` first (topo_order_buffers, dag.hpp:141-202), then
    // the rest by handle; unknown handles in `order` are ignored
    std::vector<uint8_t> seen(n, 0);
    for (uint32_t j = 0; j < norder; ++j) {
      auto it = c->index_of.find(order[j]);
      if (it == c->index_of.end() || seen[it->second]) continue;
      seen[it->second] = 1;
      L->queue.push_back(it->second);
      L->state[it->second] = 0;
    }
    for (uint32_t i = 0; i < n; ++i)
      if (!seen[i]) {
        L->queue.push_back(i);
        L->state[i] = 0;
      }
    L->running = true;
    L->th = std::thread(loader_run, c);
  });
}

// bump_front (engines.hpp:86-93): the buffer's remaining slices go next.
static uint32_t loader_want(pos_ctx* c, uint64_t handle) {
  Loader& L = *c->loader;
  auto it = c->index_of.find(handle);
  if (it == c->index_of.end()) fail(POS_E_INVALID_LOCATOR, "unknown handle");
  const uint32_t b = it->second;
  std::lock_guard<std::mutex> lk(L.mu);
  if (L.state[b] == 0) {
    auto q = std::find(L.queue.begin(), L.queue.end(), b);
    if (q != L.queue.end() && q != L.queue.begin()) {
      L.queue.erase(q);
      L.queue.push_front(b);
    }
  }
  return b;
}

int pos_restore_want(pos_ctx* c, uint64_t handle) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->loader) fail(POS_E_BAD_STATE, "no restore running");
    loader_want(c, handle);
  });
}

int pos_restore_gate(pos_ctx* c, uint64_t handle, void* stream) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->loader) return;  // nothing being restored: every buffer is ready
    const uint32_t b = loader_want(c, handle);
    Loader& L = *c->loader;
    std::unique_lock<std::mutex> lk(L.mu);
    // host waits only until the last slice is ISSUED; the device waits for it to land
    L.cv.wait(lk, [&] { return L.state[b] != 0 || L.failed; });
    if (L.failed) fail(POS_E_CUDA, "restore loader: " + L.error);
    ck(cudaStreamWaitEvent(S(stream), L.ready[b], 0), "gate wait");
  });
}

int pos_restore_ready(pos_ctx* c, uint64_t handle, int* ready) {
  return guarded([&] {
    if (!c || !ready) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->loader) {
      *ready = 1;
      return;
    }
    auto it = c->index_of.find(handle);
    if (it == c->index_of.end()) fail(POS_E_INVALID_LOCATOR, "unknown handle");
    Loader& L = *c->loader;
    std::lock_guard<std::mutex> lk(L.mu);
    *ready = L.state[it->second] == 1 && cudaEventQuery(L.ready[it->second]) == cudaSuccess;
    cudaGetLastError();
  });
}

int pos_restore_image_wait(pos_ctx* c) {
  return guarded([&] {
    if (!c) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!c->loader) return;
    std::string err;
    {
      Loader& L = *c->loader;
      if (L.th.joinable()) L.th.join();
      if (L.failed) err = L.error;
    }
    loader_finish(c);
    if (!err.empty()) fail(POS_E_CUDA, "restore loader: " + err);
  });
}

static int crc_range(uint32_t* out, uint64_t ptr, uint64_t n, cudaStream_t s) {
  return guarded([&] {
    if (!out) fail(POS_E_INVALID_ARGUMENT, "null argument");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    int cnt = 0;
    if (e != cudaSuccess || cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0)
      fail(POS_E_NO_DEVICE, "no CUDA device: the dump path has no CPU fallback");
    if (n == 0) {
      *out = 0;
      return;
    }
    if (!ptr) fail(POS_E_INVALID_ARGUMENT, "null device pointer");
    CrcTables& t = engine_for_current_device();
    // One virtual buffer of 64 KiB chunks, digests folded by k_buffer_crc.
    const uint64_t cs = 65536;
    uint64_t nc = (n + cs - 1) / cs;
    DevBuf b{};
    b.ptr = ptr;
    b.size = n;
    b.handle = 1;
    b.nchunks = (uint32_t)nc;
    uint64_t tail = n - (nc - 1) * cs;
    b.k_tail = zeros_crc(tail);
    b.x8_tail = x8nmodp(tail);
    std::vector<uint2> cmap(nc);
    for (uint64_t k = 0; k < nc; ++k) cmap[k] = make_uint2(0, (uint32_t)k);
    std::vector<uint32_t> tcs(1024);
    build_advance_table(cs, tcs.data());
    DevArray<DevBuf> db;
    DevArray<uint2> dm;
    DevArray<uint32_t> dd, dt, dc;
    DevArray<uint8_t> dz;
    db.ensure(1);
    dm.ensure(nc);
    dd.ensure(nc);
    dt.ensure(1024);
    dc.ensure(2);  // [crc out, xfold]
    dz.ensure(2);
    auto cleanup = [&] {
      db.release();
      dm.release();
      dd.release();
      dt.release();
      dc.release();
      dz.release();
    };
    try {
      ck(cudaMemcpyAsync(db.p, &b, sizeof b, cudaMemcpyHostToDevice, s), "h2d");
      ck(cudaMemcpyAsync(dm.p, cmap.data(), nc * 8, cudaMemcpyHostToDevice, s), "h2d");
      ck(cudaMemcpyAsync(dt.p, tcs.data(), 4096, cudaMemcpyHostToDevice, s), "h2d");
      ck(cudaMemsetAsync(dz.p, 0, 2, s), "memset");
      static thread_local uint32_t xf;  // pageable source: cudaMemcpyAsync stages it before returning
      xf = x8nmodp(cs * ((nc - 1 + 31) / 32));
      ck(cudaMemcpyAsync(dc.p + 1, &xf, 4, cudaMemcpyHostToDevice, s), "h2d");
      HashParams p{};
      p.bufs = db.p;
      p.chunk_map = dm.p;
      p.n_items = nc;
      p.chunk_size = cs;
      p.k_full = zeros_crc(cs);
      p.tables = t.tables.p;
      p.xinv = t.xinv.p;
      p.digest_cur = dd.p;
      p.digest_prev = dd.p;
      p.flags = nullptr;  // digests only
      p.bitmap = nullptr;
      p.nseg = 1;
      p.seg_bytes = (uint32_t)cs;
      uint64_t blocks = (nc + 15) / 16;
      int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)t.sm_count));
      launch_hash<kModeHash>(grid, s, p);
      check_launch("k_hash_chunks");
      k_buffer_crc<<<1, 32, 0, s>>>(db.p, 1, dd.p, dt.p, dc.p + 1, dz.p, 0, 1, dc.p, dz.p + 1);
      check_launch("k_buffer_crc");
      uint32_t r = 0;
      ck(cudaMemcpyAsync(&r, dc.p, 4, cudaMemcpyDeviceToHost, s), "d2h");
      ck(cudaStreamSynchronize(s), "sync");
      *out = r;
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

int pos_crc32(uint64_t dev_ptr, uint64_t n, uint32_t* out, void* stream) {
  return crc_range(out, dev_ptr, n, S(stream));
}

int pos_crc32_update(uint32_t crc, uint64_t dev_ptr, uint64_t n, uint32_t* out, void* stream) {
  uint32_t part = 0;
  int rc = crc_range(&part, dev_ptr, n, S(stream));
  if (rc != POS_OK) return rc;
  if (!out) return POS_E_INVALID_ARGUMENT;
  *out = crc32_combine(crc, part, n);  // crc32_update continues a final CRC (crc32.hpp:26-32)
  return POS_OK;
}

int pos_fill(uint64_t dev_ptr, uint64_t n, uint64_t seed, void* stream) {
  uint64_t r[3] = {dev_ptr, n, seed};
  return pos_fill_batch(r, 1, stream);
}

int pos_fill_batch(const uint64_t* ranges, uint32_t count, void* stream) {
  return guarded([&] {
    if (!ranges && count) fail(POS_E_INVALID_ARGUMENT, "null argument");
    int cnt = 0;
    if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0)
      fail(POS_E_NO_DEVICE, "no CUDA device");
    cudaStream_t s = S(stream);
    // Ranges travel by value in the kernel parameters: fully asynchronous.
    for (uint32_t base = 0; base < count; base += kFillMaxRanges) {
      FillBatch b{};
      b.count = std::min<uint32_t>(kFillMaxRanges, count - base);
      uint64_t maxn = 0;
      for (uint32_t i = 0; i < b.count; ++i) {
        const uint64_t* r = ranges + 3 * (uint64_t)(base + i);
        b.r[i] = FillRange{r[0], r[1], r[2]};
        maxn = std::max(maxn, r[1]);
      }
      uint64_t pairs = (maxn + 15) / 16;
      dim3 grid((unsigned)std::max<uint64_t>(1, std::min<uint64_t>((pairs + 255) / 256, 1184)), b.count);
      k_fill<<<grid, 256, 0, s>>>(b);
      check_launch("k_fill");
    }
  });
}

int pos_event_record(pos_ctx* c, uint32_t slot, void* stream) {
  return guarded([&] {
    if (!c || slot >= c->events.size()) fail(POS_E_INVALID_ARGUMENT, "bad event slot");
    ck(cudaEventRecord(c->events[slot], S(stream)), "event record");
  });
}

int pos_stamp(pos_ctx* c, uint32_t slot, void* stream) {
  return guarded([&] {
    if (!c || slot >= 64) fail(POS_E_INVALID_ARGUMENT, "bad stamp slot");
    c->d_stamps.ensure(64);
    k_stamp<<<1, 1, 0, S(stream)>>>(c->d_stamps.p + slot);
    check_launch("k_stamp");
  });
}

int pos_stamp_elapsed(pos_ctx* c, uint32_t a, uint32_t b, float* ms) {
  return guarded([&] {
    if (!c || !ms || a >= 64 || b >= 64) fail(POS_E_INVALID_ARGUMENT, "bad stamp slot");
    if (!c->d_stamps.p) fail(POS_E_BAD_STATE, "no stamps");
    ck(cudaDeviceSynchronize(), "sync");
    unsigned long long t[64];
    ck(cudaMemcpy(t, c->d_stamps.p, sizeof t, cudaMemcpyDeviceToHost), "stamps");
    *ms = (float)((double)((long long)(t[b] - t[a])) * 1e-6);
  });
}

int pos_event_elapsed(pos_ctx* c, uint32_t a, uint32_t b, float* ms) {
  return guarded([&] {
    if (!c || !ms || a >= c->events.size() || b >= c->events.size())
      fail(POS_E_INVALID_ARGUMENT, "bad event slot");
    ck(cudaEventSynchronize(c->events[b]), "event sync");
    ck(cudaEventElapsedTime(ms, c->events[a], c->events[b]), "elapsed");
  });
}

int pos_stream_wait_event(pos_ctx* c, uint32_t slot, void* stream) {
  return guarded([&] {
    if (!c || slot >= c->events.size()) fail(POS_E_INVALID_ARGUMENT, "bad event slot");
    ck(cudaStreamWaitEvent(S(stream), c->events[slot], 0), "stream wait event");
  });
}

int pos_timeline(pos_ctx* c, uint32_t slot, float* out) {
  return guarded([&] {
    if (!c || !out || slot >= c->events.size()) fail(POS_E_INVALID_ARGUMENT, "bad argument");
    for (int t = 0; t < 7; ++t) {
      out[2 * t] = out[2 * t + 1] = -1.f;
      if (!c->timers[t].used) continue;
      ck(cudaEventSynchronize(c->timers[t].b), "event sync");
      ck(cudaEventElapsedTime(&out[2 * t], c->events[slot], c->timers[t].a), "elapsed");
      ck(cudaEventElapsedTime(&out[2 * t + 1], c->events[slot], c->timers[t].b), "elapsed");
    }
  });
}

int pos_launch_count(pos_ctx* c, uint64_t* out) {
  return guarded([&] {
    if (!c || !out) fail(POS_E_INVALID_ARGUMENT, "null argument");
    *out = c->launches;
  });
}

int pos_last_kernel_ms(pos_ctx* c, const char* which, float* ms) {
  return guarded([&] {
    if (!c || !which || !ms) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (!std::strcmp(which, "hash_waves")) {  // sum of the last pipelined pre-copy's hash kernels
      if (!c->waves_last) fail(POS_E_BAD_STATE, "no pipelined pre-copy recorded");
      float total = 0;
      for (uint32_t w = 0; w < c->waves_last; ++w) {
        float m = 0;
        ck(cudaEventSynchronize(c->wave_hash[w][1]), "event sync");
        ck(cudaEventElapsedTime(&m, c->wave_hash[w][0], c->wave_hash[w][1]), "elapsed");
        total += m;
      }
      *ms = total;
      return;
    }
    for (int t = 0; t < kTimCount; ++t) {
      if (std::strcmp(which, kTimerNames[t]) != 0) continue;
      if (!c->timers[t].used) fail(POS_E_BAD_STATE, "no launch recorded");
      ck(cudaEventSynchronize(c->timers[t].b), "event sync");
      ck(cudaEventElapsedTime(ms, c->timers[t].a, c->timers[t].b), "elapsed");
      return;
    }
    fail(POS_E_INVALID_ARGUMENT, "unknown timer");
  });
}

// Copy out of a DMA landing buffer, then evict the source lines from the CPU
// caches: the next D2H into lines the CPU still holds runs ~40% slower
// (measured on the B200 host: 91.5 GB/s state rate without the host apply,
// 46.6 with it and a single landing buffer).
static void copy_evict(uint8_t* dst, const uint8_t* src, uint64_t len) {
  std::memcpy(dst, src, len);
  static const bool evict = [] {
    const char* e = std::getenv("POSDUMP_NO_EVICT");
    return !(e && *e == '1') && __builtin_cpu_supports("clflushopt");
  }();
  if (!evict) return;
  const uintptr_t lo = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(63);
  const uintptr_t hi = reinterpret_cast<uintptr_t>(src) + len;
  for (uintptr_t p = lo; p < hi; p += 64) __builtin_ia32_clflushopt(reinterpret_cast<void*>(p));
}

int pos_pack_apply_host(const uint8_t* pack, uint64_t pack_bytes, const uint64_t* handles,
                        uint8_t* const* hosts, const uint64_t* sizes, uint32_t nb, uint32_t threads) {
  return guarded([&] {
    if (!pack || (nb && (!handles || !hosts || !sizes))) fail(POS_E_INVALID_ARGUMENT, "null argument");
    if (pack_bytes < kPackHeader) fail(POS_E_CORRUPT_IMAGE, "pack shorter than its header");
    uint32_t magic, n;
    uint64_t cs, payload_off, payload;
    std::memcpy(&magic, pack, 4);
    std::memcpy(&cs, pack + 8, 8);
    std::memcpy(&n, pack + 16, 4);
    std::memcpy(&payload_off, pack + 24, 8);
    std::memcpy(&payload, pack + 32, 8);
    if (magic != kPackMagic) fail(POS_E_CORRUPT_IMAGE, "bad pack magic");
    if (kPackHeader + (uint64_t)kPackEntry * n > payload_off || payload_off + payload > pack_bytes)
      fail(POS_E_CORRUPT_IMAGE, "pack sections exceed its size");
    // Resolve + validate every entry before writing anything (write_content
    // checks before it copies, buffer.hpp:80).
    struct Op { uint8_t* dst; const uint8_t* src; uint64_t len; };
    std::vector<Op> ops(n);
    for (uint32_t e = 0; e < n; ++e) {
      const uint8_t* ent = pack + kPackHeader + (uint64_t)e * kPackEntry;
      uint64_t h, off;
      uint32_t c, len;
      std::memcpy(&h, ent, 8);
      std::memcpy(&off, ent + 8, 8);
      std::memcpy(&c, ent + 16, 4);
      std::memcpy(&len, ent + 20, 4);
      const uint64_t* it = std::lower_bound(handles, handles + nb, h);
      if (it == handles + nb || *it != h) fail(POS_E_INVALID_LOCATOR, "pack entry for unknown handle");
      uint32_t b = (uint32_t)(it - handles);
      if ((uint64_t)c * cs + len > sizes[b] || off + len > payload)
        fail(POS_E_INVALID_LOCATOR, "pack entry outside its buffer");
      ops[e] = Op{hosts[b] + (uint64_t)c * cs, pack + payload_off + off, len};
    }
    uint32_t nt = std::max<uint32_t>(1, std::min<uint32_t>(threads, 64));
    if (nt == 1 || n < 2 * nt) {
      for (const Op& o : ops) copy_evict(o.dst, o.src, o.len);
      return;
    }
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (uint32_t e = t; e < n; e += nt) copy_evict(ops[e].dst, ops[e].src, ops[e].len);
      });
    for (auto& th : pool) th.join();
  });
}

int pos_image_write(const pos_image_desc* img, uint8_t* out, uint64_t cap, uint64_t* size) {
  return guarded([&] {
    if (!img || !size) fail(POS_E_INVALID_ARGUMENT, "null argument");
    std::string err;
    int rc = write_posi_image(*img, out, cap, size, &err);
    if (rc != POS_OK) fail(rc, err);
  });
}

// ---- plumbing ----------------------------------------------------------

int pos_device_count(int* n) {
  return guarded([&] {
    if (!n) fail(POS_E_INVALID_ARGUMENT, "null argument");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
    cudaGetLastError();
    *n = c;
  });
}

int pos_set_device(int device) {
  return guarded([&] { require_device(device); });
}

int pos_dev_malloc(uint64_t bytes, uint64_t* dev_ptr) {
  return guarded([&] {
    if (!dev_ptr) fail(POS_E_INVALID_ARGUMENT, "null argument");
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<uint64_t>(bytes, 1));
    if (e != cudaSuccess)
      fail(e == cudaErrorMemoryAllocation ? POS_E_OUT_OF_DEVICE_MEMORY : POS_E_CUDA,
           std::string("cudaMalloc: ") + cudaGetErrorString(e));
    *dev_ptr = (uint64_t)p;
  });
}

int pos_dev_free(uint64_t dev_ptr) {
  return guarded([&] { ck(cudaFree((void*)dev_ptr), "cudaFree"); });
}

int pos_host_malloc_pinned(uint64_t bytes, void** host) {
  return guarded([&] {
    if (!host) fail(POS_E_INVALID_ARGUMENT, "null argument");
    ck(cudaHostAlloc(host, std::max<uint64_t>(bytes, 1), cudaHostAllocDefault), "cudaHostAlloc");
  });
}

int pos_host_free_pinned(void* host) {
  return guarded([&] { ck(cudaFreeHost(host), "cudaFreeHost"); });
}

int pos_memcpy(uint64_t dst, uint64_t src, uint64_t bytes, int kind, void* stream) {
  return guarded([&] {
    if (kind < 1 || kind > 3) fail(POS_E_INVALID_ARGUMENT, "bad memcpy kind");
    if (!bytes) return;
    ck(cudaMemcpyAsync((void*)dst, (const void*)src, bytes, (cudaMemcpyKind)kind, S(stream)),
       "cudaMemcpyAsync");
  });
}

int pos_memset(uint64_t dev_ptr, int value, uint64_t bytes, void* stream) {
  return guarded([&] {
    if (!bytes) return;
    ck(cudaMemsetAsync((void*)dev_ptr, value, bytes, S(stream)), "cudaMemsetAsync");
  });
}

int pos_stream_create(void** stream) {
  return guarded([&] {
    if (!stream) fail(POS_E_INVALID_ARGUMENT, "null argument");
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    *stream = s;
  });
}

int pos_stream_create_prio(int priority, void** stream) {
  return guarded([&] {
    if (!stream) fail(POS_E_INVALID_ARGUMENT, "null argument");
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    cudaStream_t s;
    ck(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority ? hi : lo), "cudaStreamCreate");
    *stream = s;
  });
}

int pos_stream_destroy(void* stream) {
  return guarded([&] { ck(cudaStreamDestroy(S(stream)), "cudaStreamDestroy"); });
}

int pos_stream_sync(void* stream) {
  return guarded([&] { ck(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize"); });
}

int pos_device_sync(void) {
  return guarded([&] { ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); });
}

int pos_stream_wait(void* waiter, void* signaller) {
  return guarded([&] {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(e, S(signaller)), "event record");
    ck(cudaStreamWaitEvent(S(waiter), e, 0), "stream wait");
    cudaEventDestroy(e);
  });
}

}  // extern "C"
