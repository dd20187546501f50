// posdump.cu -- host side of libposdump.so: the C ABI of include/posdump.h.
//
// Owns device memory for the buffer table, the per-chunk digest tables
// (double-buffered by epoch), the dirty flags/bitmap, the O3 cache and the
// launch plumbing.  There is no CPU path: every operation on buffer bytes is
// a kernel from kernels.cuh, and a missing device is an error.
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <system_error>
#include <stdexcept>
#include <thread>
#include <vector>

#include "../../include/posdump.h"
#include "crc_math.h"
#include "kernels.cuh"
#include "image_writer.h"
#include "image_reader.h"
#include "host_crc.h"

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
  } catch (const std::system_error& e) {  // std::thread / mutex
    g_last_error = std::string("system error: ") + e.what();
    return POS_E_BAD_STATE;
  } catch (const std::exception& e) {  // out_of_range, length_error, ...
    g_last_error = std::string("internal error: ") + e.what();
    return POS_E_INVARIANT_VIOLATION;
  } catch (...) {  // nothing crosses the C ABI
    g_last_error = "unknown exception";
    return POS_E_INVARIANT_VIOLATION;
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

// Large pinned host buffers (GB-sized landing slots): huge pages + cudaHostRegister
// through pos_host_image_alloc -- ~10x faster to set up than cudaHostAlloc.
struct HugePinned {
  uint8_t* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n && p) return;
    release();
    void* m = nullptr;
    const int rc = pos_host_image_alloc(std::max<size_t>(count, 1), 8, &m);
    if (rc != POS_OK) fail(rc, "pinned landing slot: " + g_last_error);
    p = static_cast<uint8_t*>(m);
    n = std::max<size_t>(count, 1);
  }
  void release() {
    if (p) pos_host_image_free(p);
    p = nullptr;
    n = 0;
  }
};

template <int MODE>
void launch_hash(int grid, cudaStream_t s, const HashParams& p) {
  if (MODE == kModeHash && p.digest2_cur)
    k_hash_chunks<kModeHash, true><<<grid, kHashThreads, kHashSmem, s>>>(p);
  else
    k_hash_chunks<MODE><<<grid, kHashThreads, kHashSmem, s>>>(p);
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
    ck(cudaStreamSynchronize(cudaStreamLegacy), "upload sync");
    ck(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device), "sm count");
    ck(cudaFuncSetAttribute(k_hash_chunks<kModeHash>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem),
       "smem attr");
    ck(cudaFuncSetAttribute(k_hash_chunks<kModeCopy>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem),
       "smem attr");
    ck(cudaFuncSetAttribute(k_hash_chunks<kModeCached>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem),
       "smem attr");
    ck(cudaFuncSetAttribute(k_hash_chunks<kModeHash, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kHashSmem),
       "smem attr");
    ck(cudaFuncSetAttribute(k_copy_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, kCopySmem),
       "smem attr");
    ck(cudaFuncSetAttribute(k_ship_runs, cudaFuncAttributeMaxDynamicSharedMemorySize, kShipSmem), "smem attr");
    // Load every kernel now: under lazy module loading (the CUDA 12 default)
    // a kernel's first launch loads it, and the load waits for the device --
    // a first launch would serialise behind the copy engine's host leg.  The
    // scan asks for the hash kernel's maximal-shared carveout: an SM's
    // L1/shared split only changes while it is idle, and a scan CTA on an SM
    // with the default split would keep the next wave's hash CTA off it.
    ck(cudaFuncSetAttribute(k_pack_scan, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared),
       "carveout");
    ck(cudaFuncSetAttribute(k_scan_tiles, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared),
       "carveout");
    cudaFuncAttributes fa;
    ck(cudaFuncGetAttributes(&fa, k_pack_scan), "load k_pack_scan");
    ck(cudaFuncGetAttributes(&fa, k_scan_tiles), "load k_scan_tiles");
    ck(cudaFuncGetAttributes(&fa, k_copy_simt), "load k_copy_simt");
    ck(cudaFuncGetAttributes(&fa, k_pack_items), "load k_pack_items");
    ck(cudaFuncGetAttributes(&fa, k_buffer_crc), "load k_buffer_crc");
    ck(cudaFuncGetAttributes(&fa, k_note_upstream), "load k_note_upstream");
    ck(cudaFuncGetAttributes(&fa, k_clear_written), "load k_clear_written");
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
  // 0 queued, 1 loaded (ready event recorded), 2 not part of the image,
  // 3 Recompute: waits for its replayed writer, 4 Recompute replayed (ready event recorded)
  std::vector<uint8_t> state;
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

// Host leg of the direct pre-copy (CopyEngine, engines.hpp:28-167): a feeder
// thread moves each wave's runs to the copy engine as slices of at most
// `slice` bytes with at most `window` slices in flight, so an application
// copy issued meanwhile (pos_app_copy) waits behind at most window x slice
// bytes of checkpoint traffic and the next slices wait for it -- app over
// ckpt at slice granularity (engines.hpp:153-159).  Measured without it: an
// application D2H of 16 MiB issued during a 7.5 GB pre-copy took 117 ms
// instead of 0.3 ms (tools/probe_app_copy.py).
struct HostLeg {
  static constexpr int kMaxWindow = 8;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  bool quit = false;
  bool pending = false;               // a job was handed over and is not finished
  uint32_t waves = 0;
  cudaStream_t ds = nullptr;
  cudaEvent_t ring[kMaxWindow] = {};
  cudaEvent_t done_ev = nullptr;      // on ds after the job's last slice
  bool done_ev_valid = false;         // recorded by the last finished job of this epoch
  std::deque<cudaEvent_t> app;        // application copies in flight (the feeder yields to them)
  uint64_t slice = 16ull << 20;
  int window = 3;
  uint64_t slices = 0, app_yields = 0, cancelled_bytes = 0;
  PinnedArray<uint64_t> ship;                 // [kMaxWindow][4][kShipMaxRuns]: a slot's short-run batch
  std::atomic<uint64_t> ship_launches{0};     // k_ship_runs launched by the feeder
  std::atomic<bool> shipped_last{false};      // the last job launched k_ship_runs
  cudaStream_t s2 = nullptr;                  // second stream for k_ship_runs batches
  int s2_prio = 0;
  cudaEvent_t join_ev = nullptr;              // ds -> s2 at the start, s2 -> ds at the end
  int error_code = 0;
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
  HostLeg* leg = nullptr;
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
  // the optional second digest of the O2 compare (pos_set_o2_digest2), same
  // double buffering as d_digest; d2_valid: the previous table is complete
  DevArray<uint32_t> d_digest2[2];
  bool digest2 = false, d2_valid = false, d2_ran = false;
  int cur = 0;
  bool prev_valid = false;
  bool fresh_target = false;  // CheckpointTarget::fresh (cr.hpp:35): this round ships every chunk
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
  int delta_slots[2] = {-1, -1};  // pos_final_stop: the STW window's events (the delta timer)
  DevArray<uint64_t> d_result;  // async pre-copy: [n, total, overflow, n_items]
  std::set<uint64_t> dirty_set;
  // record_dirty during a direct pre-copy cancels the buffer's copies still
  // to be submitted (CopyEngine::cancel, cr.hpp:909-918; engines.hpp:80-85):
  // set by the caller's thread, read by the host leg's feeder.
  std::unique_ptr<std::atomic<uint8_t>[]> cancelled;
  std::set<uint64_t> stop_excluded;  // at_final_stop's exclusions (pos_set_stop_exclusions)
  pos_metrics metrics{};             // CrMetrics of the session (final stop + finalize)
  bool dag_uploaded = false;
  uint64_t dirty_version = 0;
  // STW delta staged ahead of the stop (pos_delta_prepare)
  bool delta_ready = false;
  uint64_t delta_version = 0, delta_precopy = 0, delta_n = 0, delta_offset = 0, delta_total = 0,
           delta_payload_off = 0;
  bool delta_aligned = true;
  bool delta_drain = false;  // drain items staged with the delta
  bool drain_short = false;  // ... some of them shorter than kCeRun (k_ship_runs)
  DevArray<CopyItem> d_delta_items;
  // eager delta capture (pos_delta_pregather): per buffer index, the delta
  // pack's items [first, first + count) and whether they were gathered
  // after the buffer's last writer, ahead of the stop
  std::vector<uint2> delta_items_of;
  std::vector<uint8_t> pregathered;
  cudaEvent_t ev_pregather = nullptr;
  // host image (pos_register_image): device-visible address per buffer, and
  // the host ranges this context pinned itself (unpinned at destroy)
  bool image_ready = false;
  std::vector<void*> image_pinned;
  bool drain_pending = false;        // a STW delta awaits pos_delta_drain
  bool direct_pending = false;       // a pos_precopy_direct awaits pos_precopy_direct_result
  bool direct_epoch = false;         // this epoch ran a direct pre-copy (the final stop follows its host leg)
  // copy-engine host leg of the direct mode: run lists written by the scan
  // into mapped pinned memory = the host leg's copy list
  PinnedArray<uint64_t> h_run;   // [3][n_chunks]: src, dst, bytes
  PinnedArray<uint64_t> h_drun;  // STW delta drain runs, same layout
  PinnedArray<uint64_t> h_dship; // the drain's short-run batches (k_ship_runs)
  cudaEvent_t dship_done = nullptr;
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
  cudaEvent_t gathered = nullptr;  // the STW gather landed (the delta drain waits on it, not on the post-stop hash)
  cudaEvent_t ev_dag = nullptr;  // DAG flags uploaded on a side stream
  bool dag_side = false;
  // Pre-copy packs: one per wave, chained at a device-side cache cursor.
  static constexpr uint32_t kMaxWaves = 16;
  DevArray<uint64_t> d_cursor;                     // [1]
  cudaEvent_t scanned[kMaxWaves] = {};
  cudaEvent_t copied[kMaxWaves] = {};
  cudaEvent_t wave_hash[kMaxWaves][2] = {};
  uint32_t waves_last = 0;                          // waves of the last pre-copy (hash timing)
  bool wave_used[kMaxWaves] = {};                   // wave_hash slot holds a launch of this pre-copy
  float hash_acc_ms = 0;                            // hash time of slots reused within the pre-copy
  uint64_t scan_seq = 0, slot_seq[kMaxWaves] = {};  // host-mirror sequence numbers
  // cache-cycled pre-copy (pos_precopy_stream): 2 cache regions, 2 pinned landing slots
  HugePinned h_land[2];  // landing slots of the cache-cycled pre-copy / streaming restore
  uint8_t* h_bounce = nullptr;                // pos_image_restore from pageable bytes: 2 slots
                                              // (pos_host_image_alloc)
  cudaEvent_t ev_bounce[2] = {nullptr, nullptr};
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
  // (Measured, config-5 step, tools/ in profiles/r2/app_interference.txt:
  // short-lived hash CTAs of 64 chunks with the application at the higher
  // stream priority cut the window's slowdown from 11.8x to 4.8x at 0.82 of
  // HBM; an SM budget of 18 cuts it to 1.28x at the same dump rate.)
  int hash_grid(uint64_t items) const {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(items, (uint64_t)hash_sm_budget()));
  }
  // SMs the dump's hash may occupy (pos_set_hash_sms; 0 = all): the
  // ChecksumEngine's budget (checksum_bw, config.hpp:20-23) -- every hash CTA
  // holds its SM's shared memory for its wave (the application's CTAs
  // co-reside in the registers it leaves), the rest of the SMs are theirs.
  uint32_t hash_sms = 0;
  int hash_sm_budget() const {
    return hash_sms && (int)hash_sms < crc.sm_count ? (int)hash_sms : crc.sm_count;
  }
};

namespace {

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(POS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// Host-side setup writes device tables with cudaMemcpy / cudaMemset on the
// legacy stream, which does NOT order with the library's non-blocking
// streams: cudaMemset and pageable cudaMemcpy may return before the device
// write lands.  Every setup path ends here, before any kernel can read them
// (measured: a tile-status memset that landed after the scan launched
// deadlocked its look-back while application kernels kept the GPU busy).
void upload_barrier() { ck(cudaStreamSynchronize(cudaStreamLegacy), "upload sync"); }

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

// TMA bulk copies when every item is 16-B aligned (measured: a SIMT 16-B
// vector copy was no faster alone and ~3x slower beside a copy-engine D2H),
// else the SIMT vector/byte copy.
void launch_copy(pos_ctx* c, const CopyItem* items, const uint64_t* n_dev, uint64_t n_host,
                 bool aligned, cudaStream_t s, uint64_t max_item_bytes = 0) {
  int sms = c->crc.sm_count;
  if (aligned) {
    // 3 CTAs/SM fit in smem (64 KiB ring each); one elected thread per CTA.
    // A host-known list of items no longer than max_item_bytes is spread
    // over the grid piece by piece (more CTAs than items).
    int grid = sms * 3;
    uint32_t ppi = 0;
    if (!n_dev && max_item_bytes) {
      ppi = (uint32_t)std::max<uint64_t>(1, (max_item_bytes + kCopyPiece - 1) / kCopyPiece);
      grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(grid, n_host * ppi));
    } else if (!n_dev) {
      grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(grid, n_host));
    }
    k_copy_bulk<<<grid, 32, kCopySmem, s>>>(items, n_dev, n_host, ppi);
  } else {
    k_copy_simt<<<sms * 4, 256, 0, s>>>(items, n_dev, n_host);
  }
  check_launch("copy");
  ++c->launches;
}

// Runs of at least kCeRun bytes go to the copy engine (>= 4 MiB: 54 GB/s,
// no cost to concurrent kernels); shorter ones are shipped by k_ship_runs.
constexpr uint64_t kCeRun = 4ull << 20;
// Pack D2H (pack / stream modes): copies of up to 64 MiB -- the copy engine
// pays ~4 us per copy (8 MiB slices: ~2.7 % of the link; 64 MiB: 0.35 %).
constexpr uint64_t kD2HSlice = 64ull << 20;

// One batch of short runs, SoA [4][n] {src, dst, bytes, exclusive prefix} in
// mapped pinned memory, stored into the host image by kShipCtas CTAs.
void launch_ship(const uint64_t* runs, uint32_t n, uint64_t total, cudaStream_t s) {
  k_ship_runs<<<kShipCtas, kShipThreads, 32 * n, s>>>(runs, n, total);
  check_launch("k_ship_runs");
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

// The C ABI, by area (one translation unit).
#include "context.inc"
#include "precopy.inc"
#include "hostleg.inc"
#include "delta.inc"
#include "restore.inc"
#include "util.inc"
#include "finalize.inc"
