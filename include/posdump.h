/*
 * posdump.h -- C ABI of the B200-native buffer-dump hot path of the POS
 * checkpoint engine (libposdump.so).
 *
 * The reference (gpucrsim, /root/reference/proj) is a header-only C++20
 * library with no FFI; its hot path is a set of CrEngine member functions.
 * Each entry point below names the reference function it replaces
 * (path:line relative to /root/reference/proj).  INTEGRATION.md shows the
 * call site a maintainer would change and the ctypes / C++ bindings.
 *
 * Conventions
 *  - plain pointers and sizes; device addresses are uint64_t; streams are
 *    cudaStream_t passed as void* (NULL = legacy default stream);
 *  - every function returns int: 0 (POS_OK) or a code that maps 1:1 onto the
 *    reference's Errc (include/gpucrsim/errors.hpp:9-25) as POS_E_<Errc> =
 *    1 + enum index, plus POS_E_CUDA / POS_E_NO_DEVICE for the runtime;
 *  - no exceptions cross the ABI; pos_last_error() gives the message;
 *  - not re-entrant per context (the reference is single-threaded,
 *    SPEC.md:104-105); distinct contexts may be used from distinct threads.
 */
#ifndef POSDUMP_H
#define POSDUMP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POSDUMP_ABI_VERSION 3  /* 3: pos_delta_pregather, graph capture, precopy_direct_result waits for the landing */

enum {
  POS_OK = 0,
  /* 1 + gpucrsim::Errc index (errors.hpp:9-25) */
  POS_E_PAST_TIME = 1,
  POS_E_LIVELOCK = 2,
  POS_E_OUT_OF_DEVICE_MEMORY = 3,
  POS_E_INVALID_LOCATOR = 4,
  POS_E_USE_AFTER_FREE = 5,
  POS_E_FREED_BUFFER = 6,
  POS_E_BAD_STATE = 7,
  POS_E_PENDING_KERNELS = 8,
  POS_E_UNKNOWN_API = 9,
  POS_E_INVALID_ARGUMENT = 10,
  POS_E_CORRUPT_DAG = 11,
  POS_E_CORRUPT_IMAGE = 12,
  POS_E_INVARIANT_VIOLATION = 13,
  POS_E_STAGING_EXHAUSTED = 14,
  POS_E_ORACLE_MISMATCH = 15,
  /* runtime */
  POS_E_CUDA = 64,
  POS_E_NO_DEVICE = 65
};

typedef struct pos_ctx pos_ctx;

/* SimConfig keys of the path (include/gpucrsim/config.hpp:18-45). */
typedef struct pos_config {
  uint64_t chunk_size;       /* chunk_size (config.hpp:25); any value > 0 (config.hpp:70-71) */
  uint64_t page_size;        /* page_size (config.hpp:26) */
  uint64_t cache_capacity;   /* O3 on-device cache bytes; 0 => staging_capacity() */
  double staging_fraction;   /* staging_fraction (config.hpp:35); 0 => 1/16 */
  int32_t device;            /* CUDA ordinal */
  int32_t dedup;             /* dedup (config.hpp:36) */
  double dirty_threshold_frac; /* dirty_threshold_frac (config.hpp:32): DAG retention; 0 => 0.25 */
  int32_t trust_written_bit; /* O2 at buffer granularity first (plan_precopy, cr.hpp:396-401): a buffer
                                registered with written_since_ckpt == 0 is neither hashed nor shipped
                                in an incremental round -- exact when the caller tracks every write */
  int32_t pad;
} pos_config;

/* One active allocation of the checkpointed process: the fields of
 * GpuBuffer (buffer.hpp:27-41) and Upstream (buffer.hpp:20-25) the path reads. */
typedef struct pos_buffer_desc {
  uint64_t handle;             /* BufferHandle (buffer.hpp:14) */
  uint64_t dev_ptr;            /* device address of the allocation */
  uint64_t size;               /* GpuBuffer::size, > 0 (buffer.hpp:109) */
  uint32_t has_upstream;       /* GpuBuffer::upstream.has_value() (buffer.hpp:37) */
  uint32_t upstream_crc;       /* Upstream::crc (buffer.hpp:23) */
  uint32_t host_untouched;     /* range_write_seq <= Upstream::host_write_seq (cr.hpp:420) */
  uint32_t written_since_ckpt; /* GpuBuffer::written_since_ckpt (buffer.hpp:34) */
} pos_buffer_desc;

/* ---- errors --------------------------------------------------------- */
const char* pos_strerror(int code);
/* Message of the last failing call on this thread. */
const char* pos_last_error(void);
int pos_abi_version(void);

/* ---- context ---------------------------------------------------------- */
/* Replaces the CrEngine session state (cr.hpp:1271-1321): digest tables,
 * dirty bitmap, O3 cache, CUDA events.  Fails with POS_E_NO_DEVICE when no
 * CUDA device is present (there is no CPU fallback). */
int pos_ctx_create(const pos_config* cfg, pos_ctx** out);
int pos_ctx_destroy(pos_ctx* ctx);

/* snapshot_buffers_ = active_handles() (cr.hpp:346): the buffer set of the
 * dump, ascending handle.  Resets the epoch (next hash is "fresh"). */
int pos_register_buffers(pos_ctx* ctx, const pos_buffer_desc* bufs, uint32_t n);
/* The snapshot's buffer set changed mid-session (allocations join dirty,
 * frees are dropped: cr.hpp:301-306, 709-716).  `bufs` (ascending handle)
 * replaces the registered set; a buffer with an unchanged handle, address and
 * size keeps its digest history, flags and host-image range (the pre-copy
 * stays incremental for it); a new one joins fresh -- every chunk dirty until
 * pos_commit_epoch -- and needs pos_register_image before a direct pre-copy;
 * a missing one is never read again.  Synchronises the device. */
int pos_update_buffer_set(pos_ctx* ctx, const pos_buffer_desc* bufs, uint32_t n);
/* CheckpointTarget::fresh (cr.hpp:35, 396-401): the next round's target does
 * not hold the previous round, so every chunk ships (the O2 skip is off until
 * pos_commit_epoch; digests are still computed). */
int pos_set_target_fresh(pos_ctx* ctx, int fresh);
/* Refresh provenance / written bits of one registered buffer, e.g. after
 * note_h2d_provenance (process.hpp:505-522). */
int pos_update_buffer(pos_ctx* ctx, const pos_buffer_desc* buf);
int pos_num_chunks(pos_ctx* ctx, uint64_t* out);

/* ---- O2: chunk digests + dirty bitmap ---------------------------------- */
/* digest[g] = crc32(chunk g) for every chunk of every registered buffer
 * (per-chunk form of crc32.hpp:26-34 as applied at cr.hpp:419);
 * flag[g] = (no previous epoch) || digest[g] != previous digest[g]; sets the
 * dirty bitmap.  Replaces the O2 branch of plan_precopy (cr.hpp:396-401),
 * refined from buffer to chunk granularity. */
int pos_hash_chunks(pos_ctx* ctx, void* stream);
/* The current digest table becomes the comparison base of the next epoch
 * (finalize_image clearing written_since_ckpt, cr.hpp:745). */
int pos_commit_epoch(pos_ctx* ctx);
int pos_read_digests(pos_ctx* ctx, uint32_t* host, uint64_t n, void* stream);
int pos_read_flags(pos_ctx* ctx, uint8_t* host, uint64_t n, void* stream);
int pos_read_bitmap(pos_ctx* ctx, uint32_t* host, uint64_t nwords, void* stream);

/* ---- O1: whole-buffer CRC + dedup verdicts ----------------------------- */
/* crc[b] = crc32(buffer b) folded from the chunk digests (the value
 * scan_dedup computes, cr.hpp:419, and note_h2d_provenance records,
 * process.hpp:518); verdict[b] = has_upstream && crc == upstream_crc &&
 * host_untouched && !dag_dirty (cr.hpp:420-421, 720). Requires
 * pos_hash_chunks on the same stream first. */
int pos_buffer_crc(pos_ctx* ctx, void* stream);
int pos_read_buffer_crcs(pos_ctx* ctx, uint32_t* crcs, uint8_t* verdicts, uint32_t n,
                         void* stream);

/* ---- DAG write sets ------------------------------------------------------ */
/* dirty_set_ |= spec_writes (record_dirty, cr.hpp:901-931).  Handles not in
 * the snapshot are ignored, as in the reference. */
int pos_record_dirty(pos_ctx* ctx, const uint64_t* handles, uint32_t n);
int pos_clear_dirty(pos_ctx* ctx);

/* ---- H2D provenance (note_h2d_provenance, process.hpp:505-522) ---------- */
/* The application's host-to-device copy of [dst, dst+bytes) from host_src
 * (enqueued here on `stream` when do_copy != 0; otherwise the caller already
 * enqueued it on `stream`), followed on the device by the provenance update
 * of the buffer containing dst: a whole-buffer copy hashes the buffer's
 * chunks and folds them into Upstream::crc (k_hash_chunks + k_note_upstream,
 * no host round trip), sets has_upstream / host_untouched; a partial copy
 * drops the provenance (process.hpp:510-513).  Either way the buffer becomes
 * written_since_ckpt.  No containing buffer: only the copy.  The crc reaches
 * the host lazily (pos_read_upstream). */
int pos_h2d_provenance(pos_ctx* ctx, uint64_t dst, const void* host_src, uint64_t bytes, int do_copy,
                       void* stream);
/* GpuBuffer::upstream (buffer.hpp:37) of a registered buffer: waits for a
 * pending pos_h2d_provenance. */
int pos_read_upstream(pos_ctx* ctx, uint64_t handle, uint32_t* has_upstream, uint32_t* crc);

/* ---- O3: compaction into the on-device cache ---------------------------- */
/* Packs every flagged chunk of every non-dedup buffer (and, when
 * exclude_dag_dirty, outside dirty_set_: chunk_copied abandons those,
 * cr.hpp:487) into the cache as a POSD pack, in
 * (handle, chunk) order, at cache offset 0.  Replaces enqueue_buffer_copy /
 * chunk_copied (cr.hpp:447-504) and stage_buffers (cr.hpp:858-888).
 * Synchronises `stream` once to learn the pack size; the copy itself is left
 * running on `stream`.  POS_E_STAGING_EXHAUSTED if it does not fit. */
int pos_compact(pos_ctx* ctx, int exclude_dag_dirty, void* stream, uint64_t* pack_bytes);
/* The whole pre-copy, asynchronous (plan_precopy, cr.hpp:377-406):
 * pos_hash_chunks + pos_buffer_crc + scan + compaction, with the copy
 * kernel's item count read on the device -- no host round trip.  The pack
 * size becomes available through pos_precopy_size (waits for the scan only). */
int pos_precopy(pos_ctx* ctx, int exclude_dag_dirty, void* stream);
int pos_precopy_size(pos_ctx* ctx, uint64_t* pack_bytes);
/* Pipelined pre-copy: the buffer set in up to `waves` (<= 16) contiguous
 * groups of whole buffers; per wave, on ckpt_stream: hash -> O1 -> scan ->
 * compaction into its own POSD pack (packs chained in the cache); and, when
 * host_dst != NULL, each wave's pack is copied to host_dst at the same offset
 * on copy_stream as soon as it is in the cache -- the D2H of wave k overlaps
 * the hashing of wave k+1.  offsets[] / sizes[] (capacity 16) receive each
 * pack's cache offset and size; returns after the last scan (copies may still
 * be in flight on copy_stream). */
/* Cache-cycled pre-copy for states larger than the O3 cache (BASELINE
 * configs 3 and 5): the chunks are cut into waves whose worst-case pack fits
 * one of two cache regions of region_bytes (0 => half the cache); wave w
 * hashes/compacts into region w%2 while wave w-1 drains over PCIe into one of
 * two pinned landing slots owned by the context; `sink` receives each pack
 * (valid during the call) on the calling thread, in order.  Blocks until the
 * last pack was handed over.  O1 verdicts are decided in the wave holding a
 * buffer's last chunk (a dedup candidate larger than a region may ship chunks
 * it could have skipped; the image is unaffected). */
typedef void (*pos_pack_sink)(void* user, const uint8_t* pack, uint64_t bytes, uint32_t index);
int pos_precopy_stream(pos_ctx* ctx, int exclude_dag_dirty, void* ckpt_stream, void* copy_stream,
                       uint64_t region_bytes, pos_pack_sink sink, void* user, uint64_t* total_bytes,
                       uint32_t* n_packs);
/* NVLink peer-GPU cache for pos_precopy_stream (BASELINE config 5): `bytes`
 * of device memory on peer_device hold whole cache regions; each wave's pack
 * moves there by cudaMemcpyPeerAsync, freeing the local region at NVLink
 * speed, and the peer's copy engine drains the slots to the host (its own
 * PCIe link).  The snapshot is captured when the last wave sits in a slot.
 * bytes == 0 detaches.  peer_device may equal the context's device (a D2D
 * slot pool; single-GPU boxes).  POS_E_OUT_OF_DEVICE_MEMORY if it cannot be
 * allocated. */
int pos_peer_cache_attach(pos_ctx* ctx, int peer_device, uint64_t bytes);
/* Of the last pos_precopy_stream through the peer cache: ms from its start
 * until every pack was in the peer (capture) and until the last byte reached
 * the host (total; -1 when the peer is another device). */
int pos_peer_cache_stats(pos_ctx* ctx, float* capture_ms, float* total_ms);
int pos_precopy_pipelined(pos_ctx* ctx, int exclude_dag_dirty, uint32_t waves, void* ckpt_stream,
                          void* copy_stream, void* host_dst, uint64_t slice_bytes,
                          uint64_t* offsets, uint64_t* sizes, uint32_t* n_packs);

/* ---- direct pre-copy into the host image (chunk_copied, no host copy) -- */
/* The checkpoint target's image of captured_ (cr.hpp:499-501, the byte
 * vectors chunk_copied writes at ci * chunk_size): hosts[i] / sizes[i] is the
 * host copy of registered buffer i (ascending handle; sizes must match).
 * Pinned memory is used as is; pageable ranges are pinned and mapped here
 * (and unpinned at pos_ctx_destroy).  Re-register after pos_register_buffers. */
int pos_register_image(pos_ctx* ctx, uint8_t* const* hosts, const uint64_t* sizes, uint32_t n);
/* Pre-copy straight into the registered image (enqueue_buffer_copy /
 * chunk_copied, cr.hpp:447-504): per wave (<= 16 groups of whole buffers) on
 * ckpt_stream the hash (O2), k_buffer_crc (O1) and the tiled scan, which
 * writes maximal runs of shipped chunks into mapped pinned memory and an
 * index-only POSD pack (header + entries, flag 2) into the cache; the host
 * host leg (a feeder thread) moves each wave's runs on drain_stream the
 * moment the scan lands, as windowed slices: runs of >= 4 MiB as copy-engine
 * copies, shorter ones as k_ship_runs batches (SM stores into the mapped
 * image), so every eligible chunk moves from the live buffer to
 * image + ci*chunk_size with no gather and no host apply.  Returns once the scans are enqueued; work the caller
 * puts on drain_stream afterwards must follow pos_precopy_direct_result (or
 * the final stop, which waits for the host leg itself). */
int pos_precopy_direct(pos_ctx* ctx, int exclude_dag_dirty, uint32_t waves, void* ckpt_stream,
                       void* drain_stream);
/* Chunks and payload bytes the last pos_precopy_direct shipped, and the end
 * of its index packs in the cache.  Blocks until every byte of that
 * pre-copy is in the image (the host leg submitted its last slice and the
 * slice landed). */
int pos_precopy_direct_result(pos_ctx* ctx, uint64_t* chunks, uint64_t* payload_bytes,
                              uint64_t* index_bytes);
/* An application memcpy during a checkpoint (CopyEngine::submit(App),
 * engines.hpp:63-78): enqueued on `stream` (after its earlier work) at once;
 * while a direct pre-copy's host leg is running, the leg submits no further
 * checkpoint slice until this copy has completed -- app over ckpt at slice
 * granularity (engines.hpp:153-159): the copy waits behind at most
 * window x slice bytes of checkpoint traffic.  kind: 1 H2D, 2 D2H, 3 D2D. */
int pos_app_copy(pos_ctx* ctx, uint64_t dst, uint64_t src, uint64_t bytes, int kind, void* stream);
/* Host-leg slicing of the direct pre-copy: slices of at most slice_bytes
 * (>= 64 KiB; default 16 MiB), at most `window` (1..8, default 3) in flight. */
int pos_set_host_leg(pos_ctx* ctx, uint64_t slice_bytes, uint32_t window);
/* Since creation: slices submitted, application copies yielded to, and bytes
 * of runs cancelled because their buffer was recorded dirty (pos_record_dirty)
 * after the scan -- CopyEngine::cancel (cr.hpp:909-918): the final stop
 * re-copies those buffers. */
int pos_host_leg_stats(pos_ctx* ctx, uint64_t* slices, uint64_t* app_yields, uint64_t* cancelled_bytes);
/* After pos_delta_copy with an image registered: the delta pack's payload
 * (already in the cache -- the stop is over) moved into the image on
 * `stream` as runs merged where both sides are contiguous (>= 4 MiB by the
 * copy engine, shorter ones by k_ship_runs).
 * `stream` waits for the STW gather itself (not for the post-stop hash that
 * follows it on the dump stream). */
int pos_delta_drain(pos_ctx* ctx, void* stream);

/* ---- CoW staging (gate_cow / stage_buffers, cr.hpp:806-888) ------------- */
/* A kernel about to overwrite buffers of the snapshot before this epoch's
 * pre-copy has saved them: every chunk of those buffers (in the snapshot,
 * not staged yet) is copied -- and hashed while copying -- into a staging
 * POSD pack (flag 4) at the top of the cache, on `stream` (the application's
 * stream: its next kernel runs after the copy, stream order).  The buffers
 * keep the staged digests and are left out of this epoch's pre-copy; the
 * staged pack is part of the checkpoint.  POS_E_STAGING_EXHAUSTED when the
 * free cache cannot hold it (the reference then delays the kernel,
 * cr.hpp:837); POS_E_BAD_STATE once the epoch's pre-copy has started.  The
 * staging is released by pos_commit_epoch. */
int pos_stage_buffers(pos_ctx* ctx, const uint64_t* handles, uint32_t n, void* stream,
                      uint64_t* pack_offset, uint64_t* pack_bytes);

/* ---- STW delta-copy --------------------------------------------------- */
/* at_final_stop (cr.hpp:599-621): every chunk of the buffers in dirty_set_ is
 * gathered into the cache as a second POSD pack starting at *pack_offset
 * (256-B aligned, after the pre-copy pack).  The stop-the-world part is a
 * pure TMA bulk gather; the chunks are hashed afterwards from the gathered
 * copy (entry crcs + refreshed digests), on the same stream.  Asynchronous. */
int pos_delta_copy(pos_ctx* ctx, void* stream, uint64_t* pack_offset, uint64_t* pack_bytes);
/* Same, recording event `stw_end_slot` (>= 0) right after the gather: the end
 * of the stop-the-world window. */
int pos_delta_copy_ex(pos_ctx* ctx, void* stream, int stw_end_slot, uint64_t* pack_offset,
                      uint64_t* pack_bytes);
/* at_final_stop with the stop-the-world window delimited by the engine: on
 * `stream`, event `stw_begin_slot`, the gather, event `stw_end_slot` -- and
 * nothing else (each extra stream operation costs ~10 us while the copy
 * engine writes to the host); the post-stop hash follows.  The delta timer
 * (pos_last_kernel_ms "delta") reads the two events.  Replaces
 * at_final_stop's copy loop, cr.hpp:599-621. */
int pos_final_stop(pos_ctx* ctx, void* stream, int stw_begin_slot, int stw_end_slot, uint64_t* pack_offset,
                   uint64_t* pack_bytes);
/* Stage the delta pack's header and work list ahead of the stop (the DAG
 * write sets are known at submission, process.hpp:313-344), so the STW window
 * holds only the kernel.  pos_delta_copy re-stages if dirty_set_ or the
 * pre-copy pack changed since. */
int pos_delta_prepare(pos_ctx* ctx, void* stream, uint64_t* pack_offset, uint64_t* pack_bytes);
/* Eager delta capture: gather the listed DAG-dirty buffers into their slots
 * of the prepared delta pack now, on `stream` behind everything
 * `after_stream` has enqueued so far (their last writers), so the final stop
 * gathers only the rest.  A buffer recorded dirty again afterwards
 * (pos_record_dirty: a later writer) is re-gathered at the stop.  The image
 * equals at_final_stop's re-copy (cr.hpp:599-621) either way.  Needs a
 * current pos_delta_prepare (else POS_E_BAD_STATE). */
int pos_delta_pregather(pos_ctx* ctx, const uint64_t* handles, uint32_t n, void* after_stream, void* stream);

/* ---- host leg ------------------------------------------------------------- */
/* Pinned D2H of cache[offset, offset+bytes) into host_dst, on `stream`, in
 * slices of at most slice_bytes (0 => 8 MiB) so application copies queued on
 * other streams interleave (engines.hpp:153-159). */
int pos_d2h_async(pos_ctx* ctx, void* host_dst, uint64_t offset, uint64_t bytes,
                  uint64_t slice_bytes, void* stream);
int pos_cache_info(pos_ctx* ctx, uint64_t* dev_ptr, uint64_t* capacity);

/* ---- restore scatter ------------------------------------------------------ */
/* Apply a POSD pack resident in device memory onto the registered buffers
 * (materialize/load_complete, cr.hpp:1026-1084).  POS_E_CORRUPT_IMAGE for a
 * malformed pack, POS_E_INVALID_LOCATOR for an entry outside its buffer or
 * an unknown handle.  Synchronises `stream` once to validate. */
int pos_scatter(pos_ctx* ctx, uint64_t pack_dev_ptr, uint64_t pack_bytes, void* stream);

/* Host side of the same scatter: apply a POSD pack held in host memory onto
 * host copies of the buffers (the checkpoint target's image of captured_,
 * cr.hpp:499-501).  hosts[i]/sizes[i] belong to handles[i] (ascending).
 * Entries are applied with `threads` host threads (0 => 1). */
int pos_pack_apply_host(const uint8_t* pack, uint64_t pack_bytes, const uint64_t* handles,
                        uint8_t* const* hosts, const uint64_t* sizes, uint32_t n,
                        uint32_t threads);

/* Streaming restore (start_loads / load_complete / materialize,
 * cr.hpp:1043-1084): packs held in host memory (the base image's packs, then
 * the incremental ones -- delta-restore) are validated on the host (all or
 * nothing, like write_content, buffer.hpp:80), copied H2D through two cache
 * regions of region_bytes (0 => half the cache) on h2d_stream, and scattered
 * onto the registered buffers on `stream` in order, so a later pack overrides
 * an earlier one.  Pageable packs are staged through pinned landing slots with
 * the host's threads.  Returns when the last scatter finished. */
int pos_restore_packs(pos_ctx* ctx, const uint8_t* const* packs, const uint64_t* sizes, uint32_t n,
                      void* h2d_stream, void* stream, uint64_t region_bytes);

/* On-demand restore of a flat host image (restore(), cr.hpp:167-204:
 * start_loads / enqueue_load / gate_restore, cr.hpp:1043-1143): hosts[i] is
 * the image of registered buffer i (the direct pre-copy's image, or any host
 * copy).  A loader thread feeds H2D slices of slice_bytes (0 => 8 MiB) on
 * h2d_stream in `order` (topo_order_buffers, dag.hpp:141-202; the rest by
 * handle), at most 4 slices ahead, and records a ready event per buffer.
 * Returns at once. */
int pos_restore_image_begin(pos_ctx* ctx, uint8_t* const* hosts, const uint64_t* sizes, uint32_t n,
                            const uint64_t* order, uint32_t norder, uint64_t slice_bytes, void* h2d_stream);
/* bump_front (engines.hpp:86-93): the buffer's remaining slices go next. */
int pos_restore_want(pos_ctx* ctx, uint64_t handle);
/* gate_restore for one buffer of a kernel about to be enqueued on `stream`:
 * bumps it, waits (host) until its last slice is issued, then makes
 * `stream` wait (device) for it to land.  No restore running: no-op. */
int pos_restore_gate(pos_ctx* ctx, uint64_t handle, void* stream);
int pos_restore_ready(pos_ctx* ctx, uint64_t handle, int* ready);
/* hosts[i] == NULL marks buffer i as a Recompute record (cr.hpp:731-735): it
 * is not loaded but regenerated by delta-restore replay; after its writer is
 * enqueued, pos_restore_replayed (buffer_ready, cr.hpp:1105-1119) records its
 * ready event on the writer's stream, and pos_restore_gate on it waits (host:
 * until replayed; device: until the writer ran). */
int pos_restore_replayed(pos_ctx* ctx, uint64_t handle, void* stream);
/* All buffers loaded (check_all_loaded, cr.hpp:1091-1096) and every
 * Recompute buffer replayed (else POS_E_BAD_STATE, nothing torn down); ends
 * the restore. */
int pos_restore_image_wait(pos_ctx* ctx);

/* ---- device crc32 (crc32.hpp:26-34 over device memory) ---------------- */
int pos_crc32(uint64_t dev_ptr, uint64_t n, uint32_t* out, void* stream);
int pos_crc32_update(uint32_t crc, uint64_t dev_ptr, uint64_t n, uint32_t* out, void* stream);

/* ---- synthetic writes ------------------------------------------------- */
/* dst[0..n) = fill_bytes(seed) (rng.hpp:43-54): the kernel effect of
 * apply_kernel_effect (process.hpp:256-259).  Asynchronous. */
int pos_fill(uint64_t dev_ptr, uint64_t n, uint64_t seed, void* stream);
/* Batched form: ranges[i] = {dev_ptr, n, seed}. */
int pos_fill_batch(const uint64_t* ranges, uint32_t count, void* stream);
/* CUDA graphs for launch-bound callers (the bench's application window):
 * capture what this thread enqueues on `stream` (thread-local mode), then
 * launch the instantiated graph as ONE stream operation. */
int pos_stream_begin_capture(void* stream);
int pos_stream_end_capture(void* stream, void** graph_exec);
int pos_graph_launch(void* graph_exec, void* stream);
int pos_graph_destroy(void* graph_exec);

/* ---- timing ----------------------------------------------------------- */
int pos_event_record(pos_ctx* ctx, uint32_t slot, void* stream);
int pos_event_elapsed(pos_ctx* ctx, uint32_t a, uint32_t b, float* ms);
/* `stream` waits for event `slot` (cross-stream drain: the STW delta-copy
 * waits for the application stream, cr.hpp:591-597). */
int pos_stream_wait_event(pos_ctx* ctx, uint32_t slot, void* stream);
/* Device timeline: for each internal timer (hash, combine, scan, copy, delta,
 * scatter, d2h) the ms from event `slot` to its begin and end (-1 if unused). */
int pos_timeline(pos_ctx* ctx, uint32_t slot, float* out14);
/* Device clock (globaltimer) stamp in stream order, by a one-thread kernel;
 * pos_delta_copy_ex also stamps its stw_end_slot.  Elapsed ms between two
 * stamps (synchronises the device). */
int pos_stamp(pos_ctx* ctx, uint32_t slot, void* stream);
int pos_stamp_elapsed(pos_ctx* ctx, uint32_t a, uint32_t b, float* ms);
/* SMs the hash kernel may occupy (0 = all, the default).  Each hash CTA
 * holds an SM's shared memory for its wave (192 KiB of tables) and 3/4 of
 * its registers, so the application's kernels run beside it and on the rest -- the ChecksumEngine's rate budget (checksum_bw,
 * config.hpp:20-23) on a real GPU.  A host-link-bound dump needs ~1/8 of
 * the SMs to keep its hash ahead of the copy engine. */
int pos_set_hash_sms(pos_ctx* ctx, uint32_t sms);
/* A second, non-linear 32-bit chunk digest beside CRC-32 in the O2 compare
 * (on = 1): a chunk counts as unchanged only if both digests are.  CRC-32 is
 * GF(2)-linear, so a change by a multiple of its polynomial keeps it; the
 * second digest (a position-keyed multiply-xorshift sum) catches that.  The
 * reported digests stay the reference's CRC-32 (crc32.hpp:26-34).  Off by
 * default; the first epoch after switching it on compares CRC-32s only. */
int pos_set_o2_digest2(pos_ctx* ctx, int on);
/* Kernels this context has launched (monotone counter). */
int pos_launch_count(pos_ctx* ctx, uint64_t* out);
/* Device time of the most recent hash kernel launch (ms). */
int pos_last_kernel_ms(pos_ctx* ctx, const char* which, float* ms);

/* ---- POSI image (image.hpp:136-207, canonical writer) ------------------ */
typedef struct pos_image_rec {
  uint64_t handle;
  uint32_t kind;               /* 0 Inline, 1 DedupRef, 2 Recompute (image.hpp:42) */
  uint32_t n_recompute;
  const uint8_t* inline_bytes; /* host bytes of the buffer (kind 0) */
  uint64_t inline_len;
  uint64_t dedup_first_page;
  uint32_t dedup_page_count, dedup_offset, dedup_crc, reserved;
  const uint64_t* recompute;
} pos_image_rec;
typedef struct pos_image_alloc {
  uint64_t handle, base, size;
} pos_image_alloc;
typedef struct pos_image_page {
  uint64_t index;
  const uint8_t* bytes; /* page_size bytes */
} pos_image_page;
typedef struct pos_image_desc {
  uint64_t page_size;
  const pos_image_page* pages; uint32_t n_pages;
  const pos_image_rec* recs; uint32_t n_recs;
  const pos_image_alloc* allocs; uint32_t n_allocs;
  const uint64_t* stream_ids; uint32_t n_streams;
  uint64_t cursor, next_handle, next_base;
  const uint8_t* dag_bytes; uint64_t dag_len;
} pos_image_desc;
/* Byte-identical to gpucrsim::write_image.  *size always receives the image
 * size; bytes are written when cap >= size. */
int pos_image_write(const pos_image_desc* img, uint8_t* out, uint64_t cap, uint64_t* size);

/* ---- finalize_image (cr.hpp:680-764) ----------------------------------- */
/* One snapshot buffer still live at finalize (a dirty-bit image drops the
 * buffers freed during the session and the caller leaves them out,
 * cr.hpp:709-716). */
typedef struct pos_finalize_buf {
  uint64_t handle, base, size;     /* its AllocEntry (image.hpp:60-64) */
  const uint8_t* inline_bytes;     /* captured_[h] (cr.hpp:738-740): the host image range the dump wrote */
  uint64_t up_host_addr, up_len;   /* dedup_snapshot_[h]: the Upstream scan_dedup saw (cr.hpp:436) */
  uint32_t up_crc;
  uint32_t has_upstream;
  int32_t dedup_ok;                /* scan_dedup's verdict (dedup_ok_, cr.hpp:441); -1: the context's device O1 verdict */
  uint32_t dirty;                  /* h in dirty_set_ */
  uint32_t recompute_eligible;     /* recompute_eligible(h) (cr.hpp:938-951): decided by the kernel DAG */
  uint32_t n_recompute;
  const uint64_t* recompute_nodes; /* pending_writers(h) (dag.hpp:234-243) */
  uint32_t precopy_survived;       /* retention_ && fully_copied && !final_outstanding (cr.hpp:741) */
  uint32_t pad;
} pos_finalize_buf;

/* CrMetrics (cr.hpp:69-119): the fields the dump path accounts.  For a
 * dirty-bit checkpoint bytes_precopy + bytes_dirty + bytes_dedup_saved ==
 * the sum of the image's allocation sizes (tests/test_harness.cpp:99-112). */
typedef struct pos_metrics {
  uint64_t bytes_precopy;          /* buffer bytes whose concurrent copy survived */
  uint64_t bytes_dirty;            /* buffer bytes re-copied at the final stop */
  uint64_t bytes_dedup_saved;
  uint64_t bytes_recompute_saved;
  uint64_t image_bytes;            /* GPU section + DAG section */
  uint64_t image_file_bytes;
  uint64_t dirty_count;            /* |dirty_set_| at the final stop */
  uint64_t retention_dirty_count;
  uint32_t retention;              /* the DAG-retention threshold was crossed (cr.hpp:921-929) */
  uint32_t n_inline, n_dedup, n_recompute;
} pos_metrics;

/* finalize_image: the record kind of every buffer -- DedupRef when the O1
 * verdict holds, the buffer is not in dirty_set_ and dedup_consistent (a
 * chained crc32 over the image's host pages equals the Upstream crc,
 * cr.hpp:692-708); Recompute when dirty and recompute-eligible; else Inline
 * from captured_ -- then the POSI image (write_image, byte-identical) into
 * out (*size always receives the image size; bytes are written when cap >=
 * size) and the session metrics.  `host_side` carries what the CPU side and
 * the DAG contribute: page_size, host pages, stream ids, cursor,
 * next_handle / next_base and the DAG bytes (its recs / allocs must be
 * empty).  ctx may be NULL when no verdict is taken from a device. */
int pos_finalize_image(pos_ctx* ctx, const pos_image_desc* host_side, const pos_finalize_buf* bufs, uint32_t n,
                       uint8_t* out, uint64_t cap, uint64_t* size, pos_metrics* metrics);
/* The context's metrics of the current session (final stop + finalize). */
int pos_get_metrics(pos_ctx* ctx, pos_metrics* metrics);
/* at_final_stop's exclusions (cr.hpp:608-613): buffers of dirty_set_ the
 * final stop does NOT re-copy -- freed before the stop, recompute-eligible,
 * or (under DAG retention) already fully copied.  Replaces the previous
 * list; cleared by pos_commit_epoch. */
int pos_set_stop_exclusions(pos_ctx* ctx, const uint64_t* handles, uint32_t n);

/* read_image (image.hpp:209-361): validate a POSI image on the host -- the
 * reference's checks in its order; POS_E_CORRUPT_IMAGE with the reader
 * offset of its CorruptImageError in *corrupt_offset.  The DAG section is
 * checked as KernelDag::deserialize reads it (dag.hpp:322-387: node and edge
 * records, kinds, lengths, trailing bytes; a bad structure reports offset 0
 * like read_image's "dag: ..." rethrow) and every Recompute node must be a
 * kernel of it. */
int pos_image_check(const uint8_t* img, uint64_t size, uint64_t* corrupt_offset);
/* Restore from a POSI image (read_image + install/materialize, cr.hpp:
 * 1026-1030, dedup_content image.hpp:364-376): validate it in full (dedup
 * checksums included -- nothing is written from a corrupt image), then every
 * Inline / DedupRef record of a registered buffer is copied H2D on `stream`
 * (DedupRef assembled from the image's host pages); Recompute
 * records are left to delta-restore replay (cr.hpp:1099-1119).  Registered
 * buffers must have the image's allocation sizes (POS_E_INVALID_LOCATOR). */
int pos_image_restore(pos_ctx* ctx, const uint8_t* img, uint64_t size, void* stream, uint64_t* corrupt_offset,
                      uint32_t* n_loaded, uint32_t* n_recompute);

/* ---- plumbing (device memory / streams for hosts without their own) ---- */
int pos_device_count(int* n);
int pos_set_device(int device);
int pos_dev_malloc(uint64_t bytes, uint64_t* dev_ptr);
int pos_dev_free(uint64_t dev_ptr);
int pos_host_malloc_pinned(uint64_t bytes, void** host);
int pos_host_free_pinned(void* host);
/* Host memory for a checkpoint image (the target of pos_register_image):
 * pinned + mapped, allocated as transparent huge pages first-touched by
 * `threads` host threads (0 => 16) -- ~10x faster than cudaHostAlloc for
 * the 100+ GB images of BASELINE configs 3/5.  Zero-filled. */
int pos_host_image_alloc(uint64_t bytes, uint32_t threads, void** host);
int pos_host_image_free(void* host);
/* kind: 1 H2D, 2 D2H, 3 D2D (cudaMemcpyKind); asynchronous on `stream`. */
int pos_memcpy(uint64_t dst, uint64_t src, uint64_t bytes, int kind, void* stream);
int pos_memset(uint64_t dev_ptr, int value, uint64_t bytes, void* stream);
int pos_stream_create(void** stream);
/* priority: 0 = default, 1 = highest the device allows (the dump's kernels
 * then win SMs over queued application blocks). */
int pos_stream_create_prio(int priority, void** stream);
int pos_stream_destroy(void* stream);
int pos_stream_sync(void* stream);
int pos_device_sync(void);
/* Cross-stream ordering: `waiter` waits for work queued so far on `signaller`. */
int pos_stream_wait(void* waiter, void* signaller);

#ifdef __cplusplus
}
#endif
#endif /* POSDUMP_H */
