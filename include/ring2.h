/*
 * ring2.h — C ABI of the B200-native Ring^2 capture-and-stage path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (tapflow, /root/reference/pkg/src/tapflow). The reference is pure
 * Python with no FFI; every entry point below replaces one Python-level
 * call the reference makes on this path, cited as file:line. A host
 * binding (ctypes) re-exposes the same names.
 *
 * Conventions
 *   - every function is extern "C", returns a tf_status (0 = ok) that maps
 *     1:1 onto the reference's exception classes (errors.py), and takes only
 *     plain pointers and integer sizes;
 *   - producer entry points (tf_capture) are launch-only: they enqueue work
 *     on the caller's CUDA stream (NULL = the legacy default stream, as in
 *     the CUDA runtime), never synchronise it, and are legal
 *     inside CUDA-graph capture. Ring-full is reported through device
 *     counters and the result slot, not through the return code;
 *   - consumer entry points (poll/release/stager) run on host threads.
 *   One producer stream and one consumer context per ring (rings.py:196-202).
 */
#ifndef RING2_H_
#define RING2_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_ABI_VERSION 1
#define TF_COPY_UNIT 16u                          /* rings.py:50 */
#define TF_DESCRIPTOR_SIZE 64u                    /* rings.py:51 */
#define TF_READY_SENTINEL 0xFFFFFFFFFFFFFFFFull   /* rings.py:52 */

/* Status codes: one per exception class in errors.py:6-62. */
typedef enum {
  TF_OK = 0,
  TF_ERR_CONFIG = 1,               /* ConfigError          errors.py:10   */
  TF_ERR_ALLOCATION = 2,           /* AllocationError      errors.py:14   */
  TF_ERR_PAYLOAD_RING_FULL = 3,    /* PayloadRingFull      errors.py:26   */
  TF_ERR_META_RING_FULL = 4,       /* MetaRingFull         errors.py:30   */
  TF_ERR_OUT_OF_ORDER_RELEASE = 5, /* OutOfOrderRelease    errors.py:34   */
  TF_ERR_PROTOCOL = 6,             /* ProtocolError        errors.py:38   */
  TF_ERR_META_MISMATCH = 7,        /* MetaMismatch         errors.py:42   */
  TF_ERR_POLICY_UNDERESTIMATE = 8, /* PolicyUnderestimate  errors.py:49   */
  TF_ERR_STAGING_EXHAUSTED = 9,    /* StagingExhausted     errors.py:53   */
  TF_ERR_HOOK_DISABLED = 10,       /* HookDisabled         errors.py:57   */
  TF_ERR_VALUE = 11,               /* ValueError raised by rings.py:293-298 */
  TF_ERR_CUDA = 12,                /* CUDA runtime failure (no reference analogue) */
  TF_ERR_TIMEOUT = 13,             /* bounded wait expired (wallclock.py:183-194) */
  TF_ERR_EMPTY = 14                /* nothing to return (queue empty)      */
} tf_status;

/* 64-byte little-endian descriptor, rings.py:13-22. Bytes 0..31 are the
 * reference wire layout bit for bit; bytes 32..63 are "reserved" in the
 * reference (zero-filled by Descriptor.pack, ignored by unpack,
 * rings.py:98-113) and carry transport facts the device producer needs to
 * hand to the host consumer. */
typedef struct tf_descriptor {
  uint64_t payload_offset; /* @0  */
  uint64_t payload_len;    /* @8  unpadded */
  uint32_t hook_id;        /* @16 */
  uint32_t step_seq;       /* @20 */
  uint64_t ready_seq;      /* @24 sentinel = free */
  /* reserved area */
  uint64_t skip_before;    /* @32 dead-skip or empty-reset skip before region */
  uint32_t flags;          /* @40 TF_DESC_* */
  uint32_t n_rows;         /* @44 rows gathered into the payload */
  uint64_t capture_seq;    /* @48 producer launch counter */
  uint64_t checksum;       /* @56 mix of words 0..6; the host accepts a slot
                              only when it verifies (no fence on publish) */
} tf_descriptor;

#define TF_DESC_DEAD_SKIP 0x1u     /* skip_before bytes are a dead region */
#define TF_DESC_EMPTY_RESET 0x2u   /* skip_before bytes were an empty-ring reset */
#define TF_DESC_HOST_RESERVED 0x4u /* region registered via tf_ring_reserve */
/* Bits 16..31 of flags (device-internal, cleared before descriptors are
 * handed out): the number of capture CTAs whose completion flags the host
 * must see before it may take the slot (0: posted after completion). */
#define TF_DESC_CTA_SHIFT 16u
/* Bit 15 of flags (device-internal, cleared before descriptors are handed
 * out): posted by a TF_CAP_SEALED capture, complete per the rule above. */
#define TF_DESC_PENDING 0x8000u

typedef struct tf_ring_config {
  uint64_t payload_capacity; /* bytes, >0, multiple of 16 (rings.py:75-81) */
  uint32_t meta_slots;       /* >0 (rings.py:82-83) */
  uint32_t _pad;
  double high_watermark;     /* (0,1] (rings.py:84-85) */
  uint64_t wait_timeout_ns;  /* device wait bound for TF_FULL_WAIT; 0 = 30 s */
} tf_ring_config;

/* Snapshot, rings.py:121-144 plus the conservation counters rings.py:223-229. */
typedef struct tf_ring_state {
  uint64_t payload_head;
  uint64_t payload_tail;
  uint64_t occupancy;
  uint64_t payload_capacity;
  uint64_t meta_head;
  uint64_t meta_tail;
  uint64_t meta_slots;
  double high_watermark;
  uint64_t bytes_reserved;
  uint64_t bytes_released;
  uint64_t dead_created;
  uint64_t dead_reclaimed;
  uint64_t descriptors_published;
  uint64_t descriptors_consumed;
  /* device-side counters (no reference analogue: the reference raises) */
  uint64_t captures_launched;
  uint64_t drops;             /* captures dropped on device ring-full */
  uint64_t drop_bytes;
  uint64_t stall_events;      /* waits under TF_FULL_WAIT */
  uint64_t stall_ns;
  uint64_t device_errors;     /* bitmask of TF_DEVERR_* */
  /* Producer latency (device globaltimer), NOT the kernel duration: on the
     fast path the controller CTA stamps entry -> producer-state commit, which
     ends while copy CTAs are still copying; on the slow path the last CTA
     stamps entry -> descriptor. Time kernels with CUDA events instead. */
  uint64_t kernel_ns;         /* sum of producer latencies */
  uint64_t last_kernel_ns;    /* producer latency of the most recent capture */
} tf_ring_state;

#define TF_DEVERR_UNDERESTIMATE 0x1u /* drop under TF_FULL_DROP (best effort) */
#define TF_DEVERR_TIMEOUT 0x2u       /* TF_FULL_WAIT timed out */
#define TF_DEVERR_TOO_LARGE 0x4u     /* capture larger than the ring */
#define TF_DEVERR_PROTOCOL 0x8u      /* meta slot not at sentinel */

/* What a capture does when the ring cannot take it. */
#define TF_FULL_RAISE 0u /* fail without mutation, status in result slot (hooks.py:294-296) */
#define TF_FULL_WAIT 1u  /* spin on device until the consumer frees space (completeness) */
#define TF_FULL_DROP 2u  /* drop and count (best effort; flags PolicyUnderestimate) */
#define TF_FULL_MASK 3u
#define TF_CAP_DEFER_PUBLISH 0x4u  /* hooks.py:321-322: reserve + copy, no publish */
#define TF_CAP_KEEP_PER_OUTER 0x8u /* keep[] indexed by outer index (request keep) */
/* Completion by stream order (no reference analogue): the copy CTAs skip
 * their fence and completion bytes; the descriptor is complete once a later
 * capture on the same stream has posted the next descriptor, or a
 * tf_ring_seal launched after it on that stream has run. Requires one
 * producer stream per ring (as the producer snapshots do) and a seal at the
 * end of every burst of captures (Observer.end_step / flush). */
#define TF_CAP_SEALED 0x10u

/* Element types. The first eight are DTYPE_WIDTHS (hooks.py:24-27); fp8
 * types are a north-star extension for cast captures. */
typedef enum {
  TF_U8 = 0, TF_I8 = 1, TF_F16 = 2, TF_BF16 = 3, TF_F32 = 4, TF_I32 = 5,
  TF_F64 = 6, TF_I64 = 7, TF_F8E4M3 = 8, TF_F8E5M2 = 9
} tf_dtype;

typedef enum { TF_OP_COPY = 0, TF_OP_CAST = 1, TF_OP_REDUCE = 2 } tf_op;

/* Per-row reductions (north-star extension; f32 outputs). */
typedef enum {
  TF_RED_MEAN = 0,   /* k=1 */
  TF_RED_L2 = 1,     /* k=1  sqrt(sum x^2) */
  TF_RED_ABSMAX = 2, /* k=1 */
  TF_RED_RMS = 3,    /* k=1  sqrt(mean x^2) */
  TF_RED_STATS = 4   /* k=4  mean, l2, min, max */
} tf_reduce;

/* One capture: gather the kept rows of a strided source into one ring
 * region (hooks.py:281-324 capture + hooks.py:266-278 _gather_compact).
 * Source rows are indexed (o, m), o < outer, m < mid, at
 * src + o*stride_outer + m*stride_mid, each row_bytes long. Kept rows are
 * packed unpadded in (o, m) order. keep == NULL keeps every row. */
typedef struct tf_capture_args {
  const void* src;
  int64_t outer;
  int64_t mid;
  int64_t row_bytes;      /* input bytes per row */
  int64_t stride_outer;   /* bytes */
  int64_t stride_mid;     /* bytes */
  const uint8_t* keep;    /* device ptr: outer entries (KEEP_PER_OUTER) or outer*mid */
  const uint32_t* step_seq_ptr; /* device ptr read at run time, or NULL */
  uint32_t step_seq;      /* used when step_seq_ptr == NULL */
  uint32_t hook_id;
  uint32_t op;            /* tf_op */
  uint32_t in_dtype;      /* tf_dtype (cast/reduce) */
  uint32_t out_dtype;     /* tf_dtype (cast) */
  uint32_t reduce_op;     /* tf_reduce */
  uint32_t flags;         /* TF_FULL_* | TF_CAP_* */
  uint32_t max_ctas;      /* 0 = auto */
} tf_capture_args;

/* Result of the most recent capture launch on a ring (written by the
 * device into host-mapped memory; valid after the stream is synchronised). */
typedef struct tf_capture_result {
  uint64_t capture_seq;
  uint32_t status;      /* tf_status */
  uint32_t n_rows;
  uint64_t payload_offset;
  uint64_t payload_len;
  uint64_t skip_before;
  uint64_t ready_seq;   /* TF_READY_SENTINEL if not published */
  tf_descriptor desc;   /* the descriptor (also for DEFER_PUBLISH) */
} tf_capture_result;

typedef struct tf_ring tf_ring;

/* ---- library ---------------------------------------------------------- */
int tf_abi_version(void);
const char* tf_status_name(int status);
const char* tf_last_error(void);   /* thread-local detail string */
int tf_device_count(int* out);

/* Pure allocator, rings.py:166-193 (_plan_reservation). Same code the
 * device runs. Returns 1 and fills off/dead when it fits, else 0. */
int tf_plan_reservation(uint64_t head, uint64_t tail, uint64_t used,
                        uint64_t capacity, uint64_t length,
                        uint64_t* offset, uint64_t* dead);

/* ---- ring pair lifecycle: rings.py:204-229, 434-437 -------------------- */
int tf_ring_create(const tf_ring_config* cfg, int device, tf_ring** out);
int tf_ring_destroy(tf_ring* ring);
int tf_ring_payload_ptr(tf_ring* ring, void** device_ptr);      /* payload_view base, rings.py:278-282 */
int tf_ring_meta_ptr(tf_ring* ring, void** host_ptr);           /* meta ring (64 B slots) */

/* ---- producer role ----------------------------------------------------- */
/* hooks.py:281-324 capture(); launch-only, graph-capturable. */
int tf_capture(tf_ring* ring, void* stream, const tf_capture_args* args);
/* Output bytes per kept row for an op (slice arithmetic, hooks.py:108-109). */
int tf_capture_out_row_bytes(const tf_capture_args* args, int64_t* out);
/* rings.py:286-319 reserve_payload, run by the device allocator; synchronous. */
int tf_ring_reserve(tf_ring* ring, void* stream, uint64_t length,
                    uint64_t* offset, uint64_t* skip_before);
/* rings.py:321-342 publish, run on the device; synchronous; returns ready_seq. */
int tf_ring_publish(tf_ring* ring, void* stream, const tf_descriptor* desc,
                    uint64_t* ready_seq);
/* Result slot of the last tf_capture (after the stream is synchronised). */
int tf_ring_last_result(tf_ring* ring, tf_capture_result* out);

/* ---- consumer role: rings.py:357-431 ----------------------------------- */
int tf_ring_ready_entries(tf_ring* ring, uint64_t* n);
int tf_ring_ready_bytes(tf_ring* ring, uint64_t* n);
int tf_ring_peek_ready(tf_ring* ring, uint32_t max_entries,
                       tf_descriptor* out, uint32_t* n);
int tf_ring_poll_ready(tf_ring* ring, uint32_t max_entries,
                       tf_descriptor* out, uint32_t* n);
int tf_ring_release_payload(tf_ring* ring, uint64_t offset, uint64_t length);
/* Wait until the device sees every release/poll made so far (the cursors
 * reach device memory through stream-ordered writes). */
int tf_ring_sync_consumer(tf_ring* ring);
/* Stream-ordered seal: once every earlier kernel on `stream` has completed,
 * mark all descriptors posted so far complete (TF_CAP_SEALED captures). */
int tf_ring_seal(tf_ring* ring, void* stream);
/* Consumer-side totals the host already holds (no device access, no
 * synchronisation): reserved bytes released (dead skips excluded) and
 * descriptors consumed.
 * Monotonic; the admission gate of eager captures polls it (no reference
 * analogue: the reference producer raises instead of waiting). */
int tf_ring_host_released(tf_ring* ring, uint64_t* bytes_released, uint64_t* consumed);

/* ---- shared: rings.py:241-276 ------------------------------------------ */
/* Snapshot; the caller must have synchronised the producer stream. */
int tf_ring_get_state(tf_ring* ring, tf_ring_state* out);
int tf_ring_free_meta_slots(tf_ring* ring, uint64_t* n);
/* meta_entries < 0 means one per length (rings.py:275). */
int tf_ring_would_fit(tf_ring* ring, const uint64_t* lengths, uint32_t n,
                      int64_t meta_entries, int* fits);

/* ---- staging engine: exporter.py:35-303 ------------------------------- */
#define TF_STAGE_COPY_ENGINE 0 /* cudaMemcpyAsync on a side stream, event-fenced */
#define TF_STAGE_MAPPED 1      /* SM stores into mapped pinned memory */

/* What the page-out stage does with a landed pinned batch. */
#define TF_PAGE_OUT_COPY 0     /* copy to pageable memory, return the pinned
                                  buffer first (exporter.py:237-249) */
#define TF_PAGE_OUT_HANDOFF 1  /* zero-copy: hand the pinned buffer to the
                                  consumer; it returns on tf_stager_free_paged */
#define TF_PAGE_OUT_DISCARD 2  /* D2H-only measurement: drop after landing */

typedef struct tf_drain_config {           /* exporter.py:35-51 */
  uint64_t min_ready_entries;
  uint64_t min_ready_bytes;
  double max_wait;                         /* seconds */
  uint64_t staging_buffer_size;
  uint64_t staging_buffer_count;
  uint32_t mode;                           /* TF_STAGE_* */
  uint32_t mapped_ctas;                    /* CTAs for TF_STAGE_MAPPED (0 = auto) */
  int32_t numa_node;                       /* -1 = auto from the GPU's PCI node */
  uint32_t stage_queue_slots;              /* exporter.py:32 (0 = 16) */
  uint32_t stage_threads;                  /* pinned->pageable copy threads (0 = auto) */
  uint32_t page_out;                       /* TF_PAGE_OUT_* */
  /* 0 (reference behaviour, exporter.py:197-202): a capture larger than one
     staging buffer is a ConfigError. 1 (extension): it is staged in
     buffer-sized chunks through ceil(len / staging_buffer_size) buffers of
     the pool and paged out into one contiguous host allocation. */
  uint32_t split_oversize;
} tf_drain_config;

typedef struct tf_stager tf_stager;

typedef struct tf_batch_info {             /* exporter.py:98-110 DrainBatch */
  uint64_t batch_id;
  uint32_t n_entries;
  uint32_t buffer_index;
  uint64_t bytes_total;
  uint32_t reason;                         /* TF_REASON_* */
  uint32_t _pad;
} tf_batch_info;

#define TF_REASON_NONE 0
#define TF_REASON_ENTRIES 1
#define TF_REASON_BYTES 2
#define TF_REASON_TIMEOUT 3
#define TF_REASON_FLUSH 4

typedef struct tf_stager_stats {
  uint64_t batches_drained;
  uint64_t batches_staged;
  uint64_t entries_drained;
  uint64_t bytes_drained;        /* D2H payload bytes */
  double transfer_seconds;       /* sum of D2H durations (CUDA events) */
  uint64_t pool_checkouts;
  uint64_t pool_max_in_use;
  uint64_t max_transient_bytes;
  uint64_t pageable_bytes_in_flight;
  uint64_t staging_exhausted_waits;
  double first_drain_time;       /* monotonic seconds */
  double last_release_time;
  uint64_t pool_total;
  uint64_t pool_free;
  /* queue depths and thread phases (diagnostics) */
  uint64_t inflight_batches;     /* D2H issued, not yet complete */
  uint64_t to_stage_batches;     /* landed, waiting for page-out */
  uint64_t out_q_batches;        /* paged out, waiting for the consumer */
  uint64_t outstanding_paged;    /* taken by the consumer, not yet freed */
  uint32_t completion_phase;     /* 0 idle, 1 waiting on a D2H event, 2 releasing */
  uint32_t stage_phase;          /* 0 idle, 1 allocating, 2 copying, 3 waiting for out_q room */
} tf_stager_stats;

int tf_stager_create(tf_ring* ring, const tf_drain_config* cfg, tf_stager** out);
int tf_stager_destroy(tf_stager* st);
/* exporter.py:166-178: which threshold fires now (TF_REASON_*). */
int tf_stager_thresholds_met(tf_stager* st, double now, uint32_t* reason);
/* Publish times for the max_wait threshold (exporter.py:158-164). */
int tf_stager_note_publish(tf_stager* st, double now);
/* exporter.py:182-228: take ready descriptors that fit one buffer, D2H. */
int tf_stager_drain_once(tf_stager* st, double now, int flush, tf_batch_info* out);
int tf_stager_batch_entries(tf_stager* st, uint64_t batch_id, tf_descriptor* descs,
                            uint64_t* starts, uint32_t max_entries);
/* Host pointer of the batch's pinned buffer (waits for the transfer). */
int tf_stager_batch_buffer(tf_stager* st, uint64_t batch_id, void** host_ptr);
/* Wait for the batch's D2H and report its measured duration (no release). */
int tf_stager_transfer_seconds(tf_stager* st, uint64_t batch_id, double* seconds);
/* exporter.py:230-233: wait for the D2H, release payload regions. */
int tf_stager_complete_transfer(tf_stager* st, uint64_t batch_id, double* seconds);
/* exporter.py:237-249: copy to pageable dst, return the buffer to the pool. */
int tf_stager_stage_to_pageable(tf_stager* st, uint64_t batch_id, void* dst,
                                uint64_t dst_capacity);
/* Background engine: drain + stage threads (wallclock.py:136-181 shape). */
int tf_stager_start(tf_stager* st);
int tf_stager_stop(tf_stager* st);
/* Force drains until the ring is empty (exporter.py:283-303 flush). */
int tf_stager_flush(tf_stager* st, double timeout_s);
/* Next pageable batch (descriptors + heap payload); TF_ERR_EMPTY on timeout
 * or TF_ERR_TIMEOUT. Payload ownership passes to the caller: free it with
 * tf_free_host. */
typedef struct tf_paged_batch {
  uint64_t batch_id;
  uint32_t n_entries;
  uint32_t reason;
  uint64_t bytes_total;
  void* payload;             /* pageable (copy) or pinned (hand-off), bytes_total long */
  tf_descriptor* descs;      /* malloc'd, n_entries long */
  uint64_t* starts;          /* malloc'd, n_entries long */
  int32_t pinned_buffer;     /* pool index under TF_PAGE_OUT_HANDOFF, else -1 */
  uint32_t oversize;         /* 1: payload is a one-off allocation of a split
                                (chunked) capture, freed on return */
} tf_paged_batch;
int tf_stager_next(tf_stager* st, double timeout_s, tf_paged_batch* out);
/* Return a batch obtained from tf_stager_next (payload back to the pool). */
int tf_stager_free_paged(tf_stager* st, tf_paged_batch* batch);
int tf_stager_note_sunk(tf_stager* st, uint64_t bytes);
int tf_stager_stats_get(tf_stager* st, tf_stager_stats* out);
int tf_stager_error(tf_stager* st);       /* first background error, 0 if none */
/* The staging stream (cudaStream_t) the D2H work is issued on. */
int tf_stager_stream(tf_stager* st, void** stream);
/* Placement of one replica's staging engine: the CPUs its threads are bound
   to (the GPU's PCIe-local CPUs, sysfs local_cpulist) and the NUMA node of
   its pinned pool (-1 unknown). No reference analogue. */
int tf_stager_placement(tf_stager* st, int32_t* cpus, uint32_t max_cpus,
                        uint32_t* n_cpus, int32_t* pool_node);
void tf_free_host(void* p);

/* ---- measurement helpers (bench) ------------------------------------- */
/* Pinned D2H bandwidth of one cudaMemcpyAsync of nbytes, best of reps. */
int tf_measure_d2h(int device, uint64_t nbytes, int reps, double* gbps);
/* Wall-clock of monotonic seconds (same clock the stager uses). */
double tf_monotonic(void);

/* ---- native record sinks (SRC/sinks.py:35-136 formats) ----------------
 * Replace FileSink.write / StreamSink.write (SRC/sinks.py:53-66, 117-126)
 * for the exporter's hot path: one call per batch of captures, each
 * capture the matched TensorMeta (SRC/records.py:22-60) plus its payload in
 * host memory (a staging buffer). The sink splits each payload into
 * per-request records in batch order (SRC/exporter.py:306-327), computes
 * zlib crc32 per record on a thread pool, formats the reference's NDJSON
 * header byte-for-byte (fixed key order, compact separators, ASCII
 * escapes) and writes the sidecar / frames with large writes. The calling
 * thread never touches payload bytes in Python. */
typedef struct tf_capture_meta {
  const char* hook_name;        /* NUL-terminated */
  int64_t layer;                /* -1: null */
  int64_t step_seq;
  int64_t tp_rank, pp_stage;
  const char* dtype;            /* dtype name, NUL-terminated */
  uint32_t n_req;
  uint32_t ndim;                /* per-request shape rank (>= 1) */
  const int64_t* request_ids;   /* n_req */
  const int64_t* token_ranges;  /* 2 * n_req: [start, end) pairs */
  const int64_t* row_counts;    /* n_req (ragged: shape[0] per request) or NULL */
  const int64_t* shape;         /* ndim: per-request shape (uniform case) */
  int64_t row_bytes;            /* bytes per shape[0] row */
  const uint8_t* payload;       /* host memory, payload_len bytes */
  uint64_t payload_len;
} tf_capture_meta;

typedef struct tf_sink tf_sink;
/* records.ndjson + records.bin in `dir` (appended, like FileSink). */
int tf_sink_open_dataset(const char* dir, uint32_t threads, tf_sink** out);
/* flags: TF_SINK_DIRECT writes records.bin with O_DIRECT through aligned
   bounce buffers (fallocate'd ahead, trimmed at close) where the filesystem
   supports it, else buffered; tf_sink_is_direct tells which. */
#define TF_SINK_DIRECT 0x1u
int tf_sink_open_dataset2(const char* dir, uint32_t threads, uint32_t flags, tf_sink** out);
int tf_sink_is_direct(tf_sink* s);
/* u32-LE framed (header, payload) records on an open file descriptor. */
int tf_sink_open_stream(int fd, uint32_t threads, tf_sink** out);
int tf_sink_write(tf_sink* s, const tf_capture_meta* caps, uint32_t n_caps);
int tf_sink_stats(tf_sink* s, uint64_t* records, uint64_t* bytes);
int tf_sink_flush(tf_sink* s);   /* fsync-free: data handed to the kernel */
/* zlib.crc32(data, crc) as the sinks compute it (PCLMULQDQ folding, zlib
   fallback); records.py / SRC/records.py checksum semantics */
uint32_t tf_sink_crc32(uint32_t crc, const void* data, uint64_t n);
int tf_sink_close(tf_sink* s);   /* closes the files it opened, not a caller fd */

#ifdef __cplusplus
}
#endif
#endif /* RING2_H_ */
