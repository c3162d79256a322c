/* hps_c.h -- C ABI of the B200-native embedding lookup+update path.
 *
 * Drop-in boundary for the reference's embedding-worker / parameter-server
 * operator API (/root/reference/proj/include/hybridps). Every entry point takes
 * plain pointers and sizes; none throws. The reference has no FFI of its own,
 * so each function cites the C++ member it replaces. A C++ adapter with the
 * reference's class shapes (PsShard / ShardSet / EmbeddingWorker) sits on top
 * of this header in include/hps/compat.hpp; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Status codes map 1:1 onto the reference's exception types
 *    (errors.hpp:28-107); HPS_E_CUDA reports a CUDA runtime failure.
 *  - Batch functions take DEVICE or HOST pointers; the kind is detected per
 *    pointer (cudaPointerGetAttributes). Host inputs are staged through pinned
 *    buffers inside the library, host outputs are copied back before return.
 *  - `stream` is a cudaStream_t (NULL = the legacy default stream). Calls that
 *    must report a data-dependent error (non-finite gradient, capacity) are
 *    synchronous unless HPS_ASYNC is passed, in which case the error surfaces
 *    from the next hps_table_sync().
 *  - A table holds S logical shards (route_shard(id, S) = mix64(id) % S,
 *    core.hpp:145-150) with one init salt per shard (PsShardConfig::rng_salt,
 *    embedding_ps.hpp:41-46). With world_size > 1 a table holds the shards
 *    s with s % world_size == owner_rank; see hps_shard_* below.
 */
#ifndef HPS_C_H
#define HPS_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define HPS_ABI_VERSION 2

typedef enum hps_status {
  HPS_OK = 0,
  HPS_E_PRECONDITION = 1,      /* PreconditionError      errors.hpp:28 */
  HPS_E_CONFIG = 2,            /* ConfigError            errors.hpp:35 */
  HPS_E_PROTOCOL = 3,          /* ProtocolError          errors.hpp:42 */
  HPS_E_TRANSPORT = 4,         /* TransportError         errors.hpp:49 */
  HPS_E_CHECKPOINT_CORRUPT = 5,/* CheckpointCorruptError errors.hpp:56 */
  HPS_E_DIVERGENCE = 6,        /* DivergenceError        errors.hpp:62 */
  HPS_E_CONSISTENCY = 7,       /* ConsistencyError       errors.hpp:68 */
  HPS_E_UNDEFINED_METRIC = 8,  /* UndefinedMetricError   errors.hpp:74 */
  HPS_E_STALE_SAMPLE = 9,      /* StaleSampleError       errors.hpp:80 */
  HPS_E_BACKPRESSURE = 10,     /* BackpressureError      errors.hpp:86 */
  HPS_E_CLOCK = 11,            /* ClockError             errors.hpp:92 */
  HPS_E_SYNC_FAILURE = 12,     /* SyncFailureError       errors.hpp:98 */
  HPS_E_UNRECOVERABLE = 13,    /* UnrecoverableRunError  errors.hpp:104 */
  HPS_E_CUDA = 100             /* CUDA runtime / launch failure */
} hps_status;

typedef enum hps_optimizer { HPS_ADAGRAD = 0, HPS_SGD = 1 } hps_optimizer; /* EmbOptimizer, embedding_ps.hpp:37 */
typedef enum hps_aggregation { HPS_MEAN = 0, HPS_SUM = 1 } hps_aggregation; /* ModelConfig::Aggregation, core.hpp:178 */

/* flags */
#define HPS_ASYNC 1u   /* do not synchronise to report data-dependent errors */
/* push: take the step tag from the table's device step counter (+1) and advance it
 * after the update, so a push captured once in a CUDA graph tags every replay with a
 * new step (the step_tag argument is ignored). hps_table_device_step reads it. */
#define HPS_DEVICE_STEP 2u

typedef void* hps_stream; /* cudaStream_t */

typedef struct hps_table hps_table;
typedef struct hps_batch hps_batch;

typedef struct hps_table_cfg {
  uint32_t shard_count;        /* logical shards S (ShardSet(shard_count, ...), embedding_ps.hpp:506) */
  const uint64_t* shard_salts; /* S per-shard init salts (host pointer) */
  uint64_t capacity;           /* rows this device may hold (sum over its owned shards) */
  uint32_t embedding_dim;      /* PsShardConfig::embedding_dim */
  int32_t optimizer;           /* hps_optimizer */
  int32_t device;              /* CUDA ordinal; -1 = current device */
  uint32_t owner_rank;         /* 0 for a single-device table */
  uint32_t world_size;         /* 1 for a single-device table */
  uint32_t flags;              /* HPS_TABLE_* */
  uint32_t reserved0;          /* 0 */
  uint64_t shard_capacity;     /* HPS_TABLE_LRU: rows per logical shard (PsShardConfig::capacity) */
} hps_table_cfg;

/* Table flags.
 * HPS_TABLE_TAG_RING: keep every row's 16-deep ring of version-bump step tags
 *   (PsShard::tag_ring_, embedding_ps.hpp:493-494; one 4-byte store per bump), so
 *   count_delay is exact for any order of step tags and for tracked writes after
 *   untracked ones (apply_gradients_map). Without it each row keeps its latest bump tag
 *   only -- exact for in-order tags, which every stream-ordered pipeline produces -- and
 *   a tracked apply it could not count exactly (a step tag older than one the table
 *   already applied, or any tracked apply after an untracked write since the last
 *   clear) is refused with HPS_E_CLOCK before anything mutates. */
#define HPS_TABLE_TAG_RING 1u
/* HPS_TABLE_LRU: every logical shard holds at most shard_capacity rows and evicts its
 *   least-recently-used row when a miss finds it full (LruStore::put lru_store.hpp:86-113,
 *   PsShard::find_or_init embedding_ps.hpp:417-434): exact LRU order over the PS surface
 *   (hps_lookup / hps_table_gather / hps_apply, touches in array order); evictions and
 *   clock resets counted like PsShard. A call that fits the shards' free rows runs the
 *   parallel kernels; one that must evict runs a sequential device path (one warp walks
 *   the call's entries in order). The embedding-worker batch surface and the exchange
 *   refuse LRU tables (HPS_E_PRECONDITION). capacity is then shard_count * shard_capacity. */
#define HPS_TABLE_LRU 2u

typedef struct hps_counters {
  uint64_t misses;            /* PsShard::miss_count          embedding_ps.hpp:79 */
  uint64_t evictions;         /* PsShard::eviction_count      embedding_ps.hpp:75 (HPS_TABLE_LRU) */
  uint64_t clock_resets;      /* PsShard::clock_reset_count   embedding_ps.hpp:83 */
  uint64_t stale_epoch_drops; /* PsShard::stale_epoch_drops   embedding_ps.hpp:87 */
  uint64_t size;              /* PsShard::size                embedding_ps.hpp:95 */
  uint64_t capacity;
  uint32_t epoch;             /* PsShard::epoch               embedding_ps.hpp:91 */
  uint32_t max_delay;         /* largest staleness delay recorded (StalenessStats) */
  uint64_t delay_hist[17];    /* delays 0..15, >=16 (StalenessStats::record_delay, staleness.hpp:42-49) */
} hps_counters;

/* ---- errors / version ---------------------------------------------------------------- */
const char* hps_last_error(void);   /* thread-local message of the last failing call */
int hps_abi_version(void);

/* ---- hashing / routing (core.hpp:36-44, 145-150) ------------------------------------ */
uint64_t hps_mix64(uint64_t x);
uint32_t hps_route_shard(uint64_t id, uint32_t shard_count);
/* Device: out_shard[i] = route_shard(ids[i], S). */
hps_status hps_route(const uint64_t* ids, size_t n, uint32_t shard_count, uint32_t* out_shard,
                     hps_stream stream);

/* ---- table lifecycle (PsShard(cfg) embedding_ps.hpp:63, ShardSet embedding_ps.hpp:506) */
hps_status hps_table_create(const hps_table_cfg* cfg, hps_table** out);
hps_status hps_table_destroy(hps_table* t);
hps_status hps_table_counters(hps_table* t, hps_counters* out);
hps_status hps_table_sync(hps_table* t); /* drain async work, report deferred errors */
uint32_t hps_table_epoch(const hps_table* t);            /* PsShard::epoch         :91 */
hps_status hps_table_device_step(hps_table* t, uint32_t* out_step); /* HPS_DEVICE_STEP counter */
uint32_t hps_table_advance_epoch(hps_table* t);          /* PsShard::advance_epoch :204 */
hps_status hps_table_reset(hps_table* t);                /* PsShard::reset_for_recovery :193 */

/* ---- checkpoints (PsShard::save_checkpoint / load_checkpoint / recover_from_checkpoint,
 * embedding_ps.hpp:209-402): HPS1 images, one per logical shard ------------------------- */
/* The HPS1 image of logical shard `shard`: the reference's 64-byte header (magic, format
 * 1, optimizer, dim, capacity, salt, hwm, recency head/tail, free head, live count, epoch,
 * evictions, FNV-1a checksum) and flat arrays ids, prev, next, versions, rows [w|acc].
 * Rows are listed in slot (first insertion) order; the recency chain runs from the newest
 * slot (head) to the oldest (tail). shard_capacity goes into the header (0 = the table's
 * capacity). *out_bytes = image size; the image is written when buf != NULL and
 * cap >= *out_bytes. Synchronises the device. */
hps_status hps_table_checkpoint_save(hps_table* t, uint32_t shard, uint32_t shard_capacity,
                                     void* buf, uint64_t cap, uint64_t* out_bytes);
/* Adopt `count` HPS1 images (host buffers) as the table's whole content: every image is
 * validated first like PsShard::parse + LruStore::restore (magic, format, checksum,
 * optimizer and dim vs the table, length, recency chain and free list) and matched to a
 * shard by its salt -- any failure returns HPS_E_CHECKPOINT_CORRUPT / HPS_E_CONFIG and
 * changes nothing. Then the table is cleared and the images' live rows (weights,
 * accumulators, versions; latest-bump tags reset, adopt_locked :390-402) inserted.
 * recover = 0: load_checkpoint (epoch = the images' epoch); 1: recover_from_checkpoint
 * (epoch = max(live, image) + 1, so in-flight pushes of the old epoch are dropped). */
hps_status hps_table_checkpoint_load(hps_table* t, const void* const* images,
                                     const uint64_t* sizes, uint32_t count, int recover);

/* ---- parameter-server surface --------------------------------------------------------- */
/* PsShard::lookup (embedding_ps.hpp:105-114) / ShardSet::lookup (:531-541): duplicates
 * allowed, misses lazily initialised (find_or_init :417-434). out_values[n*D];
 * out_versions[n] optional. */
hps_status hps_lookup(hps_table* t, const uint64_t* ids, size_t n, float* out_values,
                      uint64_t* out_versions, hps_stream stream);

/* hps_lookup with flags: HPS_ASYNC defers the capacity report to hps_table_sync (no host
 * round trip; used by the owner side of the multi-GPU exchange). */
hps_status hps_table_gather(hps_table* t, const uint64_t* ids, size_t n, float* out_values,
                            uint64_t* out_versions, uint32_t flags, hps_stream stream);

/* PsShard::apply_gradients (embedding_ps.hpp:139-162), array-shaped: entry i carries
 * ids[i], grads[i*D..], read_versions[i]. Epoch fence first (*accepted = 0, nothing
 * applied, stale_epoch_drops += n); then every gradient is validated finite before
 * anything mutates (HPS_E_DIVERGENCE otherwise); then entries apply in array order
 * (rows with repeated ids see them in that order). read_versions == NULL selects the
 * untracked map-shaped surface (apply_gradients_map :165-189: version += 1 per write).
 * out_delays[n] optional (per entry, reference count_delay :454-480). */
hps_status hps_apply(hps_table* t, const uint64_t* ids, const float* grads,
                     const uint64_t* read_versions, size_t n, float lr, uint32_t step_tag,
                     uint32_t epoch, uint32_t* out_delays, int* accepted, uint32_t flags,
                     hps_stream stream);

/* Test/checkpoint hook: read rows without lazy init or touching (present[i] = 0 if absent).
 * Any output may be NULL. */
hps_status hps_peek(hps_table* t, const uint64_t* ids, size_t n, float* out_w, float* out_acc,
                    uint64_t* out_versions, uint8_t* out_present, hps_stream stream);

/* ---- embedding-worker surface (batch-shaped) ----------------------------------------- */
/* A batch is B samples x F feature groups in CSR form: ids[N], offsets[B*F+1] (uint32,
 * sample-major, group-minor; IdFeatures core.hpp:129-131). Groups may be empty and
 * may list an id more than once.
 *
 * hps_batch_register  ~ EmbeddingWorker::register_sample (embedding_worker.hpp:493) for
 *                       B samples: routes, probes/lazily inits every id and builds the
 *                       per-row apply order once; sample_keys[B] (SampleId.raw) fixes the
 *                       apply order (ascending), NULL = batch order.
 * hps_batch_pull      ~ EmbeddingWorker::serve_pull (:523-571): out_pooled[B*F*D],
 *                       out_read_versions[N] (optional, per listing).
 * hps_batch_push      ~ apply_backward + gated flush (:575-594, :777-801): grads[B*F*D];
 *                       per sample in apply order, one optimizer application per (sample,
 *                       unique id) carrying the fp64 chain-rule sum (push_to_shards
 *                       :726-775). read versions come from the last hps_batch_pull of this
 *                       batch (tracked) unless untracked = 1. Whole-batch validation
 *                       precedes mutation. out_delays must be NULL (HPS_E_PRECONDITION
 *                       otherwise): the push's delays are recorded per (sample, id) in
 *                       hps_counters.delay_hist (StalenessStats::record_delay
 *                       staleness.hpp:42-49); hps_apply returns per-entry delays.
 */
hps_status hps_batch_create(hps_table* t, int32_t aggregation, hps_batch** out); /* EmbeddingWorkerConfig::aggregation */
hps_status hps_batch_destroy(hps_batch* b);
hps_status hps_batch_register(hps_batch* b, const uint64_t* ids, size_t n_ids,
                              const uint32_t* offsets, uint32_t B, uint32_t F,
                              const uint64_t* sample_keys, hps_stream stream);
/* Pipelines that register the next batch beside the current step: with on != 0 the
 * batch's plan (its sort, running on an internal stream beside the register) is joined by
 * the batch's push -- not by the register or the pull, which do not need it -- so the
 * next pooling does not wait for it. Inside a CUDA-graph capture the caller then owns the
 * join: the push in the same capture joins it, and a capture that ends before the push
 * must call hps_batch_join_plan(b, s) on one of its streams first. */
hps_status hps_batch_defer_plan_join(hps_batch* b, int on);
hps_status hps_batch_join_plan(hps_batch* b, hps_stream stream);
hps_status hps_batch_pull(hps_batch* b, float* out_pooled, uint64_t* out_read_versions,
                          hps_stream stream);
hps_status hps_batch_push(hps_batch* b, const float* grads, float lr, uint32_t step_tag,
                          uint32_t epoch, int untracked, uint32_t* out_delays, int* accepted,
                          uint32_t flags, hps_stream stream);
/* Number of (sample, unique id) applications the last push performed (delays length). */
hps_status hps_batch_pairs(hps_batch* b, uint64_t* out_pairs);

/* Stateless one-shot forms (register + pull / register + push). */
hps_status hps_pull_batch(hps_table* t, const uint64_t* ids, size_t n_ids, const uint32_t* offsets,
                          uint32_t B, uint32_t F, int32_t aggregation, float* out_pooled,
                          uint64_t* out_read_versions, hps_stream stream);
hps_status hps_push_batch(hps_table* t, const uint64_t* ids, size_t n_ids, const uint32_t* offsets,
                          uint32_t B, uint32_t F, int32_t aggregation, const float* grads,
                          const uint64_t* read_versions, const uint64_t* sample_keys, float lr,
                          uint32_t step_tag, uint32_t epoch, int* accepted, hps_stream stream);

/* ---- multi-GPU exchange (hash-sharded tables) -------------------------
 * A row is owned by rank route_shard(id, S) % world (ShardSet::shard_of,
 * embedding_ps.hpp:521-523, with the S logical shards spread round-robin over ranks); each
 * rank's table is created with all S salts and holds the rows it owns. One step of the
 * reference's E embedding workers in front of a ShardSet (EmbeddingWorker::fetch_rows
 * :677-704 / push_to_shards :726-775, PsShardService :185-290) becomes, per rank:
 *   hps_exchange_route    distinct ids of the batch grouped by owner rank
 *   [all-to-all ids]      -> owner: hps_lookup(recv ids) = rows + versions
 *   [all-to-all rows]     -> hps_exchange_pool: serve_pull's pooling over the rows
 *   hps_exchange_pairs    one contribution per (sample, distinct id), grouped by owner
 *   [all-to-all pairs]    -> owner: hps_table_apply_pairs, applied in (source rank, sample)
 *                            order = ascending SampleId (rank << 56 | counter)
 * All buffers are DEVICE pointers; counts are host arrays of `world` entries. The
 * collectives are the caller's (NCCL); paper_2111_05897_b200/sharded.py drives them. */
typedef struct hps_exchange hps_exchange;
hps_status hps_exchange_create(uint32_t world_size, uint32_t shard_count, int32_t aggregation,
                               int32_t device, hps_exchange** out);
hps_status hps_exchange_destroy(hps_exchange* x);
/* out_send_ids[n_ids] (first sum(out_counts) used, owner-major); out_counts[world]:
 * a host array (the call synchronises) or a device array (stays stream-ordered). */
hps_status hps_exchange_route(hps_exchange* x, const uint64_t* ids, size_t n_ids,
                              const uint32_t* offsets, uint32_t B, uint32_t F,
                              uint64_t* out_send_ids, uint64_t* out_counts, hps_stream stream);
/* rows[U*dim] = the owners' rows for send_ids, same order; out_pooled[B*F*dim]. */
hps_status hps_exchange_pool(hps_exchange* x, const float* rows, uint32_t dim, float* out_pooled,
                             hps_stream stream);
/* grads[B*F*dim]; out_pair_pos[P] = index of the pair's id inside its owner's segment of
 * send_ids; out_contrib[P*dim]; out_pair_counts[world] (host: synchronises; device: no).
 * Buffers sized for n_ids pairs. */
hps_status hps_exchange_pairs(hps_exchange* x, const float* grads, uint32_t dim,
                              uint32_t* out_pair_pos, float* out_contrib,
                              uint64_t* out_pair_counts, hps_stream stream);
/* Owner: recv_ids / recv_versions = the ids received by the forward exchange (source-rank
 * major, id_counts[world]) and the versions hps_lookup returned for them; the pairs
 * (pair_pos, contrib) received from each source (pair_counts[world]) apply through
 * PsShard::apply_gradients (:139-162): epoch fence, all-finite validation, ordered update,
 * version bump per step tag. recv_versions == NULL applies untracked. A pair position
 * outside its source's segment rejects the whole call (HPS_E_PROTOCOL, at once or, with
 * HPS_ASYNC, from hps_table_sync). */
hps_status hps_table_apply_pairs(hps_table* t, const uint64_t* recv_ids,
                                 const uint64_t* recv_versions, const uint64_t* id_counts,
                                 const uint32_t* pair_pos, const float* contrib,
                                 const uint64_t* pair_counts, uint32_t world, float lr,
                                 uint32_t step_tag, uint32_t epoch, int* accepted,
                                 uint32_t flags, hps_stream stream);

/* NVLink peer transport: the same step with every payload written once, directly into the
 * consumer's HBM over NVLink (CUDA IPC peer mappings), and device-side barriers instead of
 * collectives -- no NCCL on the data path, one host round trip per step (the owner's pair
 * count before its apply). Setup, once: hps_exchange_arena allocates this rank's receive
 * arena for batches of up to max_ids listings and returns its 64-byte IPC handle; the
 * caller all-gathers the handles and passes them (world x 64 bytes, rank order) to
 * hps_exchange_connect (max_groups >= B*F enables the owners' direct pooling of
 * one-listing groups). Per step, on every rank in the same order:
 *   hps_exchange_forward   route; ids -> owners' arenas; owners find-or-init and write the
 *                          rows into the requesters' arenas (= fetch_rows)
 *   hps_exchange_pool      with rows == NULL: pool from the delivered rows (= serve_pull)
 *   hps_exchange_backward  pairs -> owners' arenas; owners apply in (source rank, sample)
 *                          order (= apply_backward + flush_step + PsShard::apply_gradients)
 * A peer missing a barrier for ~4 s fails the step with HPS_E_SYNC_FAILURE instead of
 * hanging the device. */
/* Value codec on the NVLink payloads (opt-in, lossy): with kappa > 0
 * the owners' rows (PS pull replies, PsShardService(compress) embedding_worker.hpp:183-225)
 * and the sources' contributions (push frames, EmbeddingWorkerConfig::compress_values
 * :455,769) travel as kappa-scaled binary16 rows (compress_values codec.hpp:222-244, one
 * scale per row) and are decoded (decompress_values :246-261) before pooling / applying --
 * half the bytes on the wire. Every rank must use the same kappa; set before
 * hps_exchange_arena; 0 = exact fp32 payloads (default). dim: a power of two in [4, 128]. */
hps_status hps_exchange_set_codec(hps_exchange* x, float kappa);
hps_status hps_exchange_arena(hps_exchange* x, uint64_t max_ids, uint64_t max_groups,
                              uint32_t dim, void* out_handle);
/* hps_exchange_forward in two phases, so the next batch's routing and owner lookup can run
 * beside the current batch's backward: prefetch routes the batch (distinct ids into their
 * owners' id regions), plans its backward pairs, passes the first device barrier and
 * finds-or-inits the ids every source asked for (no existing row is read or written);
 * forward_prefetched delivers the rows and passes the second barrier. Every rank issues
 * both; phase 2 must follow this rank's previous backward on its stream and phase 1 must
 * be ordered before phase 2 (same stream, or joined). */
hps_status hps_exchange_prefetch(hps_exchange* x, hps_table* t, const uint64_t* ids, size_t n_ids,
                                 const uint32_t* offsets, uint32_t B, uint32_t F,
                                 hps_stream stream);
hps_status hps_exchange_forward_prefetched(hps_exchange* x, hps_table* t, hps_stream stream);
/* The arena's pooled buffer [max_groups][dim]: hps_exchange_pool(x, NULL, dim, NULL)
 * leaves the pooled batch there (zero-copy; valid until the next forward). The owners
 * write one-listing groups into it directly during the forward. */
hps_status hps_exchange_pooled(hps_exchange* x, float** out);
hps_status hps_exchange_connect(hps_exchange* x, uint32_t rank, const void* handles);
hps_status hps_exchange_forward(hps_exchange* x, hps_table* t, const uint64_t* ids, size_t n_ids,
                                const uint32_t* offsets, uint32_t B, uint32_t F,
                                hps_stream stream);
hps_status hps_exchange_backward(hps_exchange* x, hps_table* t, const float* grads, float lr,
                                 uint32_t step_tag, uint32_t epoch, int* accepted,
                                 uint32_t flags, hps_stream stream);

/* ---- instrumentation (no reference counterpart) ---------------------------------------- */
/* Kernels this library has launched in the process (proves which code ran). */
uint64_t hps_launch_count(void);
/* CUDA-event timing of named regions on the launching stream ("probe", "sort", "heads",
 * "pool", "check", "update"); enable resets the record. */
hps_status hps_profile_enable(hps_table* t, int enable);
hps_status hps_profile_get(hps_table* t, const char* region, double* total_ms, uint64_t* count);

/* ---- batch de-duplication (codec.hpp:123-182) ----------------------------------------- */
/* Sorted unique + inverse index over a flat id array: out_unique[u] ascending,
 * out_inverse[i] = index of ids[i] in out_unique; *out_u written (host pointer).
 * Device or host pointers. */
hps_status hps_dedup(const uint64_t* ids, size_t n, uint64_t* out_unique, uint32_t* out_inverse,
                     uint64_t* out_u, hps_stream stream);
/* The reference's lossy value codec, one block per row of block_len floats (codec.hpp:
 * 208-261; per embedding row on the wire, embedding_worker.hpp:48-85):
 * compress_values: out_scales[r] = kappa / ||row r||_inf (1.0 for an all-zero row),
 * out_payload[r*block_len + i] = binary16 bits of v*scale, round to nearest even
 * (float_to_half_bits :35-73) -- bit-identical to the reference. kappa <= 0 or a
 * non-finite input -> HPS_E_PRECONDITION. decompress_values: out = widened / scale; a
 * scale that is not finite and > 0, or a non-finite widened value -> HPS_E_PROTOCOL.
 * Host or device buffers; synchronises the stream (errors are reported). */
hps_status hps_compress_values(const float* values, uint64_t rows, uint32_t block_len,
                               float kappa, float* out_scales, uint16_t* out_payload,
                               hps_stream stream);
hps_status hps_decompress_values(const float* scales, const uint16_t* payload, uint64_t rows,
                                 uint32_t block_len, float* out, hps_stream stream);

/* compress_indices (codec.hpp:123-156): per group g, unique ids ascending
 * (unique[group_u_off[g] .. group_u_off[g+1]]) each with its ascending postings
 * (postings[post_off[k] .. post_off[k+1]], u16 sample indices, within-sample duplicates
 * collapsed). B > 65535 -> HPS_E_PRECONDITION. Buffers sized for N (worst case). */
hps_status hps_compress_indices(const uint64_t* ids, size_t n_ids, const uint32_t* offsets, uint32_t B,
                                uint32_t G, uint64_t* group_u_off, uint64_t* unique,
                                uint64_t* post_off, uint16_t* postings, hps_stream stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* HPS_C_H */
