/* CPU restatement of the reference's embedding hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity oracle the CUDA path is checked against. It is plain C,
 * written from the reference's semantics, each function
 * citing the reference lines it restates. It is pinned against the reference
 * itself (oracle/_ref/libhps_ref.so, built from /root/reference headers) and
 * the reference's own known-answer tests (tests/test_oracle_pinning.py,
 * tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it; the product library (libhps.so) never links or calls it.
 */
#ifndef HPS_ORACLE_H
#define HPS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t orc_mix64(uint64_t x);
uint32_t orc_route_shard(uint64_t id, uint32_t shard_count);
void orc_init_row(uint64_t id, uint64_t shard_salt, uint32_t dim, float* out_w);

typedef struct orc_table orc_table;

/* opt: 0 Adagrad, 1 SGD. salts[S] per logical shard. */
orc_table* orc_table_create(uint32_t shard_count, const uint64_t* salts, uint32_t dim, int opt);
void orc_table_destroy(orc_table* t);
uint32_t orc_table_epoch(const orc_table* t);
uint32_t orc_table_advance_epoch(orc_table* t);
uint64_t orc_table_size(const orc_table* t);
/* counters[4]: misses, clock_resets, stale_epoch_drops, size */
void orc_table_counters(const orc_table* t, uint64_t* out4);

/* PsShard::lookup over the logical shard set. Lazily initialises misses. */
void orc_lookup(orc_table* t, const uint64_t* ids, size_t n, float* out_values,
                uint64_t* out_versions);
/* Read row state without touching it: present[i]=0 if absent. */
void orc_peek(const orc_table* t, const uint64_t* ids, size_t n, float* out_w, float* out_acc,
              uint64_t* out_versions, uint8_t* out_present);

/* PsShard::apply_gradients (tracked). Returns 0 ok, 6 divergence (nothing applied).
 * *accepted = 0 when epoch != table epoch (nothing applied). */
int orc_apply(orc_table* t, const uint64_t* ids, const float* grads, const uint64_t* read_versions,
              size_t n, float lr, uint32_t step_tag, uint32_t epoch, uint32_t* out_delays,
              int* accepted);
/* PsShard::apply_gradients_map (untracked; ids distinct). */
int orc_apply_map(orc_table* t, const uint64_t* ids, const float* grads, size_t n, float lr);

/* EmbeddingWorker::serve_pull for a CSR batch (offsets[B*F+1], sample-major).
 * agg: 0 mean, 1 sum. out_pooled[B*F*D]; out_read_versions[N] (may be NULL). */
void orc_pull_batch(orc_table* t, uint32_t B, uint32_t F, const uint64_t* ids,
                    const uint64_t* offsets, int agg, float* out_pooled,
                    uint64_t* out_read_versions);
/* EmbeddingWorker::apply_backward for a CSR batch, samples applied in ascending
 * sample_keys order (batch order when NULL). read_versions per listing or NULL
 * (untracked). Whole-batch validation precedes mutation. Returns 0 ok, 6 divergence.
 * *accepted = 0 when epoch is stale. out_delays (optional) receives, per sample in
 * apply order, per unique id in ascending id order, the reference delay. */
int orc_push_batch(orc_table* t, uint32_t B, uint32_t F, const uint64_t* ids,
                   const uint64_t* offsets, int agg, const float* grads,
                   const uint64_t* read_versions, const uint64_t* sample_keys, float lr,
                   uint32_t step_tag, uint32_t epoch, uint32_t* out_delays, uint64_t* out_n_delays,
                   int* accepted);

/* compress_indices (codec.hpp:123-156). Returns 0, or 1 (precondition: B > 65535).
 * group_u_off[G+1], unique[<=N], post_off[<=N+1], postings[<=N] */
int orc_compress_indices(uint32_t B, uint32_t G, const uint64_t* ids, const uint64_t* offsets,
                         uint64_t* group_u_off, uint64_t* unique, uint64_t* post_off,
                         uint16_t* postings);

#ifdef __cplusplus
}
#endif
#endif
