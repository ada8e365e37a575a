/*
 * uniprefill_oracle.h -- CPU restatement of the UniPrefill token-selection hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 kernels in
 * paper_2605_06221_b200/csrc.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path never links it.
 *
 * Every function restates the reference C++ implementation under
 * /root/reference/proj/core/src (cited per function in uniprefill_oracle.c) in
 * plain C with the same arithmetic: fp32 storage, double accumulation, the same
 * summation orders, so that outputs match the reference bit for bit.  This is
 * checked against the reference itself (oracle/_ref, built from the reference
 * sources by oracle/Makefile) and against committed golden vectors in
 * tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Extension over the reference: GQA.  The reference is MHA-only;
 * q-head h reads kv-head h / (H / H_kv), which is exactly the reference run on K
 * with each kv-head's columns replicated H / H_kv times.
 */
#ifndef UNIPREFILL_ORACLE_H
#define UNIPREFILL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference exception classes (errors.hpp:13-42). */
enum {
    ORC_OK = 0,
    ORC_ERR_CONFIG = 1,   /* ConfigError */
    ORC_ERR_CONTRACT = 2, /* ContractViolation */
    ORC_ERR_ALLOCATION_MISS = 3, /* AllocationMissError */
};

/* ScoreConfig (config.hpp:53-63). */
typedef struct {
    int32_t query_window_n;
    int32_t block_size_g;
    int32_t sink_count_a;
    float top_p;
} orc_score_config;

/* Result of top_p_select for one request (selection.hpp:34-57). */
typedef struct {
    int64_t cutoff_rank;
    int64_t retained_count;
    double retention_ratio;
    double covered_mass;
    int32_t degenerate_keep_all;
} orc_selection_info;

int orc_config_validate(const orc_score_config* cfg);

/* phi / PackedScore (selection.cpp:14-34).  orc_phi_encode returns ORC_ERR_CONTRACT on
 * non-finite input and writes the encoding to *out. */
int orc_phi_encode(float x, uint32_t* out);
float orc_phi_decode(uint32_t bits);
int orc_pack_score(float score, uint32_t block_index, uint64_t* out);

/* splitmix64 counter RNG (rng.cpp:10-40), used for deterministic synthetic inputs. */
uint64_t orc_hash_mix(uint64_t x);
uint64_t orc_rng_key(uint64_t seed, uint64_t stream);
uint64_t orc_rng_bits(uint64_t key, uint64_t i);
double orc_rng_uniform(uint64_t key, uint64_t i);
float orc_rng_normal(uint64_t key, uint64_t i, double stddev);

/* out[j] = normal(first + j, stddev) for j < count (CounterRng::normal, rng.cpp:34-40). */
void orc_rng_normal_fill(uint64_t key, uint64_t first, int64_t count, double stddev, float* out);

/* Acceptance criterion 3's vector stream (acceptance_main.cpp:175-199): draws trial
 * `trial`'s scores (length returned, <= 4096; scores must hold 4096 floats) and top_p from
 * CounterRng(31, 0x6333) at the running counter *ctr, which it advances exactly as the
 * reference loop does.  Call for trial = 0, 1, 2, ... in order with one counter. */
int64_t orc_c3_vector(uint64_t* ctr, int trial, float* scores, float* top_p);

/* reference_blocks (acceptance_main.cpp:148-173) -- the independent stable-sort +
 * double-cumsum oracle of criterion 3 -- plus the forced one-token query window (:205-206),
 * as a keep mask of len bytes. */
void orc_c3_reference_blocks(const float* scores, int64_t len, double top_p, uint8_t* keep);

/* Importance scorer for one request (importance.cpp:17-132).
 *   q: N x (num_heads*head_dim) fp32 row-major with row stride q_ld (floats)
 *   k: N x (num_kv_heads*head_dim) fp32 row-major with row stride k_ld
 * Heads [head_begin, head_end) are scored; q-head h reads kv-head h / (num_heads/num_kv_heads).
 * token_scores: N floats (may be NULL); block_scores: ceil(N/G) floats. */
int orc_score_tokens_heads(const float* q, int64_t q_ld, const float* k, int64_t k_ld, int64_t N,
                           int num_heads, int num_kv_heads, int head_dim, int head_begin,
                           int head_end, const orc_score_config* cfg, float* token_scores,
                           float* block_scores, int32_t* effective_n);

/* block_reduce (importance.cpp:76-90). */
int orc_block_reduce(const float* token_scores, int64_t N, int block_size, float* out);

/* allreduce_scores (tp_sim.cpp:29-49): shards[t] has shard id shard_ids[t]; sum in
 * ascending id order in fp32. */
int orc_allreduce_scores(const float* const* shards, const int32_t* shard_ids, int32_t tp,
                         int64_t length, float* out);

/* expand_mask (selection.cpp:36-49). */
int orc_expand_mask(const uint8_t* block_mask, int64_t num_blocks, int block_size,
                    int64_t num_tokens, int64_t sink_count, int64_t window_n, uint8_t* keep);

/* top_p_select (selection.cpp:51-122).  keep: num_tokens bytes. */
int orc_top_p_select(const float* block_scores, int64_t num_blocks, const orc_score_config* cfg,
                     int64_t num_tokens, uint8_t* keep, orc_selection_info* info);

/* restrict_selection after a veto (propagation.cpp:116-136, applied at :173-183):
 * keep &= !veto, then retained/ratio/covered recomputed. */
int orc_restrict_selection(uint8_t* keep, const uint8_t* veto, int64_t num_tokens,
                           const float* block_scores, int64_t num_blocks, int block_size,
                           orc_selection_info* info);

/* patch_metadata + apply_drop row compaction over a varlen batch
 * (scheduler.cpp:50-90, propagation.cpp:47-77).  keep has T bytes; segments with
 * selected[s] == 0 pass through.  Each of n_planes row planes (row_bytes[p] bytes per
 * row) is compacted src -> dst.  Writes cu_out[R+1], retained_index (source rows), and
 * returns the retained count in *num_out. */
int orc_compact(const uint8_t* keep, const int64_t* cu_seqlens, int32_t num_requests,
                const uint8_t* selected, int32_t n_planes, const void* const* src,
                void* const* dst, const int64_t* row_bytes, int64_t* cu_out,
                int64_t* retained_index, int64_t* num_out);

/* reconstitute (propagation.cpp:79-100): the full-length stream of n_orig rows (row_bytes
 * each) -- row p = parked[k] for p = parked_pos[k], else the next active row in order. */
int orc_reconstitute(const void* active, const int64_t* active_pos, int64_t n_active, const void* parked,
                     const int64_t* parked_pos, int64_t n_parked, int64_t row_bytes, int64_t n_orig,
                     void* out);

/* PagedKVCache::slot_for (kvcache.cpp:67-80), Eq. 16: table[pos / B] * B + pos % B;
 * ORC_ERR_ALLOCATION_MISS when the page is absent (negative entry or past the table). */
int orc_slot_for(const int64_t* table, int64_t table_len, int block_size, int64_t pos, int64_t* slot);

/* decode_seqused (kvcache.cpp:182-186) / DropHistory::last_event_before (:32-39), Eq. 17. */
int64_t orc_decode_seqused(int64_t original_length, int64_t decode_appended, int32_t num_events,
                           const int32_t* event_layers, const int64_t* retained_lengths, int32_t layer);

/* Scoring FLOPs (flops.cpp:35-39): 2 * n_eff * N * D * H. */
uint64_t orc_scoring_flops(int64_t effective_n, int64_t num_keys, int head_dim, int num_heads);

#ifdef __cplusplus
}
#endif
#endif
