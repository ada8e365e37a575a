/*
 * uniprefill_b200.h -- C ABI of the B200-native UniPrefill token-selection hot path.
 *
 * One entry point per reference operation on the path.  The reference
 * exposes a C++ namespace API over host matrices (/root/reference/proj/core/include/
 * uniprefill/*.hpp); this ABI replaces it for device-resident, continuous-batching varlen
 * batches indexed by cu_seqlens:
 *
 *   up_score_blocks        replaces score_tokens / score_tokens_heads
 *                          (importance.hpp:42-47, importance.cpp:17-132) and, through the
 *                          head range, sharded_block_scores (tp_sim.hpp:25-26)
 *   up_reduce_block_scores replaces allreduce_scores (tp_sim.hpp:31, tp_sim.cpp:29-49)
 *   up_peer_allreduce_scores  the same across a TP group of GPUs, over peer memory
 *                          for shard partials that are device-addressable from one GPU
 *   up_select              replaces top_p_select + expand_mask (selection.hpp:46-54,
 *                          selection.cpp:36-122) and the no-readmission veto
 *                          (restrict_selection, propagation.cpp:116-136, :173-183)
 *   up_compact             replaces apply_drop + gather_rows + patch_metadata
 *                          (propagation.cpp:47-77, :105-112; scheduler.cpp:50-90)
 *   up_drop_layer          the three above back to back (prefill_layer_step's
 *                          score -> select -> compact section, propagation.cpp:163-202)
 *
 * Conventions
 *   - Plain pointers and sizes only; every data pointer is DEVICE memory owned by the
 *     caller unless stated otherwise.  `stream` is a cudaStream_t (NULL = legacy stream).
 *   - All work is stream-ordered and asynchronous; no entry point synchronizes.
 *   - Shapes are data-dependent after a drop, so launch sizing never needs the segment
 *     lengths on the host: callers pass capacities (max_tokens) and the device-resident
 *     cu_seqlens.  The whole layer step can be captured in a CUDA graph.
 *   - Errors: host-detectable problems return a status immediately (ConfigError ->
 *     UP_ERR_CONFIG, ContractViolation -> UP_ERR_CONTRACT, errors.hpp:13-42).  Problems
 *     only visible on the device (negative / non-finite block scores, malformed
 *     cu_seqlens) raise a sticky flag in the workspace; up_device_status() reads and
 *     clears it.  No exception crosses the ABI.
 *   - Re-entrant: distinct workspaces may be used concurrently on distinct streams.
 */
#ifndef UNIPREFILL_B200_H
#define UNIPREFILL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UP_ABI_VERSION 3

typedef enum {
    UP_OK = 0,
    UP_ERR_CONFIG = 1,         /* ConfigError (errors.hpp:15-18) */
    UP_ERR_CONTRACT = 2,       /* ContractViolation (errors.hpp:22-25) */
    UP_ERR_UNSUPPORTED = 3,    /* valid input outside the implemented envelope */
    UP_ERR_WORKSPACE = 4,      /* workspace missing or too small */
    UP_ERR_CUDA = 5,           /* CUDA runtime / driver failure */
    UP_ERR_INVALID_ARGUMENT = 6,
    UP_ERR_ALLOCATION_MISS = 7  /* AllocationMissError (errors.hpp:32-35) */
} up_status;

/* ScoreConfig (config.hpp:53-63).  Defaults: n=128, G=64, A=128, p=0.99. */
typedef struct {
    int32_t query_window_n; /* n: last-n query rows per request */
    int32_t block_size_g;   /* G: tokens per selection block */
    int32_t sink_count_a;   /* A: always-kept attention sinks */
    float top_p;            /* p in (0, 1] */
} up_score_config;

/* A continuous-batching varlen batch (PackedBatch, scheduler.hpp:33-46). */
typedef struct {
    int32_t num_requests;        /* R >= 1 */
    int64_t max_tokens;          /* capacity: rows allocated in every [T, ...] buffer */
    const int32_t* cu_seqlens;   /* device int32[R+1]: 0 = cu[0] < cu[1] < ... <= max_tokens */
    const uint8_t* drop_enabled; /* device uint8[R] or NULL (all enabled).  0 marks a
                                    segment that passes through untouched (decode phase,
                                    scheduler.cpp:59-62) */
} up_batch;

/* Head layout of q / k as held by this rank.  Local q-head hl is global head
 * q_head_offset + hl and reads local kv-head (q_head_offset + hl) / gqa_group -
 * kv_head_offset.  With TP, a rank holds a contiguous head slice (tp_sim.cpp:12-27). */
typedef struct {
    int32_t num_q_heads;    /* q heads present in q */
    int32_t num_kv_heads;   /* kv heads present in k */
    int32_t head_dim;       /* D */
    int32_t gqa_group;      /* global Hq / Hkv (1 for MHA) */
    int32_t q_head_offset;  /* global index of local q-head 0 */
    int32_t kv_head_offset; /* global index of local kv-head 0 */
    int64_t q_row_stride;   /* elements between consecutive token rows of q (>= Hq*D) */
    int64_t k_row_stride;   /* elements between consecutive token rows of k (>= Hkv*D) */
} up_heads;

/* One row-major plane compacted by up_compact (hidden states, K, V, Q, positions ...). */
typedef struct {
    const void* src;  /* device, max_tokens rows */
    void* dst;        /* device, max_tokens rows (only the retained prefix is written) */
    int64_t row_bytes;
    int64_t src_stride_bytes; /* 0 = row_bytes */
    int64_t dst_stride_bytes; /* 0 = row_bytes */
} up_plane;

/* Per-request selection results (Selection, selection.hpp:34-57). */
typedef struct {
    int64_t* cutoff_rank;     /* int64[R]: k*, nb if degenerate, -1 for pass-through segments */
    int64_t* retained_count;  /* int64[R] (optional) */
    double* covered_mass;     /* double[R] (optional) */
    uint8_t* degenerate;      /* uint8[R] (optional): zero total mass -> keep-all */
} up_selection_out;

int up_abi_version(void);
const char* up_status_string(up_status status);

/* ScoreConfig::validate (config.cpp:98-103). */
up_status up_config_validate(const up_score_config* cfg);

/* Upper bound of Σ_r ceil(N_r / G) for any batch that fits the capacities. */
int64_t up_max_blocks(const up_batch* batch, const up_score_config* cfg);

/* Bytes of device workspace needed by every entry point for this batch capacity and head
 * layout (one workspace serves all of them).  The workspace must be zeroed once before
 * first use (cudaMemset) and then belongs to one stream at a time. */
size_t up_workspace_bytes(const up_batch* batch, const up_heads* heads, const up_score_config* cfg);

/* Importance scores per block (a3-a6).  q: bf16 [max_tokens, Hq_local, D] (row stride
 * q_row_stride), k: bf16 [max_tokens, Hkv_local, D].  Writes
 *   block_scores[Σ_r ceil(N_r/G)] fp32 (segment-major; zeros for pass-through segments)
 *   cu_blocks[R+1] int32 (block offsets of each segment),
 *   token_scores[max_tokens] fp32 when non-NULL (reference token_scores, importance.hpp:18-23).
 * block_scores holds the PARTIAL sum over this rank's heads; reduce over TP ranks before
 * up_select (Eq. 15). */
up_status up_score_blocks(void* stream, const up_batch* batch, const up_heads* heads,
                          const up_score_config* cfg, const void* q, const void* k,
                          float* block_scores, int32_t* cu_blocks, float* token_scores,
                          void* workspace, size_t workspace_bytes);

/* Head-sharded importance scores in one call: the local q-heads form tp contiguous
 * shards of Hq/tp heads (sharded_block_scores, tp_sim.cpp:12-27); writes every shard's
 * partial block scores to shard_scores[t * shard_stride + g] (shard_stride >=
 * up_max_blocks) and their elementwise sum in ascending shard order to block_scores
 * (allreduce_scores, tp_sim.cpp:29-49).  UP_ERR_CONFIG when tp <= 0 or Hq % tp != 0. */
up_status up_score_blocks_tp(void* stream, const up_batch* batch, const up_heads* heads,
                             const up_score_config* cfg, const void* q, const void* k, int32_t tp,
                             float* shard_scores, int64_t shard_stride, float* block_scores,
                             int32_t* cu_blocks, void* workspace, size_t workspace_bytes);

/* Elementwise sum of tp partial block-score vectors in ascending shard order
 * (allreduce_scores, tp_sim.cpp:43-47): out[g] = ((0 + s_0[g]) + s_1[g]) + ...
 * shards: HOST array of tp device pointers (peer-mapped or local). */
up_status up_reduce_block_scores(void* stream, const float* const* shards, int32_t tp,
                                 int64_t count, float* out);

/* Top-p keep mask (a9-a13).  block_scores / cu_blocks as produced by up_score_blocks
 * (after any TP reduction).  veto: device uint8[max_tokens] or NULL -- rows that may not
 * be re-admitted.  Writes keep[max_tokens] (1 = retained; pass-through segments all 1).
 * Stream-ordered: requests of more than 512 blocks are selected on a library-owned side
 * stream forked from and joined back into `stream` by events (capture-safe). */
up_status up_select(void* stream, const up_batch* batch, const up_score_config* cfg,
                    const float* block_scores, const int32_t* cu_blocks, const uint8_t* veto,
                    uint8_t* keep, const up_selection_out* out, void* workspace,
                    size_t workspace_bytes);

/* Segmented prefix sum + gather compaction (a14-a16).  Retained rows of every plane are
 * written contiguously in order (drop-enabled segments keep rows with keep != 0, the
 * others keep all rows).  Writes cu_seqlens_out[R+1], retained_index[num_out] (source row
 * of each output row; may be NULL) and *num_tokens_out (device int32). */
up_status up_compact(void* stream, const up_batch* batch, const uint8_t* keep,
                     const up_plane* planes, int32_t num_planes, int32_t* cu_seqlens_out,
                     int32_t* retained_index, int32_t* num_tokens_out, void* workspace,
                     size_t workspace_bytes);

/* up_compact for a keep mask that up_select just wrote on this workspace (same batch,
 * drop_enabled and stream, keep unmodified since): up_select's expansion already counted
 * the retained rows per tile, so the count pass is skipped (one launch fewer; what
 * up_drop_layer does). */
up_status up_compact_selected(void* stream, const up_batch* batch, const uint8_t* keep,
                              const up_plane* planes, int32_t num_planes, int32_t* cu_seqlens_out,
                              int32_t* retained_index, int32_t* num_tokens_out, void* workspace,
                              size_t workspace_bytes);

/* Row scatter, the inverse of up_compact's gather: for o < *num_rows (device int32; or
 * max_rows when num_rows is NULL) and index[o] >= 0, row o of every plane's src is copied
 * to row index[o] of its dst.  Passing up_compact's retained_index and num_tokens_out
 * writes the current compacted states back over their pre-drop rows, turning the pre-drop
 * buffer into the reconstituted stream (reconstitute, propagation.cpp:79-100; unwind the
 * drops of a block in reverse order).  Also re-admits parked rows at their positions.
 * dst may be pinned host memory (unified addressing): the kernel writes the scattered
 * rows in place over PCIe, the mirror of up_compact reading pinned host sources. */
up_status up_scatter_rows(void* stream, const int32_t* index, const int32_t* num_rows, int64_t max_rows,
                          const up_plane* planes, int32_t num_planes);

/* up_score_blocks -> up_select -> up_compact for a single-rank (non-TP) layer. */
up_status up_drop_layer(void* stream, const up_batch* batch, const up_heads* heads,
                        const up_score_config* cfg, const void* q, const void* k,
                        const uint8_t* veto, float* block_scores, int32_t* cu_blocks,
                        uint8_t* keep, const up_selection_out* sel, const up_plane* planes,
                        int32_t num_planes, int32_t* cu_seqlens_out, int32_t* retained_index,
                        int32_t* num_tokens_out, void* workspace, size_t workspace_bytes);

/* Eq. 16 slot mapping for downstream layers (recompute_slots_after_drop, kvcache.cpp:147-158;
 * slot_for, kvcache.cpp:67-80): for each row i < *num_rows (device; or max_rows when NULL)
 * of the compacted batch (segments from cu_seqlens, R of them) and each of num_layers layers,
 *   slots[l * slot_stride + i] = block_tables[(l * R + r_i) * max_pages + p_i / B] * B + p_i % B
 * with p_i = positions[i].  A page the table does not hold writes -1 and raises the sticky
 * UP_ERR_ALLOCATION_MISS flag (read by up_device_status). */
up_status up_slot_mapping(void* stream, const int32_t* cu_seqlens, int32_t num_requests, const int32_t* num_rows,
                          int64_t max_rows, const int64_t* positions, const int32_t* block_tables,
                          int32_t num_layers, int32_t max_pages, int32_t block_size, int64_t* slots,
                          int64_t slot_stride, void* workspace, size_t workspace_bytes);

/* Eq. 17 per-layer decode KV length (decode_seqused, kvcache.cpp:182-186):
 *   seqused[l * R + r] = len_k(r) + decode_appended[r]
 * where len_k is segment r's length in cu_after[k] (device cu_seqlens after drop event k,
 * HOST array of num_drops pointers) for the last drop with drop_layers[k] < l, else its
 * length in cu_orig.  drop_layers (HOST) strictly increasing; decode_appended may be NULL. */
up_status up_decode_seqused(void* stream, int32_t num_layers, int32_t num_requests, const int32_t* cu_orig,
                            int32_t num_drops, const int32_t* drop_layers, const int32_t* const* cu_after,
                            const int32_t* decode_appended, int32_t* seqused);

/* Attention readout over the retained rows of a drop layer (attention_readout,
 * model.cpp:215-263, as prefill_layer_step calls it after the selection,
 * propagation.cpp:195-205).  For every segment r of batch (its cu_seqlens describe the
 * COMPACTED rows, e.g. up_compact's cu_seqlens_out) and every local q-head, query row j
 * attends to the segment's rows i with positions[i] in (positions[j] - window, positions[j]]
 * (window <= 0: no lower bound):
 *   out[j, h, :] = Σ_i softmax_i(q[j,h,:]·k[i,kvh,:] / sqrt(D)) v[i,kvh,:]
 * q: bf16 [max_tokens, Hq_local, D] (heads->q_row_stride); k, v: bf16 [max_tokens,
 * Hkv_local, D] (both heads->k_row_stride); positions: int64, strictly increasing within
 * each segment; out: bf16 [max_tokens, Hq_local, D] (out_row_stride elements per row).
 * D in {64, 128, 256}.  A row with no visible key raises the sticky UP_ERR_CONTRACT
 * (model.cpp:237; read by up_device_status).  workspace: >= 256 bytes, zeroed once (the
 * shared workspace of the other entry points will do); the persistent D <= 128 kernel keeps
 * its work-item counter in bytes [128, 136) and returns it to 0 on exit. */
up_status up_attention_varlen(void* stream, const up_batch* batch, const up_heads* heads, const void* q,
                              const void* k, const void* v, const int64_t* positions, int64_t window,
                              void* out, int64_t out_row_stride, void* workspace, size_t workspace_bytes);

/* ---- TP score all-reduce over peer memory (NVLink P2P / NVSwitch) ----------------------
 * allreduce_scores (tp_sim.cpp:29-49) for a TP group of one process per GPU, as one kernel:
 * every rank stores its partial into row `rank` of every peer's exchange buffer (one of two
 * banks, alternating per call, so a fast rank's next call never overwrites rows a slow peer
 * is still summing), raises a
 * flag per peer, waits for the tp rows of its own buffer and sums them in ascending rank
 * order from 0.0f -- bitwise the reference's reduction on every rank (an NCCL sum is not).
 * Exchange buffers: one per rank from up_peer_buffer_alloc(tp, capacity) (zeroed), shared
 * with up_ipc_get_handle / up_ipc_open_handle (UP_IPC_HANDLE_BYTES opaque bytes, exchanged
 * by the host, e.g. over torch.distributed).  peer_buffers: HOST array of tp device
 * pointers valid in this process, [rank] = this rank's own buffer.  Every rank must issue
 * the same sequence of calls with the same count (<= capacity, the blocks of the batch);
 * CUDA-graph capturable (the rendezvous state lives on the device).  A peer that never
 * arrives raises the sticky UP_ERR_CUDA after ~2 s (read by up_device_status). */
#define UP_IPC_HANDLE_BYTES 64
size_t up_peer_buffer_bytes(int32_t tp, int64_t capacity);
up_status up_peer_buffer_alloc(int32_t tp, int64_t capacity, void** buffer);
up_status up_peer_buffer_free(void* buffer);
up_status up_ipc_get_handle(const void* buffer, void* handle);
up_status up_ipc_open_handle(const void* handle, void** buffer);
up_status up_ipc_close_handle(void* buffer);
up_status up_peer_allreduce_scores(void* stream, const float* partial, int64_t count, int32_t rank, int32_t tp,
                                   void* const* peer_buffers, int64_t capacity, float* out, void* workspace,
                                   size_t workspace_bytes);

/* up_score_blocks over this rank's head slice (heads->q_head_offset / kv_head_offset) FUSED
 * with the TP all-reduce over peer memory: the block-combine kernel stores every block's
 * partial straight into the peers' exchange buffers and, after the rendezvous, writes the
 * ascending-rank sum to block_scores -- sharded_block_scores + allreduce_scores
 * (tp_sim.cpp:12-49) across GPUs in the scorer's own launches.  capacity >= the batch's
 * blocks (up_max_blocks).  Off the tensor-core envelope: the SIMT scorer, then
 * up_peer_allreduce_scores over up_max_blocks entries. */
up_status up_score_blocks_peer(void* stream, const up_batch* batch, const up_heads* heads,
                               const up_score_config* cfg, const void* q, const void* k, int32_t rank, int32_t tp,
                               void* const* peer_buffers, int64_t capacity, float* block_scores,
                               int32_t* cu_blocks, void* workspace, size_t workspace_bytes);

/* Synchronizes `stream`, returns the sticky device-side status raised since the last call
 * (UP_OK if none) and clears it. */
up_status up_device_status(void* stream, void* workspace);

/* Which scorer implementation up_score_blocks uses for this shape: 1 = tcgen05 tensor-core
 * kernel, 2 = SIMT kernel (generic shapes or when token_scores are requested). */
int up_scorer_kind(const up_heads* heads, const up_score_config* cfg, int want_token_scores);

/* Kernel launches issued by the most recent entry point on this thread (for accounting). */
int up_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* UNIPREFILL_B200_H */
