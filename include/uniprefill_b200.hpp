// uniprefill_b200.hpp -- C++ host mirror of the reference operator API over the C ABI.
//
// The reference ships its hot path as the C++ namespace `uniprefill`
// (/root/reference/proj/core/include/uniprefill/*.hpp) over host matrices, throwing
// ConfigError / ContractViolation (errors.hpp:13-42).  This header keeps those names,
// argument meanings and error behaviour for device-resident varlen batches:
//
//   uniprefill::b200::ScoreConfig          <- ScoreConfig            (config.hpp:53-63)
//   uniprefill::b200::score_blocks         <- score_tokens[_heads]   (importance.hpp:42-47)
//   uniprefill::b200::reduce_block_scores  <- allreduce_scores       (tp_sim.hpp:31)
//   uniprefill::b200::top_p_select         <- top_p_select           (selection.hpp:53-54)
//   uniprefill::b200::compact              <- apply_drop / patch_metadata
//                                             (propagation.hpp:415, scheduler.hpp:52-53)
//   uniprefill::b200::DropLayer            <- prefill_layer_step's drop section
//                                             (propagation.cpp:163-202)
//
// All work is enqueued on the given stream; nothing synchronizes except check_device().
// Header-only; link libuniprefill_b200.so and cudart.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "uniprefill_b200.h"

namespace uniprefill::b200 {

class ConfigError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ContractViolation : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class UnsupportedError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class AllocationMissError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(up_status s, const char* what) {
    if (s == UP_OK) return;
    const std::string msg = std::string(what) + ": " + up_status_string(s);
    switch (s) {
    case UP_ERR_CONFIG: throw ConfigError(msg);
    case UP_ERR_CONTRACT: throw ContractViolation(msg);
    case UP_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    case UP_ERR_CUDA: throw CudaError(msg);
    case UP_ERR_ALLOCATION_MISS: throw AllocationMissError(msg);
    default: throw std::runtime_error(msg);
    }
}

struct ScoreConfig {
    int query_window_n = 128;
    int block_size_g = 64;
    int sink_count_a = 128;
    float top_p = 0.99f;

    up_score_config c() const { return {query_window_n, block_size_g, sink_count_a, top_p}; }
    /// ScoreConfig::validate (config.cpp:98-103): throws ConfigError.
    void validate() const {
        const up_score_config x = c();
        check(up_config_validate(&x), "ScoreConfig::validate");
    }
};

/// Device-resident varlen batch (PackedBatch, scheduler.hpp:33-46).
struct VarlenBatch {
    int32_t num_requests = 0;
    int64_t max_tokens = 0;
    const int32_t* cu_seqlens = nullptr;    // device int32[R+1]
    const uint8_t* drop_enabled = nullptr;  // device uint8[R] or null
    up_batch c() const { return {num_requests, max_tokens, cu_seqlens, drop_enabled}; }
};

struct HeadLayout {
    int num_q_heads = 0, num_kv_heads = 0, head_dim = 0;
    int gqa_group = 1, q_head_offset = 0, kv_head_offset = 0;
    int64_t q_row_stride = 0, k_row_stride = 0;
    up_heads c() const {
        return {num_q_heads, num_kv_heads, head_dim, gqa_group, q_head_offset, kv_head_offset,
                q_row_stride ? q_row_stride : int64_t(num_q_heads) * head_dim,
                k_row_stride ? k_row_stride : int64_t(num_kv_heads) * head_dim};
    }
};

/// Device scratch shared by every entry point (zeroed once).
class Workspace {
public:
    Workspace() = default;
    Workspace(const VarlenBatch& b, const HeadLayout& h, const ScoreConfig& cfg) { reserve(b, h, cfg); }
    ~Workspace() { if (ptr_) cudaFree(ptr_); }
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;

    void reserve(const VarlenBatch& b, const HeadLayout& h, const ScoreConfig& cfg) {
        const up_batch bc = b.c();
        const up_heads hc = h.c();
        const up_score_config cc = cfg.c();
        const size_t need = up_workspace_bytes(&bc, &hc, &cc);
        if (need <= bytes_) return;
        if (ptr_) cudaFree(ptr_);
        if (cudaMalloc(&ptr_, need) != cudaSuccess || cudaMemset(ptr_, 0, need) != cudaSuccess)
            throw CudaError("Workspace: cudaMalloc failed");
        bytes_ = need;
    }
    void* data() const { return ptr_; }
    size_t bytes() const { return bytes_; }

private:
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

/// Block scores of every drop-enabled segment (importance.cpp:92-132 per segment).
inline void score_blocks(cudaStream_t s, const VarlenBatch& b, const HeadLayout& h, const ScoreConfig& cfg,
                         const void* q_bf16, const void* k_bf16, float* block_scores, int32_t* cu_blocks,
                         Workspace& ws, float* token_scores = nullptr) {
    const up_batch bc = b.c();
    const up_heads hc = h.c();
    const up_score_config cc = cfg.c();
    check(up_score_blocks(s, &bc, &hc, &cc, q_bf16, k_bf16, block_scores, cu_blocks, token_scores, ws.data(),
                          ws.bytes()),
          "score_blocks");
}

/// sharded_block_scores + allreduce_scores (tp_sim.cpp:12-49) in one call: shard t's
/// partials at shard_scores + t * shard_stride, their ascending-shard sum in block_scores.
inline void sharded_block_scores(cudaStream_t s, const VarlenBatch& b, const HeadLayout& h, const ScoreConfig& cfg,
                                 const void* q_bf16, const void* k_bf16, int tp_degree, float* shard_scores,
                                 int64_t shard_stride, float* block_scores, int32_t* cu_blocks, Workspace& ws) {
    const up_batch bc = b.c();
    const up_heads hc = h.c();
    const up_score_config cc = cfg.c();
    check(up_score_blocks_tp(s, &bc, &hc, &cc, q_bf16, k_bf16, tp_degree, shard_scores, shard_stride, block_scores,
                             cu_blocks, ws.data(), ws.bytes()),
          "sharded_block_scores");
}

/// allreduce_scores (tp_sim.cpp:29-49) over device-addressable shard partials.
inline void reduce_block_scores(cudaStream_t s, const std::vector<const float*>& shards, int64_t count,
                                float* out) {
    if (shards.empty()) throw ContractViolation("allreduce_scores: no shards");
    check(up_reduce_block_scores(s, shards.data(), static_cast<int32_t>(shards.size()), count, out),
          "reduce_block_scores");
}

/// top_p_select + expand_mask (+ veto) for every drop-enabled segment.
inline void top_p_select(cudaStream_t s, const VarlenBatch& b, const ScoreConfig& cfg, const float* block_scores,
                         const int32_t* cu_blocks, uint8_t* keep, const up_selection_out& out, Workspace& ws,
                         const uint8_t* veto = nullptr) {
    const up_batch bc = b.c();
    const up_score_config cc = cfg.c();
    check(up_select(s, &bc, &cc, block_scores, cu_blocks, veto, keep, &out, ws.data(), ws.bytes()),
          "top_p_select");
}

/// apply_drop / patch_metadata: compacts every plane, rebuilds cu_seqlens.
inline void compact(cudaStream_t s, const VarlenBatch& b, const uint8_t* keep, const std::vector<up_plane>& planes,
                    int32_t* cu_seqlens_out, int32_t* retained_index, int32_t* num_tokens_out, Workspace& ws) {
    const up_batch bc = b.c();
    check(up_compact(s, &bc, keep, planes.data(), static_cast<int32_t>(planes.size()), cu_seqlens_out,
                     retained_index, num_tokens_out, ws.data(), ws.bytes()),
          "compact");
}

/// compact() right after top_p_select() on the same workspace and keep mask: the
/// selection already counted the retained rows per tile (up_compact_selected).
inline void compact_selected(cudaStream_t s, const VarlenBatch& b, const uint8_t* keep,
                             const std::vector<up_plane>& planes, int32_t* cu_seqlens_out, int32_t* retained_index,
                             int32_t* num_tokens_out, Workspace& ws) {
    const up_batch bc = b.c();
    check(up_compact_selected(s, &bc, keep, planes.data(), static_cast<int32_t>(planes.size()), cu_seqlens_out,
                              retained_index, num_tokens_out, ws.data(), ws.bytes()),
          "compact_selected");
}

/// Reconstitution step (propagation.cpp:79-100): rows 0..*num_rows of every plane's src
/// go back to rows index[o] of its dst (up_compact's retained_index unwinds a drop).
inline void scatter_rows(cudaStream_t s, const int32_t* index, const int32_t* num_rows, int64_t max_rows,
                         const std::vector<up_plane>& planes) {
    check(up_scatter_rows(s, index, num_rows, max_rows, planes.data(), static_cast<int32_t>(planes.size())),
          "scatter_rows");
}

/// recompute_slots_after_drop (kvcache.cpp:147-158), Eq. 16: KV slots of the retained rows
/// for num_layers downstream layers from their block tables [L][R][max_pages].
inline void slot_mapping(cudaStream_t s, const VarlenBatch& compacted, const int32_t* num_rows, const int64_t* positions,
                         const int32_t* block_tables, int32_t num_layers, int32_t max_pages, int32_t block_size,
                         int64_t* slots, int64_t slot_stride, Workspace& ws) {
    check(up_slot_mapping(s, compacted.cu_seqlens, compacted.num_requests, num_rows, compacted.max_tokens, positions,
                          block_tables, num_layers, max_pages, block_size, slots, slot_stride, ws.data(), ws.bytes()),
          "slot_mapping");
}

/// decode_seqused (kvcache.cpp:182-186), Eq. 17, for every (layer, request).
inline void decode_seqused(cudaStream_t s, int32_t num_layers, int32_t num_requests, const int32_t* cu_orig,
                           const std::vector<int32_t>& drop_layers, const std::vector<const int32_t*>& cu_after,
                           const int32_t* decode_appended, int32_t* seqused) {
    if (drop_layers.size() != cu_after.size()) throw ContractViolation("decode_seqused: one cu_seqlens per drop");
    check(up_decode_seqused(s, num_layers, num_requests, cu_orig, static_cast<int32_t>(drop_layers.size()),
                            drop_layers.data(), cu_after.data(), decode_appended, seqused),
          "decode_seqused");
}

/// TP all-reduce of partial block scores over peer memory (allreduce_scores,
/// tp_sim.cpp:29-49): peer_buffers[t] = rank t's exchange buffer mapped here (up_ipc_*).
inline void peer_allreduce_scores(cudaStream_t s, const float* partial, int64_t count, int32_t rank,
                                  const std::vector<void*>& peer_buffers, int64_t capacity, float* out,
                                  Workspace& ws) {
    check(up_peer_allreduce_scores(s, partial, count, rank, static_cast<int32_t>(peer_buffers.size()),
                                   peer_buffers.data(), capacity, out, ws.data(), ws.bytes()),
          "peer_allreduce_scores");
}

/// This TP rank's heads scored with the all-reduce fused into the combine kernel
/// (sharded_block_scores + allreduce_scores across GPUs, tp_sim.cpp:12-49).
inline void score_blocks_peer(cudaStream_t s, const VarlenBatch& b, const HeadLayout& h, const ScoreConfig& cfg,
                              const void* q, const void* k, int32_t rank, const std::vector<void*>& peer_buffers,
                              int64_t capacity, float* block_scores, int32_t* cu_blocks, Workspace& ws) {
    const up_batch bc = b.c();
    const up_heads hc = h.c();
    const up_score_config cc = cfg.c();
    check(up_score_blocks_peer(s, &bc, &hc, &cc, q, k, rank, static_cast<int32_t>(peer_buffers.size()),
                               peer_buffers.data(), capacity, block_scores, cu_blocks, ws.data(), ws.bytes()),
          "score_blocks_peer");
}

/// attention_readout (model.cpp:215-263) at a drop layer (propagation.cpp:195-205): every
/// retained row of `compacted` attends to its segment's retained keys with position in
/// (pos - window, pos]; out bf16 [max_tokens][out_row_stride].
inline void attention_readout(cudaStream_t s, const VarlenBatch& compacted, const HeadLayout& h, const void* q,
                              const void* k, const void* v, const int64_t* positions, int64_t window, void* out,
                              int64_t out_row_stride, Workspace& ws) {
    const up_batch b = compacted.c();
    const up_heads hc = h.c();
    check(up_attention_varlen(s, &b, &hc, q, k, v, positions, window, out,
                              out_row_stride ? out_row_stride : int64_t(h.num_q_heads) * h.head_dim, ws.data(),
                              ws.bytes()),
          "attention_readout");
}

/// Synchronizes and raises the sticky device-side ContractViolation (NaN / negative block
/// scores, malformed cu_seqlens) like the reference's exceptions.
inline void check_device(cudaStream_t s, Workspace& ws) { check(up_device_status(s, ws.data()), "device"); }

}  // namespace uniprefill::b200
