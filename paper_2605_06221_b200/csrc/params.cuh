// params.cuh -- kernel parameter blocks shared by the launchers (capi.cu) and kernels.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace up {

struct ScoreTcParams {
    const int32_t* cu_seqlens;
    const uint8_t* drop_enabled;
    const int32_t* cu_blocks;
    const int32_t* cu_chunks;
    const int32_t* cu_items;
    const int32_t* plan;
    float* P;
    float* stat_m;
    float* stat_l;
    int32_t num_requests;
    int32_t query_window_n;
    int32_t block_size_g;
    int32_t num_hgroups;
    int32_t q_head_offset;
    int32_t kv_head_offset;
    int32_t gqa_group;
    int64_t max_blocks;
    int64_t max_chunks;
    float scale_log2;  // log2(e) / sqrt(D)
};

struct ScoreSimtParams {
    const int32_t* cu_seqlens;
    const uint8_t* drop_enabled;
    const int32_t* cu_blocks;
    const __nv_bfloat16* q;
    const __nv_bfloat16* k;
    float* row_m;
    float* row_l;
    float* token_scores;
    float* block_scores;
    int64_t q_row_stride;
    int64_t k_row_stride;
    int32_t num_requests;
    int32_t num_heads;
    int32_t head_dim;
    int32_t gqa_group;
    int32_t q_head_offset;
    int32_t kv_head_offset;
    int32_t query_window_n;
    int32_t simt_n;  // row capacity of row_m / row_l per (head, request)
    int32_t block_size_g;
    float scale;     // 1 / sqrt(D)
};

struct SelectParams {
    const int32_t* cu_seqlens;
    const uint8_t* drop_enabled;
    const float* block_scores;
    const int32_t* cu_blocks;
    const uint8_t* veto;
    uint8_t* keep;
    int64_t* cutoff_rank;
    int64_t* retained_count;
    double* covered_mass;
    uint8_t* degenerate;
    uint32_t* err;
    int32_t query_window_n;
    int32_t block_size_g;
    int32_t sink_count_a;
    float top_p;
};

constexpr int kMaxPlanes = 8;

struct CompactParams {
    const int32_t* cu_seqlens;
    const uint8_t* drop_enabled;
    const uint8_t* keep;
    int32_t* cu_out;
    int32_t* retained_index;
    int32_t* num_out;
    int32_t* tile_counts;
    int32_t num_requests;
    int32_t num_planes;
    int64_t max_tokens;
    const uint8_t* src[kMaxPlanes];
    uint8_t* dst[kMaxPlanes];
    int64_t row_bytes[kMaxPlanes];
    int64_t src_stride[kMaxPlanes];
    int64_t dst_stride[kMaxPlanes];
};

}  // namespace up
