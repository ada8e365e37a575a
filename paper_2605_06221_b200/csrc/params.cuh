// params.cuh -- kernel parameter blocks shared by the launchers (capi.cu) and kernels.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace up {

struct ScoreTcParams {
    const __nv_bfloat16* q;   // [max_tokens, q_row_stride] (score_tcw TS variant loads Q rows itself)
    int64_t q_row_stride;
    const int32_t* cu_seqlens;
    const uint8_t* drop_enabled;
    int32_t* cu_blocks;       // out [R+1] (written by CTA 0)
    int32_t* cu_units_out;    // out [R+1] (written by CTA 0, read by the combine)
    int32_t* unit_sid;        // out [total units]: item id (stats row) of every unit
    uint32_t* err;
    float* P;                 // [Hq][max_blocks][128]
    float* stat_m;            // [units * HPC][128]
    float* stat_l;
    float* stat_w;
    int64_t max_tokens;
    int64_t max_blocks;
    int32_t num_requests;
    int32_t query_window_n;
    int32_t block_size_g;
    int32_t unit_keys;        // lcm(G, 128)
    int32_t num_hgroups;
    int32_t q_head_offset;
    int32_t kv_head_offset;
    int32_t gqa_group;
    // query tiles: n > 128 query rows are ceil(n/128) tiles of 128 rows; tile t of local
    // q-head h is VIRTUAL head h * q_tiles + t (num_hgroups, P and the statistics count
    // virtual heads; q_head_offset / gqa_group above are in real heads)
    int32_t q_tiles;
    // query-row packing (n <= 64, the TS variant): q_pack q-heads of one kv-group share a
    // 128-row S tile -- row r of virtual head v is window row r % (128 / q_pack) of q-head
    // v * q_pack + r / (128 / q_pack); 1 = no packing (exclusive with q_tiles > 1)
    int32_t q_pack;
    float scale_log2;         // log2(e) / sqrt(D)
    unsigned long long* dbg;  // optional per-CTA timing [grid][4] (UP_SCORE_DEBUG), else null
};

constexpr int kPwWarpItems = 2;  // pair_weights: warp path for pairs over <= 2 scorer CTAs (score_tail.cuh)

struct PairWeightsParams {
    const int32_t* cu_seqlens;
    const int32_t* cu_units;  // [R+1] from the scorer
    const float* stat_m;
    const float* stat_l;
    float* stat_w;
    uint32_t* err;
    int32_t num_requests;
    int32_t num_hgroups;
    int32_t hpc;
    int32_t npar;             // statistics rows per head (parity warpgroups of score_tcw)
    int32_t score_grid;       // the scorer's gridDim.x (defines the item ranges)
    int32_t query_window_n;
    int32_t q_tiles;          // query tiles per q-head (virtual head = h * q_tiles + t)
    int32_t q_pack;           // q-heads packed per virtual head (row r -> window row r % (128 / q_pack))
    int32_t warp_items;       // pairs over <= this many scorer CTAs take the warp path (0: none)
};

struct BlockCombineParams {
    const int32_t* cu_seqlens;
    const int32_t* cu_blocks;
    const int32_t* cu_units;
    const int32_t* unit_sid;
    const float* P;
    const float* stat_w;
    float* block_scores;
    float* shard_scores;      // optional [num_shards][shard_stride] per-shard partials
    int64_t shard_stride;
    int64_t max_blocks;
    int32_t num_requests;
    int32_t num_heads;
    int32_t num_shards;       // 1, or T contiguous head shards summed in ascending order
    int32_t hpc;
    int32_t npar;             // epilogue warpgroups per head (score_tcw): stats row hh*npar+par
    int32_t par_shift;        // par = (block start key >> par_shift) % npar: 6 (score_tcw), 7 (score_tc2)
    int32_t block_size_g;
    int32_t unit_keys;
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
    int64_t max_tokens;
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
    uint8_t* blk_keep;        // workspace [max_blocks]: per-block decisions for the expand kernel
    int32_t* tile_counts;     // workspace: kept tokens per 1024-token tile (read by up_compact_selected)
    int64_t max_tokens;
    unsigned long long* dbg;  // optional phase clocks of CTA 0 (UP_SELECT_DEBUG), else null
    int32_t nb_lo, nb_hi;     // this launch handles the requests with nb_lo < blocks <= nb_hi
    int32_t fuse_expand;      // small capacity: each select CTA writes its request's token mask
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

struct SlotMapParams {
    const int32_t* cu_seqlens;    // [R+1] of the compacted batch
    const int32_t* num_rows;      // device row count (or null: max_rows)
    const int64_t* positions;     // [rows] logical positions
    const int32_t* block_tables;  // [num_layers][R][max_pages] physical page ids (-1 = none)
    int64_t* slots;               // [num_layers][slot_stride]
    uint32_t* err;
    int64_t max_rows;
    int64_t slot_stride;
    int32_t num_requests;
    int32_t num_layers;
    int32_t max_pages;
    int32_t block_size;
};

constexpr int kMaxDrops = 64;

struct SequsedParams {
    const int32_t* cu_orig;              // [R+1] prompt lengths (original cu_seqlens)
    const int32_t* cu_after[kMaxDrops];  // cu_seqlens after each drop event
    int32_t drop_layers[kMaxDrops];      // strictly increasing
    const int32_t* decode_appended;      // [R] or null
    int32_t* seqused;                    // [num_layers][R]
    int32_t num_drops;
    int32_t num_layers;
    int32_t num_requests;
};

// Attention readout over the retained rows (attention.cu).
struct AttnParams {
    const int32_t* cu_seqlens;   // [R+1] segments of the (compacted) batch
    const int64_t* positions;    // [rows] logical positions, strictly increasing per segment
    __nv_bfloat16* out;          // [rows][out_row_stride], head h at column h*D
    const __nv_bfloat16* q;      // [rows][q_row_stride] (D = 256: rows copied into TMEM)
    int64_t q_row_stride;
    uint32_t* err;
    int64_t max_tokens;
    int64_t out_row_stride;
    int64_t window;              // > 0: keys with pos > q_pos - window only
    float scale_log2;            // log2(e) / sqrt(D)
    int32_t num_requests;
    int32_t num_q_heads;
    int32_t gqa_group;
    int32_t q_head_offset;
    int32_t kv_head_offset;
};

// One-shot TP all-reduce of partial block scores over peer memory (peer.cu).
constexpr int kPeerMaxRanks = 16;
constexpr int kPeerMaxChunks = 256;
constexpr int64_t kPeerFlagsOffset = 256;   // bytes: epoch[2] at 0, flags[kPeerMaxChunks] here,
constexpr int64_t kPeerSlotsOffset = 2048;  // slots[2][tp][capacity] here (bank = epoch & 1)
struct PeerReduceParams {
    const float* partial;                 // [count] this rank's partial
    float* peer_slots[kPeerMaxRanks];     // rank t's slots (mapped), row-major [2][tp][capacity]
    uint32_t* peer_flags[kPeerMaxRanks];  // rank t's flags (mapped)
    const float* slots;                   // own slots
    const uint32_t* flags;                // own flags
    uint32_t* epoch;                      // own epoch[2]
    float* out;
    uint32_t* err;
    int64_t count;
    int64_t capacity;
    int64_t chunk;
    int32_t rank;
    int32_t tp;
};

}  // namespace up
