// capi.cu -- the C ABI (include/uniprefill_b200.h): host-side validation, workspace
// carve-up, TMA descriptor encoding and kernel launches.  No CPU fallback: every entry
// point either launches its sm_100a kernels or returns an error status.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace up {

// Launchers defined in the kernel translation units.
struct ScoreTcParams;
struct ScoreSimtParams;
struct SelectParams;
struct CompactParams;
int tc_max_hpc(int D);
cudaError_t launch_score_tc(int D, int HPC, const CUtensorMap& qm, const CUtensorMap& km,
                            const ScoreTcParams& p, int grid, cudaStream_t stream);
cudaError_t launch_score_tcw(int D, int HPC, const CUtensorMap& qm, const CUtensorMap& km,
                             const ScoreTcParams& p, int grid, cudaStream_t stream);
bool tcw_supported(int D, int HPC, int G, int R);
int tcw_stage_keys(int D);
bool tc2_enabled();
int tcw_npar(int D, int HPC, int G, int64_t max_tokens, int nhg, int grid);
int tcw_par_shift_for(int G);
bool tc2_supported(int D, int HPC, int G, int R);
int tc2_stage_keys();
int tc2_grid(int num_sms);
cudaError_t launch_score_tc2(const CUtensorMap& qm, const CUtensorMap& km, const ScoreTcParams& p, int grid,
                             cudaStream_t stream);
cudaError_t launch_blocks_plan(const int32_t* cu, int R, int64_t max_tokens, int G, int32_t* cu_blocks,
                               uint32_t* err, cudaStream_t stream);
struct BlockCombineParams;
struct PairWeightsParams;
struct SlotMapParams;
struct SequsedParams;
struct PeerReduceParams;
cudaError_t launch_block_combine(const BlockCombineParams& p, int grid, int sms, cudaStream_t stream);
cudaError_t launch_block_combine_peer(const BlockCombineParams& p, const PeerReduceParams& pr, int grid,
                                      cudaStream_t stream);
int peer_grid(int num_sms);
cudaError_t launch_pair_weights(const PairWeightsParams& p, int grid, int items_per_pair, cudaStream_t stream);
cudaError_t launch_score_simt(const ScoreSimtParams& p, int64_t max_tokens, int num_sms,
                              cudaStream_t stream);
cudaError_t launch_select(const SelectParams& p, int R, int max_blocks_per_request, int num_sms,
                          cudaStream_t stream);
bool select_fuses_expand(int64_t max_tokens);
bool compact_is_small(int64_t max_tokens);
cudaError_t launch_reduce_shards(const float* const* shards, int tp, int64_t count, float* out,
                                 int num_sms, cudaStream_t stream);
cudaError_t launch_compact(const CompactParams& p, int num_sms, cudaStream_t stream, bool counts_ready);
cudaError_t launch_scatter_rows(const CompactParams& p, int num_sms, cudaStream_t stream);
cudaError_t launch_slot_mapping(const SlotMapParams& p, int num_sms, cudaStream_t stream);
cudaError_t launch_decode_seqused(const SequsedParams& p, cudaStream_t stream);
struct AttnParams;
bool attention_supported(int D);
int attention_kv_box_rows(int D);
int attention_rows_per_cta(int D);
cudaError_t launch_peer_allreduce(const PeerReduceParams& p, int grid, cudaStream_t stream);
cudaError_t launch_attention(int D, const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                             const AttnParams& p, int grid, cudaStream_t stream);
int64_t compact_tiles(int64_t max_tokens);
int compact_max_planes();

}  // namespace up

// Full parameter structs (shared with the kernel TUs through identical definitions).
#include "params.cuh"

using namespace up;

namespace {

thread_local int g_launches = 0;

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

up_status cuda_status(cudaError_t e) { return e == cudaSuccess ? UP_OK : UP_ERR_CUDA; }

// Per-CTA timing of the tensor-core scorer (diagnostics only, enabled by UP_SCORE_DEBUG).
unsigned long long* score_debug_buffer() {
    static unsigned long long* d = [] {
        unsigned long long* x = nullptr;
        if (std::getenv("UP_SCORE_DEBUG")) cudaMalloc(&x, sizeof(unsigned long long) * 8 * 4096);
        return x;
    }();
    return d;
}

unsigned long long* select_debug_buffer() {
    static unsigned long long* d = [] {
        unsigned long long* x = nullptr;
        if (std::getenv("UP_SELECT_DEBUG")) cudaMalloc(&x, sizeof(unsigned long long) * 16);
        return x;
    }();
    return d;
}

// ---- workspace layout --------------------------------------------------------------
struct Layout {
    size_t err, cu_units, unit_sid, P, stat_m, stat_l, stat_w, simt_m, simt_l,
        simt_tok, tile_counts, ret_idx, blk_keep, total;
    int64_t max_blocks, max_units;
    int32_t simt_n;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Query tiles: a query window of n > 128 rows is scored as ceil(n/128) tiles of 128 rows
// (the tcgen05 M); tile t of q-head h is the virtual head h * Tt + t.  Each row's softmax
// is independent and the reference sums over rows (importance.cpp:41-74), so the virtual
// heads are summed like heads, with the 1/n_eff of the whole window.
constexpr int kMaxQTiles = 8;  // n <= 1024 on the tensor cores
int q_tiles(const up_score_config* c) {
    const int n = c->query_window_n > 0 ? c->query_window_n : 1;
    return (n + kRows - 1) / kRows;
}
// Query-row packing: a window of n <= 64 rows leaves most of a 128-row S tile empty, so P
// q-heads of one kv-group share it -- virtual head v holds q-heads [vP, vP + P), row r
// being window row r % (128/P) of q-head vP + r / (128/P).  Served by score_tcw's TS
// variants (Q loaded row by row by the epilogue threads: one or two virtual heads per
// kv-head at D >= 128): P = the largest power of two with P * npad <= 128 dividing the
// kv-group and the head slice.
int q_pack(const up_heads* h, const up_score_config* c, int shard_heads) {
    const int n = c->query_window_n;
    if (n > 64 || h->head_dim < 128) return 1;
    int npad = 1;
    while (npad < n) npad <<= 1;
    int P = kRows / npad;
    while (P > 1 && (h->gqa_group % P || h->num_q_heads % P || h->q_head_offset % P || shard_heads % P)) P >>= 1;
    return P;
}
up_heads packed_heads(const up_heads* h, int P) {
    up_heads v = *h;
    v.num_q_heads /= P;
    v.gqa_group /= P;
    v.q_head_offset /= P;
    return v;
}
up_heads virtual_heads(const up_heads* h, int Tt) {
    up_heads v = *h;
    v.num_q_heads *= Tt;
    v.gqa_group *= Tt;
    v.q_head_offset *= Tt;
    return v;
}

Layout layout_for(const up_batch* b, const up_heads* h, const up_score_config* c) {
    Layout L{};
    const int64_t T = b->max_tokens;
    const int64_t R = b->num_requests;
    const int64_t G = c->block_size_g > 0 ? c->block_size_g : 1;
    // query tiles (n > 128): the scorer's P partials and statistics are per virtual head
    const int64_t H = h ? static_cast<int64_t>(h->num_q_heads) * q_tiles(c) : 0;
    L.max_blocks = T / G + R + 1;
    // Σ_r ceil(N_r / unit) * num_hgroups * HPC * npar <= Hq * npar * (T / 128 + R): bounds
    // the item statistics rows; npar <= 4 (score_tcw HPC = 1 and score_tc2 keep four
    // statistics rows per head, the HPC = 2 / SPLIT epilogues two)
    const int64_t npar = h ? 4 : 1;
    L.max_units = (H > 0 ? H : 1) * npar * (T / kTileKeys + R + 1);
    const int64_t n = c->query_window_n < T ? c->query_window_n : T;
    L.simt_n = static_cast<int32_t>(n > 0 ? n : 1);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        off = align_up(off, 256);
        const size_t at = off;
        off += bytes;
        return at;
    };
    L.err = take(256);
    L.cu_units = take(sizeof(int32_t) * (R + 1));
    L.unit_sid = take(sizeof(int32_t) * L.max_units);
    L.P = take(sizeof(float) * H * L.max_blocks * kRows);
    L.stat_m = take(sizeof(float) * L.max_units * kRows);
    L.stat_l = take(sizeof(float) * L.max_units * kRows);
    L.stat_w = take(sizeof(float) * L.max_units * kRows);
    L.simt_m = take(sizeof(float) * H * R * L.simt_n);
    L.simt_l = take(sizeof(float) * H * R * L.simt_n);
    L.simt_tok = take(sizeof(float) * (T + 1));
    L.tile_counts = take(sizeof(int32_t) * (compact_tiles(T) + 1));
    L.ret_idx = take(sizeof(int32_t) * (T + 1));
    L.blk_keep = take(static_cast<size_t>(L.max_blocks));
    L.total = align_up(off, 256);
    return L;
}

template <class T>
T* at(void* ws, size_t off) {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(ws) + off);
}

up_status check_batch(const up_batch* b) {
    if (b == nullptr || b->cu_seqlens == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (b->num_requests < 1 || b->max_tokens < 1) return UP_ERR_CONTRACT;
    if (b->max_tokens > (int64_t{1} << 31) - 1) return UP_ERR_UNSUPPORTED;
    return UP_OK;
}

up_status check_heads(const up_heads* h) {
    if (h == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (h->num_q_heads < 1 || h->num_kv_heads < 1 || h->head_dim < 1 || h->gqa_group < 1)
        return UP_ERR_CONTRACT;
    if (h->q_head_offset < 0 || h->kv_head_offset < 0) return UP_ERR_CONTRACT;
    if (h->q_row_stride < static_cast<int64_t>(h->num_q_heads) * h->head_dim) return UP_ERR_CONTRACT;
    if (h->k_row_stride < static_cast<int64_t>(h->num_kv_heads) * h->head_dim) return UP_ERR_CONTRACT;
    // Every local q-head must map to a local kv-head.
    const int first_kv = h->q_head_offset / h->gqa_group - h->kv_head_offset;
    const int last_kv = (h->q_head_offset + h->num_q_heads - 1) / h->gqa_group - h->kv_head_offset;
    if (first_kv < 0 || last_kv >= h->num_kv_heads) return UP_ERR_CONTRACT;
    return UP_OK;
}

// ---- TMA descriptors ------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 view [rows, cols] with row stride `ld` elements, box 64 cols x 128 rows, 128B swizzle.
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_rows = 128) {
    EncodeTiledFn fn = encode_fn();
    if (fn == nullptr) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// q-heads per CTA (sharing one kv-head's K tile): the largest power of two <= max_hpc
// that divides the local head count, the head offset, the GQA group and the heads of
// one TP shard.
int pick_hpc(const up_heads* h, int max_hpc, int shard_heads) {
    int hpc = max_hpc;
    if (hpc > h->gqa_group) hpc = h->gqa_group;
    while (hpc > 1 && (h->num_q_heads % hpc || h->q_head_offset % hpc || h->gqa_group % hpc || shard_heads % hpc))
        hpc >>= 1;
    return hpc < 1 ? 1 : hpc;
}

// Which tensor-core scorer serves this shape: the CTA-pair kernel (score_tc2.cu, pair =
// true) for four q-heads per kv-head at D = 128, else the four-warpgroup kernel
// (score_tcw.cu, wide = true) when it applies, else score_tc.cu.  npar = statistics rows
// (epilogue warpgroups) per head.
struct TcPlan {
    bool wide, pair;
    int hpc, npar;
};

// CTAs of the single-CTA scorers: one per SM (UP_SCORE_GRID overrides, dev sweeps)
int score_grid() {
    static const int grid_override = [] {
        const char* s = std::getenv("UP_SCORE_GRID");
        return s ? std::atoi(s) : 0;
    }();
    // at most kPwMaxRanges work ranges (the tail's shared-memory table of range boundaries)
    return grid_override > 0 ? (grid_override < 1024 ? grid_override : 1024) : num_sms();
}

TcPlan tc_plan(const up_batch* b, const up_heads* h, const up_score_config* c, int shard_heads, int hpc_cap = 4) {
    const int D = h->head_dim;
    TcPlan t{};
    static const int max_hpc_env = [] {  // dev sweeps only
        const char* s = std::getenv("UP_MAX_HPC");
        return s ? std::atoi(s) : 0;
    }();
    const int want = max_hpc_env > 0 ? max_hpc_env : (D == 256 ? 2 : 4);
    t.hpc = pick_hpc(h, want < hpc_cap ? want : hpc_cap, shard_heads);
    t.pair = tc2_supported(D, t.hpc, c->block_size_g, b->num_requests);
    t.wide = !t.pair && tcw_supported(D, t.hpc, c->block_size_g, b->num_requests);
    if (!t.wide && !t.pair) t.hpc = pick_hpc(h, tc_max_hpc(D), shard_heads);
    t.npar = t.pair ? 4
                    : (t.wide ? tcw_npar(D, t.hpc, c->block_size_g, b->max_tokens, h->num_q_heads / t.hpc,
                                         score_grid())
                              : 1);
    return t;
}

bool tc_eligible(const up_heads* h, const up_score_config* c, int want_tokens) {
    const int D = h->head_dim;
    if (want_tokens) return false;
    if (!(D == 64 || D == 128 || D == 256)) return false;
    if (c->query_window_n > kRows * kMaxQTiles) return false;  // n > 128: query tiles (score_tcw only)
    if (c->block_size_g % 32 != 0) return false;
    if ((static_cast<int64_t>(h->q_row_stride) * 2) % 16 || (static_cast<int64_t>(h->k_row_stride) * 2) % 16)
        return false;
    return true;
}

int64_t lcm64(int64_t a, int64_t b) {
    int64_t x = a, y = b;
    while (y) { const int64_t t = x % y; x = y; y = t; }
    return a / x * b;
}

}  // namespace

extern "C" {

int up_abi_version(void) { return UP_ABI_VERSION; }

const char* up_status_string(up_status s) {
    switch (s) {
    case UP_OK: return "ok";
    case UP_ERR_CONFIG: return "ConfigError: invalid score configuration";
    case UP_ERR_CONTRACT: return "ContractViolation: operation precondition broken";
    case UP_ERR_UNSUPPORTED: return "unsupported: valid input outside the implemented envelope";
    case UP_ERR_WORKSPACE: return "workspace missing or too small";
    case UP_ERR_CUDA: return "CUDA error";
    case UP_ERR_INVALID_ARGUMENT: return "invalid argument";
    case UP_ERR_ALLOCATION_MISS: return "AllocationMissError: KV page not allocated";
    }
    return "unknown status";
}

int up_last_launch_count(void) { return g_launches; }

up_status up_config_validate(const up_score_config* c) {
    if (c == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (c->query_window_n <= 0) return UP_ERR_CONFIG;
    if (c->block_size_g <= 0) return UP_ERR_CONFIG;
    if (c->sink_count_a < 0) return UP_ERR_CONFIG;
    if (!(c->top_p > 0.0f && c->top_p <= 1.0f)) return UP_ERR_CONFIG;
    return UP_OK;
}

int64_t up_max_blocks(const up_batch* b, const up_score_config* c) {
    if (b == nullptr || c == nullptr || c->block_size_g <= 0) return 0;
    return b->max_tokens / c->block_size_g + b->num_requests + 1;
}

size_t up_workspace_bytes(const up_batch* b, const up_heads* h, const up_score_config* c) {
    if (b == nullptr || c == nullptr) return 0;
    return layout_for(b, h, c).total;
}

int up_scorer_kind(const up_heads* h, const up_score_config* c, int want_token_scores) {
    if (h == nullptr || c == nullptr) return 0;
    return tc_eligible(h, c, want_token_scores) ? 1 : 2;
}

// Tensor-core path: scorer kernel -> pair_weights -> block_combine.  With tp > 1 the local
// q-heads form tp contiguous shards; block_combine writes each shard's partial to
// shard_scores[t * shard_stride + g] (when non-null) and their ascending-order fp32 sum to
// block_scores (sharded_block_scores + allreduce_scores, tp_sim.cpp:12-49).
static up_status score_tc_path(cudaStream_t stream, const up_batch* b, const up_heads* h,
                               const up_score_config* c, const void* q, const void* k, int tp,
                               float* shard_scores, int64_t shard_stride, float* block_scores,
                               int32_t* cu_blocks, const Layout& L, void* ws,
                               const PeerReduceParams* peer = nullptr) {
    const int D = h->head_dim;
    const int R = b->num_requests;
    const int G = c->block_size_g;
    uint32_t* err = at<uint32_t>(ws, L.err);
    // the scorer works on virtual heads: query tiles (n > 128) or packed heads (n <= 64)
    const int Tt = q_tiles(c);
    int Pk = Tt == 1 && !std::getenv("UP_NO_QPACK") ? q_pack(h, c, h->num_q_heads / tp) : 1;
    up_heads hv = Pk > 1 ? packed_heads(h, Pk) : virtual_heads(h, Tt);
    TcPlan plan = tc_plan(b, &hv, c, hv.num_q_heads / tp, Pk > 1 ? 2 : 4);
    if (Pk > 1 && !(plan.wide && plan.hpc <= 2)) {  // packing needs score_tcw's TS variants
        Pk = 1;
        hv = *h;
        plan = tc_plan(b, &hv, c, hv.num_q_heads / tp);
    }
    if (Tt > 1 && !plan.wide) return UP_ERR_UNSUPPORTED;  // query tiles: score_tcw only (nothing enqueued)
    if (L.max_units >= (int64_t{1} << kUsidParShift)) return UP_ERR_CONTRACT;  // item ids share unit_sid with a parity
    const int hpc = plan.hpc;
    const int nhg = hv.num_q_heads / hpc;
    CUtensorMap qm, km;
    if (!make_map(&qm, q, b->max_tokens, static_cast<int64_t>(h->num_q_heads) * D, h->q_row_stride, 128) ||
        !make_map(&km, k, b->max_tokens, static_cast<int64_t>(h->num_kv_heads) * D, h->k_row_stride,
                  plan.pair ? tc2_stage_keys() : (plan.wide ? tcw_stage_keys(D) : 128)))
        return UP_ERR_CUDA;
    ScoreTcParams p{};
    p.q = static_cast<const __nv_bfloat16*>(q);
    p.q_row_stride = h->q_row_stride;
    p.cu_seqlens = b->cu_seqlens;
    p.drop_enabled = b->drop_enabled;
    p.cu_blocks = cu_blocks;
    p.cu_units_out = at<int32_t>(ws, L.cu_units);
    p.unit_sid = at<int32_t>(ws, L.unit_sid);
    p.err = err;
    p.P = at<float>(ws, L.P);
    p.stat_m = at<float>(ws, L.stat_m);
    p.stat_l = at<float>(ws, L.stat_l);
    p.stat_w = at<float>(ws, L.stat_w);
    p.max_tokens = b->max_tokens;
    p.max_blocks = L.max_blocks;
    p.num_requests = R;
    p.query_window_n = c->query_window_n;
    p.block_size_g = G;
    p.unit_keys = static_cast<int32_t>(lcm64(G, kTileKeys));
    p.num_hgroups = nhg;
    p.q_head_offset = h->q_head_offset;
    p.kv_head_offset = h->kv_head_offset;
    p.gqa_group = h->gqa_group;
    p.q_tiles = Tt;
    p.q_pack = Pk;
    p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D)));
    const int grid = plan.pair ? tc2_grid(num_sms()) : score_grid();
    // work ranges: one per CTA, or one per CTA pair
    const int ranges = plan.pair ? grid / 2 : grid;
    p.dbg = score_debug_buffer();
    if (p.dbg != nullptr) cudaMemsetAsync(p.dbg + 4 * 4096, 0, sizeof(unsigned long long) * 4 * 4096, stream);
    if (std::getenv("UP_SCORE_VERBOSE"))
        fprintf(stderr, "scorer: pair=%d wide=%d hpc=%d npar=%d grid=%d tiles=%d pack=%d\n", plan.pair, plan.wide, hpc,
                plan.npar, grid, Tt, Pk);
    cudaError_t e = plan.pair ? launch_score_tc2(qm, km, p, grid, stream)
                    : plan.wide ? launch_score_tcw(D, hpc, qm, km, p, grid, stream)
                                : launch_score_tc(D, hpc, qm, km, p, grid, stream);
    if (e != cudaSuccess) return e == cudaErrorInvalidValue ? UP_ERR_UNSUPPORTED : UP_ERR_CUDA;
    PairWeightsParams wp{};
    wp.cu_seqlens = b->cu_seqlens;
    wp.cu_units = p.cu_units_out;
    wp.stat_m = p.stat_m;
    wp.stat_l = p.stat_l;
    wp.stat_w = p.stat_w;
    wp.err = err;
    wp.num_requests = R;
    wp.num_hgroups = nhg;
    wp.hpc = hpc;
    wp.npar = plan.npar;
    wp.score_grid = ranges;
    wp.query_window_n = c->query_window_n;
    wp.q_tiles = Tt;
    wp.q_pack = Pk;
    {
        // UP_PW_WARP_ITEMS: test hook -- 0 sends every pair down the CTA path (same arithmetic)
        static const int wi = [] {
            const char* e = std::getenv("UP_PW_WARP_ITEMS");
            return e == nullptr ? kPwWarpItems : std::atoi(e);
        }();
        wp.warp_items = wi < 0 ? 0 : (wi > kPwWarpItems ? kPwWarpItems : wi);
    }
    const int64_t wtasks = static_cast<int64_t>(R) * nhg * hpc * 4;
    const int wgrid = static_cast<int>(wtasks < num_sms() * 16 ? wtasks : num_sms() * 16);
    // CTAs one (request, head-group) pair spans, for equal-length requests
    const int items_est = ranges / (R * nhg > 0 ? R * nhg : 1) + 2;
    if ((e = launch_pair_weights(wp, wgrid, items_est, stream)) != cudaSuccess) return UP_ERR_CUDA;
    BlockCombineParams bp{};
    bp.cu_seqlens = b->cu_seqlens;
    bp.cu_blocks = cu_blocks;
    bp.cu_units = p.cu_units_out;
    bp.unit_sid = p.unit_sid;
    bp.P = p.P;
    bp.stat_w = p.stat_w;
    bp.block_scores = block_scores;
    bp.shard_scores = shard_scores;
    bp.shard_stride = shard_stride;
    bp.max_blocks = L.max_blocks;
    bp.num_requests = R;
    bp.num_heads = hv.num_q_heads;
    bp.num_shards = tp;
    bp.hpc = hpc;
    bp.npar = plan.npar;
    bp.par_shift = plan.pair ? 7 : tcw_par_shift_for(G);
    bp.block_size_g = G;
    bp.unit_keys = p.unit_keys;
    if (peer != nullptr) {  // fused with the TP all-reduce over peer memory
        if ((e = launch_block_combine_peer(bp, *peer, peer_grid(num_sms()), stream)) != cudaSuccess)
            return UP_ERR_CUDA;
        g_launches = 3;
        return UP_OK;
    }
    const int64_t cgrid = (L.max_blocks + 7) / 8;  // warp per block, 8 warps per CTA
    if ((e = launch_block_combine(bp, static_cast<int>(cgrid < num_sms() * 8 ? cgrid : num_sms() * 8), num_sms(), stream)) !=
        cudaSuccess)
        return UP_ERR_CUDA;
    g_launches = 3;
    return UP_OK;
}

up_status up_score_blocks(void* stream_, const up_batch* b, const up_heads* h,
                          const up_score_config* c, const void* q, const void* k,
                          float* block_scores, int32_t* cu_blocks, float* token_scores, void* ws,
                          size_t ws_bytes) {
    g_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    up_status st = up_config_validate(c);
    if (st != UP_OK) return st;
    if ((st = check_batch(b)) != UP_OK) return st;
    if ((st = check_heads(h)) != UP_OK) return st;
    if (q == nullptr || k == nullptr || block_scores == nullptr || cu_blocks == nullptr)
        return UP_ERR_INVALID_ARGUMENT;
    const Layout L = layout_for(b, h, c);
    if (ws == nullptr || ws_bytes < L.total) return UP_ERR_WORKSPACE;
    const int R = b->num_requests;
    const int G = c->block_size_g;
    uint32_t* err = at<uint32_t>(ws, L.err);

    // TMA needs 16-byte aligned bases (strides are checked by tc_eligible)
    const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) & 15) == 0;
    if (aligned && tc_eligible(h, c, token_scores != nullptr)) {
        st = score_tc_path(stream, b, h, c, q, k, 1, nullptr, 0, block_scores, cu_blocks, L, ws);
        // UNSUPPORTED = the tensor-core kernels' shared-memory plan cannot hold R segments
        // (score_tcw: 4096; score_tc: ~5900 at D = 128); nothing was enqueued, so the SIMT
        // path below serves the batch
        if (st != UP_ERR_UNSUPPORTED) return st;
    }

    // Generic SIMT path.
    cudaError_t e = launch_blocks_plan(b->cu_seqlens, R, b->max_tokens, G, cu_blocks, err, stream);
    if (e != cudaSuccess) return UP_ERR_CUDA;
    ScoreSimtParams p{};
    p.cu_seqlens = b->cu_seqlens;
    p.drop_enabled = b->drop_enabled;
    p.cu_blocks = cu_blocks;
    p.q = static_cast<const __nv_bfloat16*>(q);
    p.k = static_cast<const __nv_bfloat16*>(k);
    p.row_m = at<float>(ws, L.simt_m);
    p.row_l = at<float>(ws, L.simt_l);
    p.token_scores = token_scores ? token_scores : at<float>(ws, L.simt_tok);
    p.block_scores = block_scores;
    p.q_row_stride = h->q_row_stride;
    p.k_row_stride = h->k_row_stride;
    p.num_requests = R;
    p.num_heads = h->num_q_heads;
    p.head_dim = h->head_dim;
    p.gqa_group = h->gqa_group;
    p.q_head_offset = h->q_head_offset;
    p.kv_head_offset = h->kv_head_offset;
    p.query_window_n = c->query_window_n;
    p.simt_n = L.simt_n;
    p.max_tokens = b->max_tokens;
    p.block_size_g = G;
    p.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(h->head_dim)));
    if ((e = launch_score_simt(p, b->max_tokens, num_sms(), stream)) != cudaSuccess) return UP_ERR_CUDA;
    g_launches = 4;
    return UP_OK;
}

up_status up_score_blocks_tp(void* stream_, const up_batch* b, const up_heads* h,
                             const up_score_config* c, const void* q, const void* k, int32_t tp,
                             float* shard_scores, int64_t shard_stride, float* block_scores,
                             int32_t* cu_blocks, void* ws, size_t ws_bytes) {
    g_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (tp <= 0) return UP_ERR_CONFIG;  // "tp_degree must be positive" (tp_sim.cpp:14)
    up_status st = up_config_validate(c);
    if (st != UP_OK) return st;
    if ((st = check_batch(b)) != UP_OK) return st;
    if ((st = check_heads(h)) != UP_OK) return st;
    if (h->num_q_heads % tp != 0) return UP_ERR_CONFIG;  // tp_sim.cpp:15-17
    if (q == nullptr || k == nullptr || block_scores == nullptr || cu_blocks == nullptr || shard_scores == nullptr)
        return UP_ERR_INVALID_ARGUMENT;
    if (shard_stride < up_max_blocks(b, c)) return UP_ERR_INVALID_ARGUMENT;
    const Layout L = layout_for(b, h, c);
    if (ws == nullptr || ws_bytes < L.total) return UP_ERR_WORKSPACE;
    const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) & 15) == 0;
    if (aligned && tc_eligible(h, c, 0) && tp <= 32) {  // the combine holds one shard sum per lane
        st = score_tc_path(stream, b, h, c, q, k, tp, shard_scores, shard_stride, block_scores, cu_blocks, L, ws);
        if (st != UP_ERR_UNSUPPORTED) return st;  // else nothing was enqueued: the per-shard path below
    }
    // Generic shapes: one SIMT scoring pass per shard, then the ordered shard sum.
    if (tp > 16) return UP_ERR_UNSUPPORTED;
    const int hps = h->num_q_heads / tp;
    const float* shards[16];
    int launches = 0;
    for (int t = 0; t < tp; ++t) {
        up_heads ht = *h;
        ht.num_q_heads = hps;
        ht.q_head_offset = h->q_head_offset + t * hps;
        const void* qt = static_cast<const __nv_bfloat16*>(q) + static_cast<int64_t>(t) * hps * h->head_dim;
        float* out_t = shard_scores + static_cast<int64_t>(t) * shard_stride;
        if ((st = up_score_blocks(stream_, b, &ht, c, qt, k, out_t, cu_blocks, nullptr, ws, ws_bytes)) != UP_OK)
            return st;
        launches += g_launches;
        shards[t] = out_t;
    }
    const cudaError_t e = launch_reduce_shards(shards, tp, up_max_blocks(b, c), block_scores, num_sms(), stream);
    g_launches = launches + 1;
    return cuda_status(e);
}

up_status up_reduce_block_scores(void* stream, const float* const* shards, int32_t tp,
                                 int64_t count, float* out) {
    g_launches = 0;
    if (shards == nullptr || out == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (tp < 1 || tp > 16) return tp < 1 ? UP_ERR_CONTRACT : UP_ERR_UNSUPPORTED;
    if (count < 0) return UP_ERR_CONTRACT;
    for (int t = 0; t < tp; ++t)
        if (shards[t] == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (count == 0) return UP_OK;
    const cudaError_t e = launch_reduce_shards(shards, tp, count, out, num_sms(),
                                               static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return cuda_status(e);
}

up_status up_select(void* stream, const up_batch* b, const up_score_config* c,
                    const float* block_scores, const int32_t* cu_blocks, const uint8_t* veto,
                    uint8_t* keep, const up_selection_out* out, void* ws, size_t ws_bytes) {
    g_launches = 0;
    up_status st = up_config_validate(c);
    if (st != UP_OK) return st;
    if ((st = check_batch(b)) != UP_OK) return st;
    if (block_scores == nullptr || cu_blocks == nullptr || keep == nullptr || out == nullptr ||
        out->cutoff_rank == nullptr)
        return UP_ERR_INVALID_ARGUMENT;
    const Layout L = layout_for(b, nullptr, c);
    if (ws == nullptr || ws_bytes < L.total) return UP_ERR_WORKSPACE;
    SelectParams p{};
    p.cu_seqlens = b->cu_seqlens;
    p.drop_enabled = b->drop_enabled;
    p.block_scores = block_scores;
    p.cu_blocks = cu_blocks;
    p.veto = veto;
    p.keep = keep;
    p.cutoff_rank = out->cutoff_rank;
    p.retained_count = out->retained_count;
    p.covered_mass = out->covered_mass;
    p.degenerate = out->degenerate;
    p.err = at<uint32_t>(ws, L.err);
    p.query_window_n = c->query_window_n;
    p.block_size_g = c->block_size_g;
    p.sink_count_a = c->sink_count_a;
    p.top_p = c->top_p;
    p.dbg = select_debug_buffer();
    p.blk_keep = at<uint8_t>(ws, L.blk_keep);
    p.tile_counts = at<int32_t>(ws, L.tile_counts);
    p.max_tokens = b->max_tokens;
    const int64_t per_req = (b->max_tokens + c->block_size_g - 1) / c->block_size_g;
    p.fuse_expand = select_fuses_expand(b->max_tokens) ? 1 : 0;
    const cudaError_t e = launch_select(p, b->num_requests, static_cast<int>(per_req < kMaxSortBlocks ? per_req : kMaxSortBlocks),
                                        num_sms(), static_cast<cudaStream_t>(stream));
    // size classes + the expand launch (folded into the select CTAs at small capacities)
    g_launches = 1 + (per_req > 512 ? 1 : 0) + (per_req > 2048 ? 1 : 0) + (p.fuse_expand ? 0 : 1);
    return cuda_status(e);
}

static up_status compact_impl(void* stream, const up_batch* b, const uint8_t* keep, const up_plane* planes,
                              int32_t num_planes, int32_t* cu_out, int32_t* retained_index, int32_t* num_out,
                              void* ws, size_t ws_bytes, bool counts_ready) {
    g_launches = 0;
    up_status st = check_batch(b);
    if (st != UP_OK) return st;
    if (keep == nullptr || cu_out == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (num_planes < 0 || num_planes > compact_max_planes()) return UP_ERR_UNSUPPORTED;
    if (num_planes > 0 && planes == nullptr) return UP_ERR_INVALID_ARGUMENT;
    // G only sizes the block-decision region, unused here: a huge G keeps this layout a
    // prefix of up_select's (same tile-count offset, no larger workspace requirement)
    up_score_config dummy{1, 1 << 20, 0, 1.0f};
    const Layout L = layout_for(b, nullptr, &dummy);
    if (ws == nullptr || ws_bytes < L.total) return UP_ERR_WORKSPACE;
    CompactParams p{};
    p.cu_seqlens = b->cu_seqlens;
    p.drop_enabled = b->drop_enabled;
    p.keep = keep;
    p.cu_out = cu_out;
    p.retained_index = retained_index ? retained_index : at<int32_t>(ws, L.ret_idx);
    p.num_out = num_out;
    p.tile_counts = at<int32_t>(ws, L.tile_counts);
    p.num_requests = b->num_requests;
    p.num_planes = num_planes;
    p.max_tokens = b->max_tokens;
    for (int i = 0; i < num_planes; ++i) {
        const up_plane& pl = planes[i];
        if (pl.src == nullptr || pl.dst == nullptr || pl.row_bytes <= 0) return UP_ERR_INVALID_ARGUMENT;
        p.src[i] = static_cast<const uint8_t*>(pl.src);
        p.dst[i] = static_cast<uint8_t*>(pl.dst);
        p.row_bytes[i] = pl.row_bytes;
        p.src_stride[i] = pl.src_stride_bytes > 0 ? pl.src_stride_bytes : pl.row_bytes;
        p.dst_stride[i] = pl.dst_stride_bytes > 0 ? pl.dst_stride_bytes : pl.row_bytes;
        if (p.src_stride[i] < pl.row_bytes || p.dst_stride[i] < pl.row_bytes) return UP_ERR_CONTRACT;
    }
    const cudaError_t e = launch_compact(p, num_sms(), static_cast<cudaStream_t>(stream), counts_ready);
    g_launches = compact_is_small(b->max_tokens) ? 1 : (num_planes > 0 ? 3 : 2) - (counts_ready ? 1 : 0);
    return cuda_status(e);
}

up_status up_compact(void* stream, const up_batch* b, const uint8_t* keep, const up_plane* planes,
                     int32_t num_planes, int32_t* cu_out, int32_t* retained_index,
                     int32_t* num_out, void* ws, size_t ws_bytes) {
    return compact_impl(stream, b, keep, planes, num_planes, cu_out, retained_index, num_out, ws, ws_bytes, false);
}

up_status up_compact_selected(void* stream, const up_batch* b, const uint8_t* keep, const up_plane* planes,
                              int32_t num_planes, int32_t* cu_out, int32_t* retained_index, int32_t* num_out,
                              void* ws, size_t ws_bytes) {
    return compact_impl(stream, b, keep, planes, num_planes, cu_out, retained_index, num_out, ws, ws_bytes, true);
}

up_status up_scatter_rows(void* stream, const int32_t* index, const int32_t* num_rows, int64_t max_rows,
                          const up_plane* planes, int32_t num_planes) {
    g_launches = 0;
    if (index == nullptr || max_rows < 0) return index == nullptr ? UP_ERR_INVALID_ARGUMENT : UP_ERR_CONTRACT;
    if (num_planes < 0 || num_planes > compact_max_planes()) return UP_ERR_UNSUPPORTED;
    if (num_planes > 0 && planes == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (max_rows > (int64_t{1} << 31) - 1) return UP_ERR_UNSUPPORTED;
    CompactParams p{};
    p.retained_index = const_cast<int32_t*>(index);
    p.num_out = const_cast<int32_t*>(num_rows);
    p.num_planes = num_planes;
    p.max_tokens = max_rows;
    for (int i = 0; i < num_planes; ++i) {
        const up_plane& pl = planes[i];
        if (pl.src == nullptr || pl.dst == nullptr || pl.row_bytes <= 0) return UP_ERR_INVALID_ARGUMENT;
        p.src[i] = static_cast<const uint8_t*>(pl.src);
        p.dst[i] = static_cast<uint8_t*>(pl.dst);
        p.row_bytes[i] = pl.row_bytes;
        p.src_stride[i] = pl.src_stride_bytes > 0 ? pl.src_stride_bytes : pl.row_bytes;
        p.dst_stride[i] = pl.dst_stride_bytes > 0 ? pl.dst_stride_bytes : pl.row_bytes;
        if (p.src_stride[i] < pl.row_bytes || p.dst_stride[i] < pl.row_bytes) return UP_ERR_CONTRACT;
    }
    const cudaError_t e = launch_scatter_rows(p, num_sms(), static_cast<cudaStream_t>(stream));
    g_launches = num_planes > 0 && max_rows > 0 ? 1 : 0;
    return cuda_status(e);
}

up_status up_drop_layer(void* stream, const up_batch* b, const up_heads* h,
                        const up_score_config* c, const void* q, const void* k,
                        const uint8_t* veto, float* block_scores, int32_t* cu_blocks,
                        uint8_t* keep, const up_selection_out* sel, const up_plane* planes,
                        int32_t num_planes, int32_t* cu_out, int32_t* retained_index,
                        int32_t* num_out, void* ws, size_t ws_bytes) {
    up_status st = up_score_blocks(stream, b, h, c, q, k, block_scores, cu_blocks, nullptr, ws, ws_bytes);
    if (st != UP_OK) return st;
    const int n1 = g_launches;
    st = up_select(stream, b, c, block_scores, cu_blocks, veto, keep, sel, ws, ws_bytes);
    if (st != UP_OK) return st;
    const int n2 = g_launches;
    st = up_compact_selected(stream, b, keep, planes, num_planes, cu_out, retained_index, num_out, ws, ws_bytes);
    g_launches += n1 + n2;
    return st;
}

up_status up_slot_mapping(void* stream, const int32_t* cu_seqlens, int32_t num_requests, const int32_t* num_rows,
                          int64_t max_rows, const int64_t* positions, const int32_t* block_tables,
                          int32_t num_layers, int32_t max_pages, int32_t block_size, int64_t* slots,
                          int64_t slot_stride, void* ws, size_t ws_bytes) {
    g_launches = 0;
    if (cu_seqlens == nullptr || positions == nullptr || block_tables == nullptr || slots == nullptr || ws == nullptr)
        return UP_ERR_INVALID_ARGUMENT;
    if (num_requests < 1 || num_layers < 0 || max_pages < 1 || max_rows < 0) return UP_ERR_CONTRACT;
    if (block_size <= 0) return UP_ERR_CONFIG;  // PagedKVCache: kv_block_size must be positive
    if (slot_stride < max_rows) return UP_ERR_INVALID_ARGUMENT;
    if (ws_bytes < 256) return UP_ERR_WORKSPACE;
    if (num_layers == 0 || max_rows == 0) return UP_OK;
    SlotMapParams p{};
    p.cu_seqlens = cu_seqlens;
    p.num_rows = num_rows;
    p.positions = positions;
    p.block_tables = block_tables;
    p.slots = slots;
    p.err = static_cast<uint32_t*>(ws);  // the sticky flags word at the workspace start
    p.max_rows = max_rows;
    p.slot_stride = slot_stride;
    p.num_requests = num_requests;
    p.num_layers = num_layers;
    p.max_pages = max_pages;
    p.block_size = block_size;
    const cudaError_t e = launch_slot_mapping(p, num_sms(), static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return cuda_status(e);
}

up_status up_decode_seqused(void* stream, int32_t num_layers, int32_t num_requests, const int32_t* cu_orig,
                            int32_t num_drops, const int32_t* drop_layers, const int32_t* const* cu_after,
                            const int32_t* decode_appended, int32_t* seqused) {
    g_launches = 0;
    if (cu_orig == nullptr || seqused == nullptr || (num_drops > 0 && (drop_layers == nullptr || cu_after == nullptr)))
        return UP_ERR_INVALID_ARGUMENT;
    if (num_layers < 0 || num_requests < 1 || num_drops < 0) return UP_ERR_CONTRACT;
    if (num_drops > kMaxDrops) return UP_ERR_UNSUPPORTED;
    SequsedParams p{};
    for (int d = 0; d < num_drops; ++d) {
        // DropHistory::validate: layers strictly increasing (drop_history.hpp:27-29)
        if (d > 0 && drop_layers[d] <= drop_layers[d - 1]) return UP_ERR_CONTRACT;
        if (cu_after[d] == nullptr) return UP_ERR_INVALID_ARGUMENT;
        p.drop_layers[d] = drop_layers[d];
        p.cu_after[d] = cu_after[d];
    }
    if (num_layers == 0) return UP_OK;
    p.cu_orig = cu_orig;
    p.decode_appended = decode_appended;
    p.seqused = seqused;
    p.num_drops = num_drops;
    p.num_layers = num_layers;
    p.num_requests = num_requests;
    const cudaError_t e = launch_decode_seqused(p, static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return cuda_status(e);
}

up_status up_attention_varlen(void* stream, const up_batch* b, const up_heads* h, const void* q, const void* k,
                              const void* v, const int64_t* positions, int64_t window, void* out,
                              int64_t out_row_stride, void* ws, size_t ws_bytes) {
    g_launches = 0;
    if (b == nullptr || h == nullptr || q == nullptr || k == nullptr || v == nullptr || positions == nullptr ||
        out == nullptr || ws == nullptr || b->cu_seqlens == nullptr)
        return UP_ERR_INVALID_ARGUMENT;
    if (b->num_requests < 1 || b->max_tokens < 0 || h->num_q_heads < 1 || h->num_kv_heads < 1 || h->gqa_group < 1)
        return UP_ERR_CONTRACT;
    if (ws_bytes < 256) return UP_ERR_WORKSPACE;
    const int D = h->head_dim;
    if (!attention_supported(D)) return UP_ERR_UNSUPPORTED;
    // every local q-head must read a local kv-head
    const int kv_lo = h->q_head_offset / h->gqa_group - h->kv_head_offset;
    const int kv_hi = (h->q_head_offset + h->num_q_heads - 1) / h->gqa_group - h->kv_head_offset;
    if (kv_lo < 0 || kv_hi >= h->num_kv_heads) return UP_ERR_CONTRACT;
    const int64_t qcols = static_cast<int64_t>(h->num_q_heads) * D, kcols = static_cast<int64_t>(h->num_kv_heads) * D;
    if (h->q_row_stride < qcols || h->k_row_stride < kcols || out_row_stride < qcols) return UP_ERR_INVALID_ARGUMENT;
    // TMA: 16-byte aligned bases and row strides
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
         reinterpret_cast<uintptr_t>(out)) & 15 || (h->q_row_stride | h->k_row_stride | out_row_stride) & 7)
        return UP_ERR_UNSUPPORTED;
    if (b->max_tokens == 0) return UP_OK;
    CUtensorMap qm, km, vm;
    if (!make_map(&qm, q, b->max_tokens, qcols, h->q_row_stride) ||
        !make_map(&km, k, b->max_tokens, kcols, h->k_row_stride, attention_kv_box_rows(D)) ||
        !make_map(&vm, v, b->max_tokens, kcols, h->k_row_stride, attention_kv_box_rows(D)))
        return UP_ERR_CUDA;
    AttnParams p{};
    p.cu_seqlens = b->cu_seqlens;
    p.positions = positions;
    p.out = static_cast<__nv_bfloat16*>(out);
    p.q = static_cast<const __nv_bfloat16*>(q);
    p.q_row_stride = h->q_row_stride;
    p.err = static_cast<uint32_t*>(ws);
    p.max_tokens = b->max_tokens;
    p.out_row_stride = out_row_stride;
    p.window = window;
    p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(D)));
    p.num_requests = b->num_requests;
    p.num_q_heads = h->num_q_heads;
    p.gqa_group = h->gqa_group;
    p.q_head_offset = h->q_head_offset;
    p.kv_head_offset = h->kv_head_offset;
    const int rows = attention_rows_per_cta(D);  // Σ_r ⌈n_r/rows⌉ <= ⌈max_tokens/rows⌉ + R
    const int64_t tiles = (b->max_tokens + rows - 1) / rows + b->num_requests;
    int64_t grid = tiles * h->num_q_heads;
    if (rows == 256 && grid > num_sms()) grid = num_sms();  // persistent two-tile kernel
    if (grid > 0x7fffffff) return UP_ERR_UNSUPPORTED;
    const cudaError_t e = launch_attention(D, qm, km, vm, p, static_cast<int>(grid), static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return cuda_status(e);
}

size_t up_peer_buffer_bytes(int32_t tp, int64_t capacity) {
    if (tp < 1 || tp > kPeerMaxRanks || capacity < 0) return 0;
    // two banks of [tp][capacity] fp32, alternating by epoch parity (peer.cuh)
    return static_cast<size_t>(kPeerSlotsOffset) + 2 * static_cast<size_t>(tp) * static_cast<size_t>(capacity) * 4;
}

up_status up_peer_buffer_alloc(int32_t tp, int64_t capacity, void** buffer) {
    if (buffer == nullptr) return UP_ERR_INVALID_ARGUMENT;
    const size_t bytes = up_peer_buffer_bytes(tp, capacity);
    if (bytes == 0) return tp < 1 || capacity < 0 ? UP_ERR_CONTRACT : UP_ERR_UNSUPPORTED;
    if (cudaMalloc(buffer, bytes) != cudaSuccess) return UP_ERR_CUDA;
    if (cudaMemset(*buffer, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return UP_ERR_CUDA;
    return UP_OK;
}

up_status up_peer_buffer_free(void* buffer) {
    return cudaFree(buffer) == cudaSuccess ? UP_OK : UP_ERR_CUDA;
}

up_status up_ipc_get_handle(const void* buffer, void* handle) {
    if (buffer == nullptr || handle == nullptr) return UP_ERR_INVALID_ARGUMENT;
    static_assert(sizeof(cudaIpcMemHandle_t) == UP_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, const_cast<void*>(buffer)) != cudaSuccess) return UP_ERR_CUDA;
    std::memcpy(handle, &h, sizeof(h));
    return UP_OK;
}

up_status up_ipc_open_handle(const void* handle, void** buffer) {
    if (buffer == nullptr || handle == nullptr) return UP_ERR_INVALID_ARGUMENT;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    return cudaIpcOpenMemHandle(buffer, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? UP_OK : UP_ERR_CUDA;
}

up_status up_ipc_close_handle(void* buffer) {
    return cudaIpcCloseMemHandle(buffer) == cudaSuccess ? UP_OK : UP_ERR_CUDA;
}

static up_status peer_params(int32_t rank, int32_t tp, void* const* peer_buffers, int64_t capacity, float* out,
                             uint32_t* err, PeerReduceParams* p) {
    if (peer_buffers == nullptr || out == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (tp < 1 || rank < 0 || rank >= tp || capacity < 0) return UP_ERR_CONTRACT;
    if (tp > kPeerMaxRanks) return UP_ERR_UNSUPPORTED;
    for (int t = 0; t < tp; ++t)
        if (peer_buffers[t] == nullptr) return UP_ERR_INVALID_ARGUMENT;
    *p = PeerReduceParams{};
    for (int t = 0; t < tp; ++t) {
        uint8_t* b = static_cast<uint8_t*>(peer_buffers[t]);
        p->peer_slots[t] = reinterpret_cast<float*>(b + kPeerSlotsOffset);
        p->peer_flags[t] = reinterpret_cast<uint32_t*>(b + kPeerFlagsOffset);
    }
    uint8_t* own = static_cast<uint8_t*>(peer_buffers[rank]);
    p->slots = reinterpret_cast<const float*>(own + kPeerSlotsOffset);
    p->flags = reinterpret_cast<const uint32_t*>(own + kPeerFlagsOffset);
    p->epoch = reinterpret_cast<uint32_t*>(own);
    p->out = out;
    p->err = err;
    p->capacity = capacity;
    p->rank = rank;
    p->tp = tp;
    return UP_OK;
}

up_status up_peer_allreduce_scores(void* stream, const float* partial, int64_t count, int32_t rank, int32_t tp,
                                   void* const* peer_buffers, int64_t capacity, float* out, void* ws,
                                   size_t ws_bytes) {
    g_launches = 0;
    if (partial == nullptr || ws == nullptr) return UP_ERR_INVALID_ARGUMENT;
    if (count < 0 || count > capacity) return UP_ERR_CONTRACT;
    if (ws_bytes < 256) return UP_ERR_WORKSPACE;
    PeerReduceParams p;
    const up_status st = peer_params(rank, tp, peer_buffers, capacity, out, static_cast<uint32_t*>(ws), &p);
    if (st != UP_OK) return st;
    if (count == 0) return UP_OK;
    p.partial = partial;
    p.count = count;
    // A fixed grid of one CTA per SM whatever the count (every chunk's CTA is resident
    // while it waits for its peers, and every flag advances by tp per call, which the
    // epoch-based targets rely on); trailing CTAs may own an empty chunk.
    const int grid = peer_grid(num_sms());
    const int64_t chunk = (count + grid - 1) / grid;
    p.chunk = (chunk + 63) / 64 * 64;
    const cudaError_t e = launch_peer_allreduce(p, grid, static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return cuda_status(e);
}

up_status up_score_blocks_peer(void* stream_, const up_batch* b, const up_heads* h, const up_score_config* c,
                               const void* q, const void* k, int32_t rank, int32_t tp, void* const* peer_buffers,
                               int64_t capacity, float* block_scores, int32_t* cu_blocks, void* ws, size_t ws_bytes) {
    g_launches = 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    up_status st = up_config_validate(c);
    if (st != UP_OK) return st;
    if ((st = check_batch(b)) != UP_OK) return st;
    if ((st = check_heads(h)) != UP_OK) return st;
    if (q == nullptr || k == nullptr || block_scores == nullptr || cu_blocks == nullptr)
        return UP_ERR_INVALID_ARGUMENT;
    const Layout L = layout_for(b, h, c);
    if (ws == nullptr || ws_bytes < L.total) return UP_ERR_WORKSPACE;
    PeerReduceParams pr;
    if ((st = peer_params(rank, tp, peer_buffers, capacity, block_scores, at<uint32_t>(ws, L.err), &pr)) != UP_OK)
        return st;
    const bool aligned = ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) & 15) == 0;
    if (aligned && tc_eligible(h, c, 0)) {
        st = score_tc_path(stream, b, h, c, q, k, 1, nullptr, 0, block_scores, cu_blocks, L, ws, &pr);
        if (st != UP_ERR_UNSUPPORTED) return st;  // else nothing was enqueued: SIMT + peer all-reduce below
    }
    // off the tensor-core envelope: SIMT scoring, then the stand-alone peer all-reduce over
    // the capacity-sized vector (the same count on every rank)
    if ((st = up_score_blocks(stream_, b, h, c, q, k, block_scores, cu_blocks, nullptr, ws, ws_bytes)) != UP_OK)
        return st;
    const int n = g_launches;
    const int64_t count = up_max_blocks(b, c);
    if (count > capacity) return UP_ERR_UNSUPPORTED;
    st = up_peer_allreduce_scores(stream_, block_scores, count, rank, tp, peer_buffers, capacity, block_scores,
                                  at<uint32_t>(ws, L.err), 256);
    g_launches += n;
    return st;
}

up_status up_device_status(void* stream, void* ws) {
    if (ws == nullptr) return UP_ERR_INVALID_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t flags = 0;
    if (cudaMemcpyAsync(&flags, ws, sizeof(flags), cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return UP_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return UP_ERR_CUDA;
    if (flags != 0) {
        if (cudaMemsetAsync(ws, 0, sizeof(uint32_t), s) != cudaSuccess) return UP_ERR_CUDA;
        if (cudaStreamSynchronize(s) != cudaSuccess) return UP_ERR_CUDA;
    }
    if (flags & kErrTooManyBlocks) return UP_ERR_UNSUPPORTED;
    if (flags & kErrAllocationMiss) return UP_ERR_ALLOCATION_MISS;
    if (flags & kErrPeerTimeout) return UP_ERR_CUDA;
    if (flags & (kErrBadScore | kErrBadSeqlens | kErrMaskedRow | kErrNoVisibleKey)) return UP_ERR_CONTRACT;
    return UP_OK;
}

}  // extern "C"

// Diagnostics (not part of the ABI header): phase clocks of the select kernel's CTA 0.
extern "C" int up_internal_select_debug(unsigned long long* host) {
    unsigned long long* d = select_debug_buffer();
    if (d == nullptr || host == nullptr) return -1;
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    return cudaMemcpy(host, d, sizeof(unsigned long long) * 16, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -3;
}

// Diagnostics (not part of the ABI header): copy the scorer's per-CTA timing records
// [cta][start_ns, end_ns, units, smid] of the last launch to host memory.
// Diagnostics: score_tcw's per-CTA phase clocks [cta][first Q landed (MMA warp), first S
// region drained start (epilogue warp 2), first item done (epilogue warp 2), -].
extern "C" int up_internal_score_phases(unsigned long long* host, int max_ctas) {
    unsigned long long* d = score_debug_buffer();
    if (d == nullptr || host == nullptr) return -1;
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    return cudaMemcpy(host, d + 4 * 4096, sizeof(unsigned long long) * 4 * max_ctas, cudaMemcpyDeviceToHost) ==
                   cudaSuccess ? 0 : -3;
}

extern "C" int up_internal_score_debug(unsigned long long* host, int max_ctas) {
    unsigned long long* d = score_debug_buffer();
    if (d == nullptr || host == nullptr) return -1;
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    return cudaMemcpy(host, d, sizeof(unsigned long long) * 4 * max_ctas, cudaMemcpyDeviceToHost) ==
                   cudaSuccess ? 0 : -3;
}
