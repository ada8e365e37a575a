// score_tail.cuh -- the scorer's tail, shared by the standalone kernels (score_tc.cu) and
// the peer-fused combine (peer.cu): per-pair row weights from the per-item softmax
// statistics, then the per-block combine over heads (and TP shards).  (An in-kernel tail
// behind a grid barrier in score_tcw was measured slower than the two PDL launches.)
#pragma once
#include <cstdint>
#include <type_traits>

#include "score_common.cuh"

namespace up {

// Row weights of every (request, head-group) pair, from the per-item statistics the
// scorer wrote: w[item][hh][j] = 2^(m_item - M) / (L n_eff), M = max_items m,
// L = Σ_items l 2^(m - M) -- the softmax denominator over the full key range
// (online_softmax_reduce pass 1, importance.cpp:41-58) assembled from the items' partial
// denominators.  One CTA per (pair, head, 32-row chunk): warp w folds items w, w+W, ...
// (lane = row, coalesced; 4 items' loads in flight per warp), the W partial (M, L) are
// merged in warp order (deterministic), then the warps write the weights.
constexpr int kPwWarps = 32;


// Pair weights for tasks t0, t0 + tstep, ... (task = (pair, head, 32-row chunk)); every
// thread of the CTA calls it (CTA barriers inside); warps >= nwarps only join the barriers.
// rb: shared-memory table of the scorer's range boundaries range_begin(c), c <= score_grid
// (kPwMaxRanges entries): the items of a pair are looked up there instead of by 64-bit
// divisions per item and lane (measured: those divisions made the tail 18 us for one long
// request spread over 148 items).
constexpr int kPwMaxRanges = 1024;

// Pairs that span at most p.warp_items (kPwWarpItems) scorer CTAs -- short requests: one
// item -- are done by one warp per pair with no CTA barriers, in the same arithmetic as the
// CTA path (each item's rows folded from (-inf, 0), the item partials merged in item order;
// tests/test_gpu_scorer.py checks the two bitwise); the CTA path is left to pairs spread
// over more CTAs (measured: 2000 requests of 100 tokens, LLaMA layout, spent ~1 ms in
// per-task CTA barriers; 0.13 ms now).

__device__ __forceinline__ void pair_weights_run(const PairWeightsParams& p, int64_t t0, int64_t tstep, int nwarps,
                                                 float* sM, float* sL, int64_t* rb) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int R = p.num_requests, hpc = p.hpc, nhg = p.num_hgroups, npar = p.npar;
    Part P;
    P.cu_units = p.cu_units;
    P.R = R;
    P.nhg = nhg;
    P.U = static_cast<int64_t>(p.cu_units[R]) * nhg;
    P.grid = p.score_grid;
    if (P.U == 0) return;  // uniform across the CTA
    for (int c = threadIdx.x; c <= P.grid; c += blockDim.x) rb[c] = range_begin(P, c);
    __syncthreads();
    const int64_t tasks = static_cast<int64_t>(R) * nhg * hpc * 4;
    // ---- warp path: pairs spanning <= kPwWarpItems CTAs.  Warp task = one pair: its index
    // chain once, then its hpc * 4 (head, 32-row chunk) sub-tasks two at a time (both
    // sub-tasks' statistics loads in flight together).
    if (warp < nwarps) {
        const int64_t pairs = static_cast<int64_t>(R) * nhg;
        for (int64_t pr = t0 * nwarps + warp; pr < pairs; pr += tstep * nwarps) {
            const int r = static_cast<int>(pr / nhg), hg = static_cast<int>(pr - static_cast<int64_t>(r) * nhg);
            const int units_r = p.cu_units[r + 1] - p.cu_units[r];
            if (units_r == 0) continue;
            const int64_t seg_start = static_cast<int64_t>(p.cu_units[r]) * nhg + static_cast<int64_t>(hg) * units_r;
            const int c_first = cta_of(P, seg_start);
            const int n_items = cta_of(P, seg_start + units_r - 1) - c_first + 1;
            if (n_items > p.warp_items) continue;  // the CTA path below
            const int N = p.cu_seqlens[r + 1] - p.cu_seqlens[r];
            const int neff = min(p.query_window_n, N);
            int64_t sid[kPwWarpItems];
#pragma unroll
            for (int k = 0; k < kPwWarpItems; ++k) {
                sid[k] = -1;
                if (k < n_items) {
                    const int64_t b = rb[c_first + k];
                    sid[k] = (k > 0 && b == rb[c_first + k + 1]) ? -1 : (b > seg_start ? b : seg_start);
                }
            }
#pragma unroll 1
            for (int st = 0; st < hpc * 4; st += 2) {
                float mc[2][kPwWarpItems * 4], lc[2][kPwWarpItems * 4];
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const int hh = (st + x) >> 2, j = ((st + x) & 3) * 32 + lane;
#pragma unroll
                    for (int y = 0; y < kPwWarpItems * 4; ++y) {
                        const int k = y >> 2, q = y & 3;
                        const bool on = sid[k] >= 0 && q < npar;
                        const int64_t xx = ((sid[k] * hpc + hh) * npar + q) * kRows + j;
                        mc[x][y] = on ? __ldcg(&p.stat_m[xx]) : -INFINITY;
                        lc[x][y] = on ? __ldcg(&p.stat_l[xx]) : 0.f;
                    }
                }
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const int hh = (st + x) >> 2, j = ((st + x) & 3) * 32 + lane;
                    // each item's rows folded from (-inf, 0), then the items in order: the
                    // CTA path's arithmetic (one item per warp, warp partials in order)
                    float M = -INFINITY, L = 0.f;
#pragma unroll
                    for (int k = 0; k < kPwWarpItems; ++k) {
                        float Mk = -INFINITY, Lk = 0.f;
#pragma unroll
                        for (int q = 0; q < 4; ++q) lse_merge(Mk, Lk, mc[x][k * 4 + q], lc[x][k * 4 + q]);
                        lse_merge(M, L, Mk, Lk);
                    }
                    const int tile = p.q_tiles > 1 ? static_cast<int>((static_cast<int64_t>(hg) * hpc + hh) % p.q_tiles) : 0;
                    const int jr = p.q_pack > 1 ? j % (kRows / p.q_pack) : tile * kRows + j;  // window row
                    const bool valid = jr < neff;
                    if (valid && !(L > 0.f)) raise_error(p.err, kErrMaskedRow);
                    const float inv = valid && L > 0.f ? 1.f / (L * static_cast<float>(neff)) : 0.f;
#pragma unroll
                    for (int y = 0; y < kPwWarpItems * 4; ++y) {
                        const int k = y >> 2, q = y & 3;
                        if (sid[k] >= 0 && q < npar)
                            p.stat_w[((sid[k] * hpc + hh) * npar + q) * kRows + j] =
                                mc[x][y] != -INFINITY ? ex2_approx(mc[x][y] - M) * inv : 0.f;
                    }
                }
            }
        }
    }
    // ---- CTA path: pairs spread over many CTAs.  With many pairs (continuous batches of
    // short requests) the tasks are enumerated by candidate instead of by pair: a pair
    // spread over several CTAs holds the first unit of the range of every CTA after its
    // first, so the candidates are the pairs holding rb[c] (c < score_grid), each taken at
    // its smallest c -- grid * hpc * 4 tasks instead of a walk over every pair.
    const int64_t ctasks = static_cast<int64_t>(P.grid) * hpc * 4;
    // (candidates cover every pair over >= 2 CTAs; pairs inside one CTA need the warp path)
    const bool by_pair = tasks <= ctasks || p.warp_items < 1;
    const int64_t ntasks = by_pair ? tasks : ctasks;
    for (int64_t t = t0; t < ntasks; t += tstep) {
        const int chunk = static_cast<int>(t & 3);
        const int hh = static_cast<int>((t >> 2) % hpc);
        int r, hg, units_r;
        int64_t seg_start;
        if (by_pair) {
            const int64_t pair = (t >> 2) / hpc;
            r = static_cast<int>(pair / nhg);
            hg = static_cast<int>(pair - static_cast<int64_t>(r) * nhg);
            units_r = p.cu_units[r + 1] - p.cu_units[r];
            if (units_r == 0) continue;  // CTA-uniform
            seg_start = static_cast<int64_t>(p.cu_units[r]) * nhg + static_cast<int64_t>(hg) * units_r;
        } else {
            const int cand = static_cast<int>((t >> 2) / hpc);
            const int64_t pos = rb[cand];
            if (pos >= P.U) continue;  // CTA-uniform
            const Item at = make_item(P, pos, P.U);
            r = at.r;
            hg = at.hg;
            units_r = at.units_r;
            seg_start = at.seg_start;
            if (cand > 0 && rb[cand - 1] >= seg_start) continue;  // not the pair's first candidate
        }
        const int N = p.cu_seqlens[r + 1] - p.cu_seqlens[r];
        const int neff = min(p.query_window_n, N);
        const int64_t seg_end = seg_start + units_r;
        const int c_first = cta_of(P, seg_start);
        const int n_items = cta_of(P, seg_end - 1) - c_first + 1;  // CTAs spanned
        if (n_items <= p.warp_items) continue;  // done by the warp path (CTA-uniform)
        const int j = chunk * 32 + lane;
        // Item k = the part of the pair in CTA c_first + k; CTAs with empty ranges (more
        // CTAs than units) hold no item.
        auto sid_of = [&](int k) -> int64_t {
            const int64_t b = rb[c_first + k];
            if (k > 0 && b == rb[c_first + k + 1]) return -1;
            return b > seg_start ? b : seg_start;
        };
        // statistics rows of head hh: (sid * hpc + hh) * npar + par, par < npar <= 4 (the
        // parity warpgroups of score_tcw / score_tc2 keep separate running (m, l) for one
        // head).
        // KB items per warp step: all their loads are issued before the merges (a pair
        // spread over many CTAs -- one long request -- has ~148 items, so the merge is a
        // chain of L2 round trips unless many are in flight).
        constexpr int KB = 4;
        float M = -INFINITY, L = 0.f;
        for (int k = warp; warp < nwarps && k < n_items; k += KB * nwarps) {
            float mc[KB * 4], lc[KB * 4];
#pragma unroll
            for (int x = 0; x < KB; ++x) {
                const int kk = k + x * nwarps;
                const int64_t sid = kk < n_items ? sid_of(kk) : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    mc[x * 4 + q] = -INFINITY;
                    lc[x * 4 + q] = 0.f;
                    if (sid >= 0 && q < npar) {
                        const int64_t xx = ((sid * hpc + hh) * npar + q) * kRows + j;
                        mc[x * 4 + q] = __ldcg(&p.stat_m[xx]);
                        lc[x * 4 + q] = __ldcg(&p.stat_l[xx]);
                    }
                }
            }
#pragma unroll
            for (int y = 0; y < KB * 4; ++y) lse_merge(M, L, mc[y], lc[y]);
        }
        if (warp < nwarps) {
            sM[warp * 32 + lane] = M;
            sL[warp * 32 + lane] = L;
        }
        __syncthreads();
        if (warp == 0) {  // one warp merges the warp partials (in warp order) for every warp
            M = -INFINITY;
            L = 0.f;
            for (int w = 0; w < nwarps; ++w) lse_merge(M, L, sM[w * 32 + lane], sL[w * 32 + lane]);
            sM[lane] = M;
            sL[lane] = L;
        }
        __syncthreads();
        M = sM[lane];
        L = sL[lane];
        __syncthreads();  // sM / sL are rewritten by the next task
        // row j of this virtual head's query tile is window row 128 t + j
        const int tile = p.q_tiles > 1 ? static_cast<int>((static_cast<int64_t>(hg) * hpc + hh) % p.q_tiles) : 0;
        const int jr = p.q_pack > 1 ? j % (kRows / p.q_pack) : tile * kRows + j;  // window row
        const bool valid = jr < neff;
        if (valid && !(L > 0.f) && warp == 0) raise_error(p.err, kErrMaskedRow);
        const float inv = valid && L > 0.f ? 1.f / (L * static_cast<float>(neff)) : 0.f;
        for (int k = warp; warp < nwarps && k < n_items; k += KB * nwarps) {
            int64_t xs[KB * 4];
            float mc[KB * 4];
#pragma unroll
            for (int x = 0; x < KB; ++x) {
                const int kk = k + x * nwarps;
                const int64_t sid = kk < n_items ? sid_of(kk) : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    xs[x * 4 + q] = sid >= 0 && q < npar ? ((sid * hpc + hh) * npar + q) * kRows + j : -1;
                    mc[x * 4 + q] = xs[x * 4 + q] >= 0 ? __ldcg(&p.stat_m[xs[x * 4 + q]]) : -INFINITY;
                }
            }
#pragma unroll
            for (int y = 0; y < KB * 4; ++y)
                if (xs[y] >= 0) p.stat_w[xs[y]] = mc[y] != -INFINITY ? ex2_approx(mc[y] - M) * inv : 0.f;
        }
    }
}

// Warp per block: b_g = (1/|g|) Σ_h Σ_j P[h][g][j] w[item(h,g)][hh][j].
// With num_shards = T > 1 the heads form T contiguous shards (sharded_block_scores,
// tp_sim.cpp:12-27): each shard's partial b_g^t is formed on its own (written to
// shard_scores[t] when non-null) and block_scores[g] = ((0 + b^0) + b^1) + ... in fp32,
// ascending shard order (allreduce_scores, tp_sim.cpp:43-47).
// Global warps gw0, gw0 + gwstep, ... each take one block below min(limit, #blocks); the
// block's score goes to out(gb, value) (lane 0) -- by default block_scores[gb].
struct StoreBlockScore {
    float* block_scores;
    __device__ __forceinline__ void operator()(int gb, float v) const { block_scores[gb] = v; }
};

template <class Out = StoreBlockScore>
__device__ __forceinline__ void block_combine_run(const BlockCombineParams& p, int64_t gw0, int64_t gwstep,
                                                  int64_t limit = INT64_MAX, Out out = Out{nullptr}) {
    if constexpr (std::is_same_v<Out, StoreBlockScore>) out.block_scores = p.block_scores;
    const int lane = threadIdx.x & 31;
    const int R = p.num_requests;
    const int total = p.cu_blocks[R] < limit ? p.cu_blocks[R] : static_cast<int>(limit);
    const int nhg = p.num_heads / p.hpc;
    const int T = p.num_shards;
    const int hps = p.num_heads / T;  // heads per shard (a multiple of hpc)
    for (int64_t gbl = gw0; gbl < total; gbl += gwstep) {
        const int gb = static_cast<int>(gbl);
        const int r = find_segment(p.cu_blocks, R, gb);
        const int units_r = p.cu_units[r + 1] - p.cu_units[r];
        if (units_r == 0) {  // pass-through segment
            if (lane == 0) {
                out(gb, 0.f);
                if (p.shard_scores != nullptr)
                    for (int t = 0; t < T; ++t) p.shard_scores[static_cast<int64_t>(t) * p.shard_stride + gb] = 0.f;
            }
            continue;
        }
        const int g = gb - p.cu_blocks[r];
        const int N = p.cu_seqlens[r + 1] - p.cu_seqlens[r];
        const int size = min(p.block_size_g, N - g * p.block_size_g);
        const int u = (g * p.block_size_g) / p.unit_keys;
        const int64_t pair0 = static_cast<int64_t>(p.cu_units[r]) * nhg;
        // statistics row of head hh: hh * npar + parity, the parity of the unit's first
        // subtile (top bits of unit_sid) plus the block's offset in the unit in parity units
        // (64 keys in score_tcw, 128 in score_tc2 / score_tcw at G = 128)
        const int poff = ((g * p.block_size_g) % p.unit_keys) >> p.par_shift;
        const int hpcv = p.hpc * p.npar;
        if (T > 1) {
            // Sharded: every head's dot product is reduced across the warp and added, in
            // head order, to its shard's sum held by lane t = h / hps; loads of 8 heads
            // are in flight together.
            float shard_acc = 0.f;
            for (int hg0 = 0; hg0 < nhg; hg0 += 32) {
                const int my_hg = hg0 + lane;
                const int my_sid = my_hg < nhg ? p.unit_sid[pair0 + static_cast<int64_t>(my_hg) * units_r + u] : 0;
                const int h_end = min(p.num_heads, (hg0 + 32) * p.hpc);
                for (int h = hg0 * p.hpc; h < h_end; h += 8) {
                    float d[8];
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        const int hx = min(h + x, h_end - 1);
                        const int hgx = hx / p.hpc;
                        const int32_t us = __shfl_sync(0xffffffffu, my_sid, hgx - hg0);
                        const int64_t sid = usid_item(us);
                        const int par = usid_par(us, poff, p.npar);
                        const float4 pv = __ldcs(reinterpret_cast<const float4*>(
                            p.P + (static_cast<int64_t>(hx) * p.max_blocks + gb) * kRows) + lane);
                        const float4 wv = __ldg(reinterpret_cast<const float4*>(
                            p.stat_w + (sid * hpcv + (hx - hgx * p.hpc) * p.npar + par) * kRows) + lane);
                        d[x] = fmaf(pv.x, wv.x, fmaf(pv.y, wv.y, fmaf(pv.z, wv.z, pv.w * wv.w)));
                    }
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        if (h + x >= h_end) break;
                        float v = d[x];
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        if (lane == (h + x) / hps) shard_acc += v;
                    }
                }
            }
            const float bt = shard_acc / static_cast<float>(size);
            if (p.shard_scores != nullptr && lane < T) p.shard_scores[static_cast<int64_t>(lane) * p.shard_stride + gb] = bt;
            float red = 0.f;
            for (int t = 0; t < T; ++t) red += __shfl_sync(0xffffffffu, bt, t);  // ascending shard order
            if (lane == 0) out(gb, red);
            continue;
        }
        // Unsharded: heads in chunks of 8 (one batch of loads in flight), per chunk an FMA
        // chain per head slot, a fixed tree and a warp sum, the chunk sums added in order --
        // the same arithmetic as block_combine_chunked (so the peer-fused combine, which runs
        // this path, stays bitwise the ascending sum of the plain scorer's partials).
        float red = 0.f;
        // item ids of up to 32 head groups, one per lane, broadcast by shuffles (one
        // round trip ahead of the chunks instead of one per chunk)
        const int my_sid = lane < nhg ? p.unit_sid[pair0 + static_cast<int64_t>(lane) * units_r + u] : 0;
        for (int h0 = 0; h0 < p.num_heads; h0 += 8) {
            const int h1 = min(h0 + 8, p.num_heads);
            float4 pv[8], wv[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                const int hx = min(h0 + x, h1 - 1);
                const int hgx = hx / p.hpc;
#ifdef UP_COMBINE_SID_PER_HEAD  // dev A/B
                const int32_t us = p.unit_sid[pair0 + static_cast<int64_t>(hgx) * units_r + u];
#else
                const int32_t us = nhg <= 32 ? __shfl_sync(0xffffffffu, my_sid, hgx & 31)
                                             : p.unit_sid[pair0 + static_cast<int64_t>(hgx) * units_r + u];
#endif
                const int64_t sid = usid_item(us);
                const int par = usid_par(us, poff, p.npar);
                pv[x] = __ldcs(reinterpret_cast<const float4*>(p.P + (static_cast<int64_t>(hx) * p.max_blocks + gb) * kRows) + lane);
                wv[x] = __ldg(reinterpret_cast<const float4*>(
                            p.stat_w + (sid * hpcv + (hx - hgx * p.hpc) * p.npar + par) * kRows) + lane);
            }
            float acc[8];
#pragma unroll
            for (int x = 0; x < 8; ++x)
                acc[x] = h0 + x < h1 ? fmaf(pv[x].x, wv[x].x, fmaf(pv[x].y, wv[x].y, fmaf(pv[x].z, wv[x].z, pv[x].w * wv[x].w)))
                                     : 0.f;
            float part = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            red += part;
        }
        const float bt = red / static_cast<float>(size);
        if (p.shard_scores != nullptr && lane == 0) p.shard_scores[gb] = bt;
        if (lane == 0) out(gb, bt);
    }
}

// Unsharded combine with the heads of a block split over NCH warps of the CTA (8 heads per
// warp, one batch of loads in flight each), for Hq <= 64: a block's 32 heads cost one L2
// round trip instead of four.  The warp partials are added in chunk order by the block's
// first warp (deterministic).  blockDim = 256: 8 / NCH blocks per CTA step.
__device__ __forceinline__ void block_combine_chunked(const BlockCombineParams& p, float* s_part) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int R = p.num_requests;
    const int total = p.cu_blocks[R];
    const int nhg = p.num_heads / p.hpc;
    const int nch = (p.num_heads + 7) / 8;           // head chunks per block (<= 8)
    const int bpc = 8 / nch;                          // blocks per CTA step
    const int bl = warp / nch, ch = warp - bl * nch;  // this warp's block slot and chunk
    const int hpcv = p.hpc * p.npar;
    for (int64_t gb0 = static_cast<int64_t>(blockIdx.x) * bpc; gb0 < total; gb0 += static_cast<int64_t>(gridDim.x) * bpc) {
        const int64_t gbl = gb0 + bl;
        float part = 0.f;
        int size = 1;
        bool pass = false;
        if (bl < bpc && gbl < total) {
            const int gb = static_cast<int>(gbl);
            const int r = find_segment(p.cu_blocks, R, gb);
            const int units_r = p.cu_units[r + 1] - p.cu_units[r];
            pass = units_r == 0;
            if (!pass) {
                const int g = gb - p.cu_blocks[r];
                const int N = p.cu_seqlens[r + 1] - p.cu_seqlens[r];
                size = min(p.block_size_g, N - g * p.block_size_g);
                const int u = (g * p.block_size_g) / p.unit_keys;
                const int64_t pair0 = static_cast<int64_t>(p.cu_units[r]) * nhg;
                const int poff = ((g * p.block_size_g) % p.unit_keys) >> p.par_shift;
                const int h0 = ch * 8, h1 = min(h0 + 8, p.num_heads);
                float4 pv[8], wv[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const int hx = min(h0 + x, h1 - 1);
                    const int hgx = hx / p.hpc;
                    const int32_t us = p.unit_sid[pair0 + static_cast<int64_t>(hgx) * units_r + u];
                    const int64_t sid = usid_item(us);
                    const int par = usid_par(us, poff, p.npar);
                    pv[x] = __ldcs(reinterpret_cast<const float4*>(p.P + (static_cast<int64_t>(hx) * p.max_blocks + gb) * kRows) + lane);
                    wv[x] = __ldg(reinterpret_cast<const float4*>(
                                p.stat_w + (sid * hpcv + (hx - hgx * p.hpc) * p.npar + par) * kRows) + lane);
                }
                float acc[8];
#pragma unroll
                for (int x = 0; x < 8; ++x)
                    acc[x] = h0 + x < h1 ? fmaf(pv[x].x, wv[x].x, fmaf(pv[x].y, wv[x].y, fmaf(pv[x].z, wv[x].z, pv[x].w * wv[x].w)))
                                         : 0.f;
                part = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            }
        }
        if (lane == 0) s_part[warp] = part;
        __syncthreads();
        if (ch == 0 && lane == 0 && bl < bpc && gbl < total) {
            float a = 0.f;
            for (int c = 0; c < nch; ++c) a += s_part[bl * nch + c];
            p.block_scores[gbl] = pass ? 0.f : a / static_cast<float>(size);
        }
        __syncthreads();
    }
}

}  // namespace up
