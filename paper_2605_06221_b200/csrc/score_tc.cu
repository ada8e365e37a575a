// score_tc.cu -- block-wise importance scorer on tcgen05 tensor cores (sm_100a).
//
// Computes, for every drop-enabled request r of a varlen batch and every local q-head h,
// the reference's block scores (importance.cpp:92-132):
//
//   raw(j,i) = q_j . k_i / sqrt(D), masked for i > N - n_eff + j         (:17-33)
//   A(j,i)   = softmax_i(raw(j,.)) over the full key range                (:35-74)
//   b_g      = (1/|g|) Σ_{i∈g} Σ_h (1/n_eff) Σ_j A_h(j,i)                 (:76-90)
//
// in one pass over K (no second QK^T for normalisation):
//
//  * score_tc_kernel (persistent, warp-specialised).  A work item is (request, key chunk,
//    group of HPC q-heads sharing one kv-head).  Warp 0 streams K tiles with TMA into a
//    2-stage SWIZZLE_128B ring (Q tiles of the HPC heads stay resident); warp 1 issues
//    tcgen05.mma (M=128 query rows x N=128 keys x K=D, bf16 -> fp32 in TMEM, one region of
//    128 TMEM columns per (tile, head), 4 regions); warps 2..9 (two warpgroups, thread =
//    query row) drain TMEM and compute e = 2^(s*log2e/sqrt(D) - m) against a per-(row,
//    chunk) reference m that is only moved when a value would exceed it by 2^20 (rare;
//    the already-written partials of the chunk are rescaled then).  Per (row, block) the
//    partial Σ e goes to P, per (row, chunk) (m, l = Σ e) to the stats.
//  * row_weights_kernel: per (request, head, row) the global max M and denominator
//    L = Σ_c l_c 2^(m_c - M) over chunks -> weight w_c = 2^(m_c - M) / (L n_eff).
//  * block_combine_kernel: b_g = (1/|g|) Σ_h Σ_j P[h][g][j] w[h][c(g)][j] (warp per block).
#include "params.cuh"

namespace up {

struct ItemInfo {
    int r, c, hg;
    int seg0, N, neff, key0, klen, ntiles;
};

__device__ __forceinline__ ItemInfo decode_item(const ScoreTcParams& p, int item, int chunk_keys) {
    ItemInfo it;
    it.r = find_segment(p.cu_items, p.num_requests, item);
    const int local = item - p.cu_items[it.r];
    it.c = local / p.num_hgroups;
    it.hg = local - it.c * p.num_hgroups;
    it.seg0 = p.cu_seqlens[it.r];
    it.N = p.cu_seqlens[it.r + 1] - it.seg0;
    it.neff = min(p.query_window_n, it.N);
    it.key0 = it.c * chunk_keys;
    it.klen = min(chunk_keys, it.N - it.key0);
    it.ntiles = (it.klen + kTileKeys - 1) / kTileKeys;
    return it;
}

// Device-side work plan (no host knowledge of segment lengths needed): validates
// cu_seqlens, writes cu_blocks, picks the key-chunk length and enumerates work items.
__global__ void score_plan_kernel(const int32_t* __restrict__ cu, const uint8_t* __restrict__ en,
                                  int R, int64_t max_tokens, int G, int unit_tiles, int nhg,
                                  int target_items, int32_t* __restrict__ cu_blocks,
                                  int32_t* __restrict__ cu_chunks, int32_t* __restrict__ cu_items,
                                  int32_t* __restrict__ plan, uint32_t* __restrict__ err) {
    if (threadIdx.x != 0) return;
    bool ok = cu[0] == 0;
    int64_t tiles = 0;
    for (int r = 0; r < R && ok; ++r) {
        const int64_t n = static_cast<int64_t>(cu[r + 1]) - cu[r];
        if (n <= 0) ok = false;
        if (en == nullptr || en[r]) tiles += (n + kTileKeys - 1) / kTileKeys;
    }
    if (ok && cu[R] > max_tokens) ok = false;
    if (!ok) {
        raise_error(err, kErrBadSeqlens);
        for (int r = 0; r <= R; ++r) { cu_blocks[r] = 0; cu_chunks[r] = 0; cu_items[r] = 0; }
        plan[0] = unit_tiles * kTileKeys;
        plan[1] = 0;
        return;
    }
    int64_t chunk_tiles = (tiles * nhg + target_items - 1) / target_items;
    if (chunk_tiles < 1) chunk_tiles = 1;
    if (chunk_tiles > 64) chunk_tiles = 64;
    chunk_tiles = (chunk_tiles + unit_tiles - 1) / unit_tiles * unit_tiles;
    const int chunk_keys = static_cast<int>(chunk_tiles) * kTileKeys;
    int32_t b = 0, c = 0, it = 0;
    for (int r = 0; r < R; ++r) {
        cu_blocks[r] = b; cu_chunks[r] = c; cu_items[r] = it;
        const int n = cu[r + 1] - cu[r];
        b += (n + G - 1) / G;
        if (en == nullptr || en[r]) {
            const int nc = (n + chunk_keys - 1) / chunk_keys;
            c += nc;
            it += nc * nhg;
        }
    }
    cu_blocks[R] = b; cu_chunks[R] = c; cu_items[R] = it;
    plan[0] = chunk_keys;
    plan[1] = it;
}

template <int D, int HPC>
struct TcCfg {
    static constexpr int KC = D / 64;                 // 128-byte K-chunks per row
    static constexpr int SUB = 128 * 128;             // bytes of one [128 rows x 64 bf16] tile
    static constexpr int Q_BYTES = HPC * KC * SUB;
    static constexpr int K_STAGE = KC * SUB;
    static constexpr int KST = 2;
    static constexpr int NREG = 4;                    // TMEM regions of 128 columns
    static constexpr int NSLOT = HPC >= 2 ? HPC / 2 : 1;
    static constexpr int NBAR = 2 + 2 * KST + 2 * NREG;
    static constexpr int SMEM = Q_BYTES + KST * K_STAGE + NBAR * 8 + 16 + 1024;
    static constexpr int THREADS = 320;
};

template <int D, int HPC>
__global__ void __launch_bounds__(320, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                const ScoreTcParams p) {
    using C = TcCfg<D, HPC>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sq = smem;
    uint8_t* sk = smem + C::Q_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sk + C::KST * C::K_STAGE);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;
    uint64_t* k_empty = bars + 2 + C::KST;
    uint64_t* t_full = bars + 2 + 2 * C::KST;
    uint64_t* t_empty = bars + 2 + 2 * C::KST + C::NREG;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int s = 0; s < C::KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < C::NREG; ++s) { mbar_init(&t_full[s], 1); mbar_init(&t_empty[s], 4); }
        fence_barrier_init();
        prefetch_tensormap(&qmap);
        prefetch_tensormap(&kmap);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int chunk_keys = p.plan[0];
    const int total_items = p.plan[1];

    if (warp == 0) {
        // ===== TMA producer =====
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t qiter = 0;
            for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
                const ItemInfo it = decode_item(p, item, chunk_keys);
                const int kv_local =
                    (p.q_head_offset + it.hg * HPC) / p.gqa_group - p.kv_head_offset;
                mbar_wait(q_empty, (qiter & 1) ^ 1);
                ++qiter;
                mbar_arrive_expect_tx(q_full, C::Q_BYTES);
                const int qrow = it.seg0 + it.N - it.neff;
#pragma unroll
                for (int hh = 0; hh < HPC; ++hh) {
#pragma unroll
                    for (int kc = 0; kc < C::KC; ++kc) {
                        tma_load_2d(sq + (hh * C::KC + kc) * C::SUB, &qmap, q_full,
                                    (it.hg * HPC + hh) * D + kc * 64, qrow);
                    }
                }
                for (int t = 0; t < it.ntiles; ++t) {
                    mbar_wait(&k_empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&k_full[stage], C::K_STAGE);
                    const int krow = it.seg0 + it.key0 + t * kTileKeys;
#pragma unroll
                    for (int kc = 0; kc < C::KC; ++kc) {
                        tma_load_2d(sk + stage * C::K_STAGE + kc * C::SUB, &kmap, &k_full[stage],
                                    kv_local * D + kc * 64, krow);
                    }
                    if (++stage == C::KST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (single thread) =====
        if (elect_one()) {
            constexpr uint32_t kIdesc = idesc_bf16_f32(128, kTileKeys);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t qiter = 0;
            uint32_t seq = 0;
            const uint32_t sq_addr = smem_u32(sq);
            const uint32_t sk_addr = smem_u32(sk);
            for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
                const ItemInfo it = decode_item(p, item, chunk_keys);
                mbar_wait(q_full, qiter & 1);
                ++qiter;
                tc_fence_after();
                for (int t = 0; t < it.ntiles; ++t) {
                    mbar_wait(&k_full[stage], phase);
                    tc_fence_after();
#pragma unroll
                    for (int hh = 0; hh < HPC; ++hh) {
                        const uint32_t reg = seq % C::NREG;
                        mbar_wait(&t_empty[reg], ((seq / C::NREG) & 1) ^ 1);
                        tc_fence_after();
                        const uint32_t d_tmem = tmem_base + reg * kTileKeys;
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t off = (kk >> 2) * C::SUB + (kk & 3) * 32;
                            const uint64_t a = smem_desc_sw128(sq_addr + hh * C::KC * C::SUB + off);
                            const uint64_t b = smem_desc_sw128(sk_addr + stage * C::K_STAGE + off);
                            mma_bf16_ss(d_tmem, a, b, kIdesc, kk > 0 ? 1u : 0u);
                        }
                        mma_commit(&t_full[reg]);
                        ++seq;
                    }
                    mma_commit(&k_empty[stage]);
                    if (++stage == C::KST) { stage = 0; phase ^= 1; }
                }
                mma_commit(q_empty);
            }
        }
    } else {
        // ===== epilogue: two warpgroups, thread = query row =====
        const int wg = (warp - 2) >> 2;
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int j = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const float sc = p.scale_log2;
        const int G = p.block_size_g;
        uint32_t seq = 0;
        for (int item = blockIdx.x; item < total_items; item += gridDim.x) {
            const ItemInfo it = decode_item(p, item, chunk_keys);
            const bool row_valid = j < it.neff;
            const int qpos = it.N - it.neff + j;  // last key this row may see (segment-relative)
            const int gc = p.cu_chunks[it.r] + it.c;
            const int64_t gb_seg = p.cu_blocks[it.r];  // global index of the segment's block 0
            const int blk_chunk0 = it.key0 / G;
            float m[C::NSLOT], l[C::NSLOT], bsum[C::NSLOT];
#pragma unroll
            for (int s = 0; s < C::NSLOT; ++s) { m[s] = -INFINITY; l[s] = 0.f; bsum[s] = 0.f; }

            for (int t = 0; t < it.ntiles; ++t) {
                const int colbase = it.key0 + t * kTileKeys;
                const bool tail = colbase + kTileKeys - 1 > it.N - it.neff;  // warp-uniform
#pragma unroll
                for (int hh = 0; hh < HPC; ++hh) {
                    const bool mine = HPC == 1 ? (wg == 0) : ((hh & 1) == wg);
                    if (mine) {
                        const int slot = HPC >= 2 ? hh / 2 : 0;
                        const int h_local = it.hg * HPC + hh;
                        const uint32_t reg = seq % C::NREG;
                        mbar_wait(&t_full[reg], (seq / C::NREG) & 1);
                        tc_fence_after();
                        float* Prow = p.P + (static_cast<int64_t>(h_local) * p.max_blocks + gb_seg) * kRows + j;
#pragma unroll 1
                        for (int q4 = 0; q4 < kTileKeys / 32; ++q4) {
                            const int c0 = colbase + q4 * 32;
                            if (c0 >= it.N) break;  // warp-uniform
                            uint32_t v[32];
                            tmem_ld32(tmem_base + lane_base + reg * kTileKeys + q4 * 32, v);
                            tmem_ld_wait();
                            const float mneg = -m[slot];
                            float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
                            if (!tail) {
#pragma unroll
                                for (int k = 0; k < 32; k += 4) {
                                    acc0 += ex2_approx(fmaf(__uint_as_float(v[k + 0]), sc, mneg));
                                    acc1 += ex2_approx(fmaf(__uint_as_float(v[k + 1]), sc, mneg));
                                    acc2 += ex2_approx(fmaf(__uint_as_float(v[k + 2]), sc, mneg));
                                    acc3 += ex2_approx(fmaf(__uint_as_float(v[k + 3]), sc, mneg));
                                }
                            } else {
#pragma unroll
                                for (int k = 0; k < 32; k += 4) {
                                    const float e0 = ex2_approx(fmaf(__uint_as_float(v[k + 0]), sc, mneg));
                                    const float e1 = ex2_approx(fmaf(__uint_as_float(v[k + 1]), sc, mneg));
                                    const float e2 = ex2_approx(fmaf(__uint_as_float(v[k + 2]), sc, mneg));
                                    const float e3 = ex2_approx(fmaf(__uint_as_float(v[k + 3]), sc, mneg));
                                    acc0 += (c0 + k + 0 <= qpos) ? e0 : 0.f;
                                    acc1 += (c0 + k + 1 <= qpos) ? e1 : 0.f;
                                    acc2 += (c0 + k + 2 <= qpos) ? e2 : 0.f;
                                    acc3 += (c0 + k + 3 <= qpos) ? e3 : 0.f;
                                }
                            }
                            float gs = (acc0 + acc1) + (acc2 + acc3);
                            if (!(gs <= 0x1p20f)) {
                                // Rebase: the reference for this (row, chunk) moves to the max seen.
                                float gmax = -INFINITY;
#pragma unroll
                                for (int k = 0; k < 32; ++k) {
                                    const bool valid = !tail || (c0 + k <= qpos);
                                    if (valid) gmax = fmaxf(gmax, __uint_as_float(v[k]) * sc);
                                }
                                const float mold = m[slot];
                                const float mnew = fmaxf(mold, gmax);
                                if (mold != -INFINITY) {
                                    const float f = ex2_approx(mold - mnew);
                                    l[slot] *= f;
                                    bsum[slot] *= f;
                                    const int cur_blk = c0 / G;
                                    for (int g = blk_chunk0; g < cur_blk; ++g) Prow[static_cast<int64_t>(g) * kRows] *= f;
                                }
                                m[slot] = mnew;
                                gs = 0.f;
#pragma unroll
                                for (int k = 0; k < 32; ++k) {
                                    const bool valid = !tail || (c0 + k <= qpos);
                                    const float e = ex2_approx(fmaf(__uint_as_float(v[k]), sc, -mnew));
                                    gs += valid ? e : 0.f;
                                }
                            }
                            bsum[slot] += gs;
                            if (((c0 + 32) % G) == 0 || c0 + 32 >= it.N) {
                                Prow[static_cast<int64_t>(c0 / G) * kRows] = row_valid ? bsum[slot] : 0.f;
                                l[slot] += bsum[slot];
                                bsum[slot] = 0.f;
                            }
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&t_empty[reg]);
                    }
                    ++seq;
                }
            }
            // Chunk statistics for the owned heads.
#pragma unroll
            for (int hh = 0; hh < HPC; ++hh) {
                const bool mine = HPC == 1 ? (wg == 0) : ((hh & 1) == wg);
                if (mine) {
                    const int slot = HPC >= 2 ? hh / 2 : 0;
                    const int h_local = it.hg * HPC + hh;
                    const int64_t si = (static_cast<int64_t>(h_local) * p.max_chunks + gc) * kRows + j;
                    p.stat_m[si] = row_valid ? m[slot] : -INFINITY;
                    p.stat_l[si] = row_valid ? l[slot] : 0.f;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// Per (request, head, row): combine chunk statistics into per-chunk weights.
__global__ void row_weights_kernel(const int32_t* __restrict__ cu, const uint8_t* __restrict__ en,
                                   const int32_t* __restrict__ cu_chunks,
                                   const float* __restrict__ stat_m, const float* __restrict__ stat_l,
                                   float* __restrict__ stat_w, int n, int64_t max_chunks,
                                   uint32_t* __restrict__ err) {
    const int r = blockIdx.x;
    const int h = blockIdx.y;
    const int j = threadIdx.x;
    if (en != nullptr && !en[r]) return;
    const int N = cu[r + 1] - cu[r];
    const int neff = min(n, N);
    const int c0 = cu_chunks[r], c1 = cu_chunks[r + 1];
    const int64_t base = static_cast<int64_t>(h) * max_chunks * kRows + j;
    float M = -INFINITY;
    for (int c = c0; c < c1; ++c) M = fmaxf(M, stat_m[base + static_cast<int64_t>(c) * kRows]);
    float L = 0.f;
    for (int c = c0; c < c1; ++c) {
        const float mc = stat_m[base + static_cast<int64_t>(c) * kRows];
        if (mc != -INFINITY) L += stat_l[base + static_cast<int64_t>(c) * kRows] * ex2_approx(mc - M);
    }
    const bool valid = j < neff;
    if (valid && !(L > 0.f)) raise_error(err, kErrMaskedRow);
    const float inv = valid && L > 0.f ? 1.f / (L * static_cast<float>(neff)) : 0.f;
    for (int c = c0; c < c1; ++c) {
        const float mc = stat_m[base + static_cast<int64_t>(c) * kRows];
        stat_w[base + static_cast<int64_t>(c) * kRows] = (mc != -INFINITY) ? ex2_approx(mc - M) * inv : 0.f;
    }
}

// Warp per block: b_g = (1/|g|) Σ_h Σ_j P[h][g][j] w[h][c(g)][j].
__global__ void block_combine_kernel(const int32_t* __restrict__ cu, const uint8_t* __restrict__ en,
                                     const int32_t* __restrict__ cu_blocks,
                                     const int32_t* __restrict__ cu_chunks,
                                     const int32_t* __restrict__ plan, const float* __restrict__ P,
                                     const float* __restrict__ stat_w, float* __restrict__ block_scores,
                                     int R, int G, int num_heads, int64_t max_blocks,
                                     int64_t max_chunks) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total = cu_blocks[R];
    const int chunk_keys = plan[0];
    for (int gb = blockIdx.x * (blockDim.x >> 5) + warp; gb < total; gb += gridDim.x * (blockDim.x >> 5)) {
        const int r = find_segment(cu_blocks, R, gb);
        if (en != nullptr && !en[r]) {
            if (lane == 0) block_scores[gb] = 0.f;
            continue;
        }
        const int g = gb - cu_blocks[r];
        const int N = cu[r + 1] - cu[r];
        const int gc = cu_chunks[r] + (g * G) / chunk_keys;
        const int size = min(G, N - g * G);
        float acc = 0.f;
        for (int h = 0; h < num_heads; ++h) {
            const float4 pv = *reinterpret_cast<const float4*>(
                P + (static_cast<int64_t>(h) * max_blocks + gb) * kRows + lane * 4);
            const float4 wv = *reinterpret_cast<const float4*>(
                stat_w + (static_cast<int64_t>(h) * max_chunks + gc) * kRows + lane * 4);
            acc += pv.x * wv.x + pv.y * wv.y + pv.z * wv.z + pv.w * wv.w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) block_scores[gb] = acc / static_cast<float>(size);
    }
}

// ---------------------------------------------------------------- host launchers
template <int D, int HPC>
static cudaError_t launch_tc(const CUtensorMap& qm, const CUtensorMap& km, const ScoreTcParams& p,
                             int grid, cudaStream_t stream) {
    using C = TcCfg<D, HPC>;
    cudaError_t e = cudaFuncSetAttribute(score_tc_kernel<D, HPC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    score_tc_kernel<D, HPC><<<grid, C::THREADS, C::SMEM, stream>>>(qm, km, p);
    return cudaGetLastError();
}

int tc_max_hpc(int D) { return D == 64 ? 8 : (D == 128 ? 4 : 1); }

cudaError_t launch_score_tc(int D, int HPC, const CUtensorMap& qm, const CUtensorMap& km,
                            const ScoreTcParams& p, int grid, cudaStream_t stream) {
#define UP_TC_CASE(d, h) \
    if (D == d && HPC == h) return launch_tc<d, h>(qm, km, p, grid, stream);
    UP_TC_CASE(64, 1) UP_TC_CASE(64, 2) UP_TC_CASE(64, 4) UP_TC_CASE(64, 8)
    UP_TC_CASE(128, 1) UP_TC_CASE(128, 2) UP_TC_CASE(128, 4)
    UP_TC_CASE(256, 1)
#undef UP_TC_CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_score_plan(const int32_t* cu, const uint8_t* en, int R, int64_t max_tokens,
                              int G, int unit_tiles, int nhg, int target_items, int32_t* cu_blocks,
                              int32_t* cu_chunks, int32_t* cu_items, int32_t* plan, uint32_t* err,
                              cudaStream_t stream) {
    score_plan_kernel<<<1, 32, 0, stream>>>(cu, en, R, max_tokens, G, unit_tiles, nhg, target_items,
                                            cu_blocks, cu_chunks, cu_items, plan, err);
    return cudaGetLastError();
}

cudaError_t launch_row_weights(const int32_t* cu, const uint8_t* en, const int32_t* cu_chunks,
                               const float* stat_m, const float* stat_l, float* stat_w, int R,
                               int num_heads, int n, int64_t max_chunks, uint32_t* err,
                               cudaStream_t stream) {
    row_weights_kernel<<<dim3(R, num_heads), kRows, 0, stream>>>(cu, en, cu_chunks, stat_m, stat_l,
                                                                 stat_w, n, max_chunks, err);
    return cudaGetLastError();
}

cudaError_t launch_block_combine(const int32_t* cu, const uint8_t* en, const int32_t* cu_blocks,
                                 const int32_t* cu_chunks, const int32_t* plan, const float* P,
                                 const float* stat_w, float* block_scores, int R, int G,
                                 int num_heads, int64_t max_blocks, int64_t max_chunks, int grid,
                                 cudaStream_t stream) {
    block_combine_kernel<<<grid, 256, 0, stream>>>(cu, en, cu_blocks, cu_chunks, plan, P, stat_w,
                                                   block_scores, R, G, num_heads, max_blocks,
                                                   max_chunks);
    return cudaGetLastError();
}

}  // namespace up
