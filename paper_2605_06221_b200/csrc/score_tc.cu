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
//  * score_tc_kernel -- persistent, one CTA per SM, warp-specialised.
//    Work decomposition: the key range of every (request, head-group) pair is cut into
//    units of lcm(G,128) keys; the flattened sequence of (request, head-group, unit) is
//    split into gridDim.x contiguous, equal ranges (exact load balance for any mix of
//    lengths), so a CTA reloads Q only when its range crosses into the next pair.  The
//    plan is computed in every CTA's prologue from the device-resident cu_seqlens (no
//    host round trip); CTA 0 publishes cu_blocks.
//    Warp 0 streams K tiles with TMA into a 2-stage SWIZZLE_128B ring while the Q tiles of
//    the HPC heads of one kv-head stay resident; warp 1 issues tcgen05.mma (M=128 query
//    rows x N=128 keys x K=D, bf16 -> fp32 in TMEM, 4 regions of 128 columns); warps 2..9
//    (two warpgroups, thread = query row, alternating heads) drain TMEM and compute
//    e = 2^(s*log2e/sqrt(D) - m) against a per-(row, item) reference m that moves only
//    when a value would exceed it by ~2^20 (rare; the item's already-written partials are
//    rescaled then).  Per (row, block) Σ e goes to P, per (row, item) (m, l = Σ e) to the
//    stats.  This kernel serves the shapes score_tcw.cu does not (HPC 1 or 8, block
//    sizes other than 32/64 at two heads per CTA, more than 256 segments).
//  * pair_weights_kernel (score_tail.cuh) -- per (request, head-group) pair, the items'
//    statistics become row weights w = 2^(m - M) / (L n_eff), M = max_items m,
//    L = Σ_items l 2^(m - M);
//  * block_combine_kernel (score_tail.cuh) -- b_g = (1/|g|) Σ_h Σ_j P[h][g][j] w[item(h,g)][j].
#include <cstdlib>
#include "score_tail.cuh"
#include "peer.cuh"

namespace up {

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
    static constexpr int FIXED = Q_BYTES + KST * K_STAGE + NBAR * 8 + 64 + 1024;
    static constexpr int THREADS = 320;
    static int smem(int R) { return FIXED + 5 * NSLOT * 256 * 4 + 2 * (R + 1) * 4; }
};


template <int D, int HPC>
__global__ void __launch_bounds__(320, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                const ScoreTcParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
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
    uint32_t* misc = reinterpret_cast<uint32_t*>(bars + C::NBAR);  // [0] tmem base, [1] flag, [2] last
    float* s_state = reinterpret_cast<float*>(misc + 16);  // [5][NSLOT][256] epilogue state
    int32_t* s_cu_units = reinterpret_cast<int32_t*>(s_state + 5 * C::NSLOT * 256);
    int32_t* s_cu_blocks = s_cu_units + (p.num_requests + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int R = p.num_requests;
    const int G = p.block_size_g;
    const int unit_keys = p.unit_keys;
    unsigned long long t_start = 0;
    if (p.dbg != nullptr && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    // ---- prologue: plan from cu_seqlens (warp 2), barriers (warp 0), TMEM (warp 1) ----
    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int s = 0; s < C::KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < C::NREG; ++s) { mbar_init(&t_full[s], 1); mbar_init(&t_empty[s], 4); }
        fence_barrier_init();
        prefetch_tensormap(&qmap);
        prefetch_tensormap(&kmap);
    }
    if (warp == 1) tmem_alloc(misc, 512);
    if (warp == 2) {
        // Warp-parallel inclusive scans of per-request unit and block counts; validation
        // of cu_seqlens (PackedBatch::validate, scheduler.cpp:33-48).
        bool ok = p.cu_seqlens[0] == 0;
        int carry_u = 0, carry_b = 0;
        for (int base = 0; base < R; base += 32) {
            const int r = base + lane;
            int units = 0, blocks = 0;
            if (r < R) {
                const int n = p.cu_seqlens[r + 1] - p.cu_seqlens[r];
                if (n <= 0) ok = false;
                blocks = n > 0 ? (n + G - 1) / G : 0;
                const bool en = p.drop_enabled == nullptr || p.drop_enabled[r] != 0;
                units = en && n > 0 ? (n + unit_keys - 1) / unit_keys : 0;
            }
            int x = units, y = blocks;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int a = __shfl_up_sync(0xffffffffu, x, o);
                const int b = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) { x += a; y += b; }
            }
            if (r < R) {
                s_cu_units[r + 1] = carry_u + x;
                s_cu_blocks[r + 1] = carry_b + y;
            }
            carry_u += __shfl_sync(0xffffffffu, x, 31);
            carry_b += __shfl_sync(0xffffffffu, y, 31);
        }
        ok = __all_sync(0xffffffffu, ok);
        if (lane == 0) {
            s_cu_units[0] = 0;
            s_cu_blocks[0] = 0;
            if (ok && p.cu_seqlens[R] > p.max_tokens) ok = false;
            misc[1] = ok ? 1u : 0u;
            if (!ok && blockIdx.x == 0) raise_error(p.err, kErrBadSeqlens);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = misc[0];
    if (blockIdx.x == 0) {
        // Publish the segment block offsets for the combine / select / compact kernels.
        for (int r = threadIdx.x; r <= R; r += blockDim.x) {
            p.cu_blocks[r] = misc[1] ? s_cu_blocks[r] : 0;
            p.cu_units_out[r] = misc[1] ? s_cu_units[r] : 0;
        }
    }

    Part P;
    P.cu_units = s_cu_units;
    P.R = R;
    P.nhg = p.num_hgroups;
    P.U = misc[1] ? static_cast<int64_t>(s_cu_units[R]) * p.num_hgroups : 0;
    P.grid = gridDim.x;
    const int64_t my_begin = P.U > 0 ? range_begin(P, blockIdx.x) : 0;
    const int64_t my_end = P.U > 0 ? range_begin(P, blockIdx.x + 1) : 0;

    if (warp == 0) {
        // ===== TMA producer =====
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t qiter = 0;
            for (int64_t pos = my_begin; pos < my_end;) {
                const Item it = make_item(P, pos, my_end);
                pos += it.u1 - it.u0;
                const int seg0 = p.cu_seqlens[it.r];
                const int N = p.cu_seqlens[it.r + 1] - seg0;
                const int neff = min(p.query_window_n, N);
                const int key0 = it.u0 * unit_keys;
                const int key1 = min(it.u1 * unit_keys, N);
                const int ntiles = (key1 - key0 + kTileKeys - 1) / kTileKeys;
                const int kv_local = (p.q_head_offset + it.hg * HPC) / p.gqa_group - p.kv_head_offset;
                mbar_wait(q_empty, (qiter & 1) ^ 1);
                ++qiter;
                mbar_arrive_expect_tx(q_full, C::Q_BYTES);
                const int qrow = seg0 + N - neff;
#pragma unroll
                for (int hh = 0; hh < HPC; ++hh) {
#pragma unroll
                    for (int kc = 0; kc < C::KC; ++kc)
                        tma_load_2d(sq + (hh * C::KC + kc) * C::SUB, &qmap, q_full,
                                    (it.hg * HPC + hh) * D + kc * 64, qrow);
                }
                for (int t = 0; t < ntiles; ++t) {
                    mbar_wait(&k_empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&k_full[stage], C::K_STAGE);
                    const int krow = seg0 + key0 + t * kTileKeys;
#pragma unroll
                    for (int kc = 0; kc < C::KC; ++kc)
                        tma_load_2d(sk + stage * C::K_STAGE + kc * C::SUB, &kmap, &k_full[stage],
                                    kv_local * D + kc * 64, krow);
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
            for (int64_t pos = my_begin; pos < my_end;) {
                const Item it = make_item(P, pos, my_end);
                pos += it.u1 - it.u0;
                const int N = p.cu_seqlens[it.r + 1] - p.cu_seqlens[it.r];
                const int key0 = it.u0 * unit_keys;
                const int key1 = min(it.u1 * unit_keys, N);
                const int ntiles = (key1 - key0 + kTileKeys - 1) / kTileKeys;
                mbar_wait(q_full, qiter & 1);
                ++qiter;
                tc_fence_after();
                for (int t = 0; t < ntiles; ++t) {
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
        const int etid = threadIdx.x - 64;   // 0..255
        const int wg = (warp - 2) >> 2;
        const int quarter = warp & 3;        // TMEM lane quarter this warp may access
        const int j = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const float sc = p.scale_log2;
        const int gpb = G / 32;              // 32-column groups per block
        // Per-(head slot, thread) running state lives in shared memory so that one copy of
        // the region body serves every head (keeps the hot loop small for the I-cache).
        float* st_m = s_state;
        float* st_l = st_m + C::NSLOT * 256;
        float* st_b = st_l + C::NSLOT * 256;
        int* st_gib = reinterpret_cast<int*>(st_b + C::NSLOT * 256);
        int* st_blk = st_gib + C::NSLOT * 256;
        const int hh_first = HPC >= 2 ? wg : 0;
        const int hh_step = HPC >= 2 ? 2 : 1;
        const bool active = HPC >= 2 || wg == 0;
        uint32_t seq_base = 0;
        for (int64_t pos = my_begin; pos < my_end;) {
            const Item it = make_item(P, pos, my_end);
            pos += it.u1 - it.u0;
            const int seg0 = p.cu_seqlens[it.r];
            const int N = p.cu_seqlens[it.r + 1] - seg0;
            const int neff = min(p.query_window_n, N);
            const int key0 = it.u0 * unit_keys;
            const int key1 = min(it.u1 * unit_keys, N);
            const int ntiles = (key1 - key0 + kTileKeys - 1) / kTileKeys;
            const bool row_valid = j < neff;
            const int qpos = N - neff + j;   // last key this row may see (segment-relative)
            const int64_t gb_seg = s_cu_blocks[it.r];  // global block index of block 0
            const int blk0 = key0 / G;
            for (int s = 0; s < C::NSLOT; ++s) {
                st_m[s * 256 + etid] = -INFINITY;
                st_l[s * 256 + etid] = 0.f;
                st_b[s * 256 + etid] = 0.f;
                st_gib[s * 256 + etid] = 0;
                st_blk[s * 256 + etid] = blk0;
            }

            for (int t = 0; t < ntiles && active; ++t) {
                const int colbase = key0 + t * kTileKeys;
                const bool tail = colbase + kTileKeys - 1 > N - neff;  // warp-uniform
#pragma unroll 1
                for (int hh = hh_first; hh < HPC; hh += hh_step) {
                    const int si = (HPC >= 2 ? hh >> 1 : 0) * 256 + etid;
                    const uint32_t sq_ = seq_base + t * HPC + hh;
                    const uint32_t reg = sq_ % C::NREG;
                    float* Prow = p.P + (static_cast<int64_t>(it.hg * HPC + hh) * p.max_blocks + gb_seg) * kRows + j;
                    float m = st_m[si], l = st_l[si], bsum = st_b[si];
                    int gib = st_gib[si], blk = st_blk[si];
                    mbar_wait(&t_full[reg], (sq_ / C::NREG) & 1);
                    tc_fence_after();
                    const uint32_t taddr = tmem_base + lane_base + reg * kTileKeys;
#pragma unroll 1
                    for (int q4 = 0; q4 < kTileKeys / 32; ++q4) {
                        const int c0 = colbase + q4 * 32;
                        uint32_t v[32];
                        tmem_ld32(taddr + q4 * 32, v);
                        tmem_ld_wait();
                        if (q4 == kTileKeys / 32 - 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[reg]);
                        }
                        if (c0 >= N) continue;  // warp-uniform
                        float gs;
                        if (!tail) {
                            gs = group_sum_pk(v, pk(sc, sc), pk(-m, -m));
                        } else {
                            const int lim = qpos - c0;  // column k valid iff k <= lim
                            float a0 = 0.f, a1 = 0.f;
#pragma unroll
                            for (int k = 0; k < 32; k += 2) {
                                const float e0 = ex2_approx(fmaf(__uint_as_float(v[k + 0]), sc, -m));
                                const float e1 = ex2_approx(fmaf(__uint_as_float(v[k + 1]), sc, -m));
                                a0 += (k + 0 <= lim) ? e0 : 0.f;
                                a1 += (k + 1 <= lim) ? e1 : 0.f;
                            }
                            gs = a0 + a1;
                        }
                        // Rebase only when a value exceeds the reference by ~2^40: partial sums
                        // stay < 2^53 (l over <= 2^13 keys) and values down to 2^-166 of the
                        // row max stay representable, so this fires essentially only on the
                        // item's first group (m = -inf).
                        if (!(gs <= 0x1p40f)) {
                            const int lim = tail ? qpos - c0 : 31;
                            float gmax = -INFINITY;
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (k <= lim) gmax = fmaxf(gmax, __uint_as_float(v[k]));
                            const float mnew = fmaxf(m, gmax * sc);
                            if (m != -INFINITY) {
                                const float f = ex2_approx(m - mnew);
                                l *= f;
                                bsum *= f;
                                rescale_rows(Prow, blk0, blk, f);
                            }
                            m = mnew;
                            gs = 0.f;
#pragma unroll
                            for (int k = 0; k < 32; ++k) {
                                const float e = ex2_approx(fmaf(__uint_as_float(v[k]), sc, -mnew));
                                gs += (k <= lim) ? e : 0.f;
                            }
                        }
                        bsum += gs;
                        if (++gib == gpb || c0 + 32 >= N) {
                            Prow[static_cast<int64_t>(blk) * kRows] = row_valid ? bsum : 0.f;
                            l += bsum;
                            bsum = 0.f;
                            gib = 0;
                            ++blk;
                        }
                    }
                    st_m[si] = m; st_l[si] = l; st_b[si] = bsum; st_gib[si] = gib; st_blk[si] = blk;
                }
            }
            seq_base += ntiles * HPC;
            // Item statistics for the owned heads: stats[sid][hh][row].
            if (active) {
                for (int hh = hh_first; hh < HPC; hh += hh_step) {
                    const int si = (HPC >= 2 ? hh >> 1 : 0) * 256 + etid;
                    const int64_t x = (it.sid * HPC + hh) * kRows + j;
                    p.stat_m[x] = row_valid ? st_m[si] : -INFINITY;
                    p.stat_l[x] = row_valid ? st_l[si] : 0.f;
                }
            }
            for (int u = it.u0 + etid; u < it.u1; u += 256) p.unit_sid[it.seg_start + u] = static_cast<int32_t>(it.sid);

        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
    if (p.dbg != nullptr && threadIdx.x == 0) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        p.dbg[blockIdx.x * 4 + 0] = t_start;
        p.dbg[blockIdx.x * 4 + 1] = t_end;
        p.dbg[blockIdx.x * 4 + 2] = static_cast<unsigned long long>(my_end - my_begin);
        unsigned nsm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(nsm));
        p.dbg[blockIdx.x * 4 + 3] = nsm;
    }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32)
pair_weights_kernel(const PairWeightsParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    // dynamic shared memory: rb[score_grid + 1], then sM / sL [warps][32]
    extern __shared__ __align__(16) unsigned char pw_smem[];
    int64_t* rb = reinterpret_cast<int64_t*>(pw_smem);
    float* sM = reinterpret_cast<float*>(rb + p.score_grid + 1);
    pair_weights_run(p, blockIdx.x, gridDim.x, NW, sM, sM + NW * 32, rb);
}

// items_per_pair: the launcher's estimate of the CTAs one pair spans (sizes the CTA: 4
// items per warp step, up to 32 warps -- the register budget follows the CTA size, so the
// small-CTA variants keep the warp path spill-free).
cudaError_t launch_pair_weights(const PairWeightsParams& p, int grid, int items_per_pair, cudaStream_t stream) {
    int warps = 2;
    while (warps < kPwWarps && 4 * warps < items_per_pair) warps *= 2;
    static const int force = [] {  // dev A/B: UP_PW_WARPS = 2 / 4 / 8 / 16 / 32
        const char* e = std::getenv("UP_PW_WARPS");
        return e == nullptr ? 0 : std::atoi(e);
    }();
    if (force == 2 || force == 4 || force == 8 || force == 16 || force == 32) warps = force;
    const size_t smem = sizeof(int64_t) * (p.score_grid + 1) + sizeof(float) * 2 * warps * 32;
    switch (warps) {
        case 2: return launch_k(kPdlScore, pair_weights_kernel<2>, grid, 64, smem, stream, p);
        case 4: return launch_k(kPdlScore, pair_weights_kernel<4>, grid, 128, smem, stream, p);
        case 8: return launch_k(kPdlScore, pair_weights_kernel<8>, grid, 256, smem, stream, p);
        case 16: return launch_k(kPdlScore, pair_weights_kernel<16>, grid, 512, smem, stream, p);
        default: return launch_k(kPdlScore, pair_weights_kernel<32>, grid, 1024, smem, stream, p);
    }
}

__global__ void __launch_bounds__(256)
block_combine_kernel(const BlockCombineParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    const int nw = blockDim.x >> 5;
    block_combine_run(p, static_cast<int64_t>(blockIdx.x) * nw + (threadIdx.x >> 5), static_cast<int64_t>(gridDim.x) * nw);
}

__global__ void __launch_bounds__(256)
block_combine_chunked_kernel(const BlockCombineParams p) {
    pdl_wait();
    pdl_trigger();
    __shared__ float s_part[8];
    block_combine_chunked(p, s_part);
}

// Fused combine + TP all-reduce over peer memory (Eq. 15): CTA c forms
// the scores of a contiguous chunk of blocks from this rank's heads and stores them straight
// into row `rank` of every peer's exchange buffer (no local partial vector), then runs the
// rendezvous of peer.cuh and writes the ascending-rank fp32 sum (allreduce_scores,
// tp_sim.cpp:43-47) to block_scores.  Fixed grid peer_grid() on every rank.
struct StorePeers {
    const PeerReduceParams* pr;
    int64_t row;  // peer_row_offset(epoch, rank): this launch's bank
    __device__ __forceinline__ void operator()(int gb, float v) const {
        for (int t = 0; t < pr->tp; ++t) pr->peer_slots[t][row + gb] = v;
    }
};

__global__ void __launch_bounds__(1024)
block_combine_peer_kernel(const __grid_constant__ BlockCombineParams p, const __grid_constant__ PeerReduceParams pr) {
    pdl_wait();
    __shared__ uint32_t s_epoch;
    if (threadIdx.x == 0) s_epoch = peer_epoch(pr);
    __syncthreads();
    int64_t total = p.cu_blocks[p.num_requests];
    if (total > pr.capacity) {  // more blocks than the exchange buffers hold
        if (threadIdx.x == 0) raise_error(pr.err, kErrTooManyBlocks);
        total = pr.capacity;
    }
    const int64_t chunk = (total + gridDim.x - 1) / gridDim.x;
    const int64_t c0 = min(static_cast<int64_t>(blockIdx.x) * chunk, total), c1 = min(c0 + chunk, total);
    block_combine_run(p, c0 + (threadIdx.x >> 5), blockDim.x >> 5, c1,
                      StorePeers{&pr, peer_row_offset(pr, s_epoch, pr.rank)});
    peer_publish_and_wait(pr, blockIdx.x, s_epoch);
    peer_sum_chunk(pr, c0, c1, s_epoch);
    pdl_trigger();
    peer_epoch_advance(pr);
}

// SIMT-path plan: validates cu_seqlens and writes cu_blocks (one warp).
__global__ void blocks_plan_kernel(const int32_t* __restrict__ cu, int R, int64_t max_tokens, int G,
                                   int32_t* __restrict__ cu_blocks, uint32_t* __restrict__ err) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    const int lane = threadIdx.x;
    bool ok = cu[0] == 0;
    int carry = 0;
    for (int base = 0; base < R; base += 32) {
        const int r = base + lane;
        int blocks = 0;
        if (r < R) {
            const int n = cu[r + 1] - cu[r];
            if (n <= 0) ok = false;
            blocks = (n + G - 1) / G;
        }
        int y = blocks;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int b = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += b;
        }
        if (r < R) cu_blocks[r + 1] = carry + y;
        carry += __shfl_sync(0xffffffffu, y, 31);
    }
    ok = __all_sync(0xffffffffu, ok) && cu[R] <= max_tokens;
    if (lane == 0) {
        cu_blocks[0] = 0;
        if (!ok) raise_error(err, kErrBadSeqlens);
    }
    if (!ok)  // malformed batch: no blocks, so nothing downstream indexes past its buffers
        for (int r = lane; r <= R; r += 32) cu_blocks[r] = 0;
}

// ---------------------------------------------------------------- host launchers
template <int D, int HPC>
static cudaError_t launch_tc(const CUtensorMap& qm, const CUtensorMap& km, const ScoreTcParams& p,
                             int grid, cudaStream_t stream) {
    using C = TcCfg<D, HPC>;
    const int smem = C::smem(p.num_requests);
    if (smem > 232448) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(score_tc_kernel<D, HPC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_k(kPdlScore, score_tc_kernel<D, HPC>, grid, C::THREADS, smem, stream, qm, km, p);
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

cudaError_t launch_blocks_plan(const int32_t* cu, int R, int64_t max_tokens, int G, int32_t* cu_blocks,
                               uint32_t* err, cudaStream_t stream) {
    return launch_k(kPdlScore, blocks_plan_kernel, 1, 32, 0, stream, cu, R, max_tokens, G, cu_blocks, err);
}

// Small unsharded combines (capacity blocks x head chunks within ~2 waves of 8 warps per
// SM, <= 64 heads, no per-shard outputs) split each block's heads over warps
// (block_combine_chunked): LLaMA 1x4K scorer stage 31.1 -> 29.6 us.  Large ones keep one
// warp per block (LLaMA 4x32K: 160.2 vs 164.7 us chunked).  UP_COMBINE_CHUNKED=0/1 forces.
cudaError_t launch_block_combine(const BlockCombineParams& p, int grid, int sms, cudaStream_t stream) {
    static const int force = [] {
        const char* s = std::getenv("UP_COMBINE_CHUNKED");
        return s == nullptr ? -1 : (s[0] == '0' ? 0 : 1);
    }();
    const int nch = (p.num_heads + 7) / 8;
    const bool small = p.max_blocks * nch <= 16LL * sms;
    if ((force == 1 || (force < 0 && small)) && p.num_shards == 1 && p.shard_scores == nullptr && p.num_heads <= 64) {
        const int64_t steps = (p.max_blocks + (8 / nch) - 1) / (8 / nch);  // CTA steps over the capacity
        const int64_t g = steps < static_cast<int64_t>(grid) * 4 ? steps : static_cast<int64_t>(grid) * 4;
        return launch_k(kPdlScore, block_combine_chunked_kernel, static_cast<int>(g < 1 ? 1 : g), 256, 0, stream, p);
    }
    return launch_k(kPdlScore, block_combine_kernel, grid, 256, 0, stream, p);
}

cudaError_t launch_block_combine_peer(const BlockCombineParams& p, const PeerReduceParams& pr, int grid,
                                      cudaStream_t stream) {
    // 32 warps per CTA: the grid is one CTA per SM (peer_grid, co-resident for the flag
    // waits), so more warps put every block of a chunk in flight at once -- c3-rank score
    // stage 56 -> 51 us against 256 threads (512: 54 us).  UP_PEER_COMBINE_THREADS: A/B.
    static const int threads = [] {
        const char* e = std::getenv("UP_PEER_COMBINE_THREADS");
        const int t = e == nullptr ? 1024 : std::atoi(e);
        return t == 256 || t == 512 ? t : 1024;
    }();
    return launch_k(kPdlScore, block_combine_peer_kernel, grid, threads, 0, stream, p, pr);
}

}  // namespace up
