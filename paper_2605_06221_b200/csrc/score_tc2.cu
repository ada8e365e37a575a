// score_tc2.cu -- the block scorer on CTA pairs: tcgen05.mma.cta_group::2, M = 256.
//
// Same math, work partition, per-item statistics and tail (pair_weights_kernel,
// block_combine_kernel) as score_tcw.cu, whose header restates importance.cpp:17-132 as a
// single pass over K.  What changes is the MMA shape, for the four q-heads of one kv-head
// (LLaMA-3.1-8B: GQA 4, D = 128):
//  * a cluster of two CTAs (one TPC) owns a range of (request, head-group, 128-key unit)
//    work; CTA rank c holds the Q tiles of heads 2c and 2c+1 of the group (64 KB) and HALF
//    of every 128-key K subtile (keys 64c .. 64c+63, 16 KB per stage), both loaded by TMA
//    into its own shared memory and signalling the leader's mbarriers;
//  * the leader's MMA thread issues, per subtile and head slot s, ONE M = 256 MMA: rows
//    0..127 are CTA 0's head s, rows 128..255 CTA 1's head 2+s, N = 128 keys (64 from each
//    CTA), so each SM's shared memory supplies 4 KB of A and 2 KB of B per 64-cycle MMA
//    step (96 B/clk instead of the 128 B/clk the single-CTA N = 128 MMA needs);
//  * the MMA works in chunks of four 128-key subtiles: head slot 0 over the chunk, then
//    slot 1 over the same K stages; job (slot, subtile a) goes to TMEM region a % 4 of four
//    128-column regions, so every region has three others' worth of work between its
//    drain and its refill (commits multicast to both CTAs' barriers);
//  * epilogue: four warpgroups per CTA, warpgroup w drains region w (both heads of the
//    CTA, subtiles a = w mod 4) and keeps running statistics per (head, w) -- "virtual
//    heads" hh * 4 + w, read by pair_weights / block_combine with npar = 4 and the parity
//    taken at 128-key granularity -- so a block must lie inside one subtile: G in
//    {32, 64, 128}.
#include "score_common.cuh"

namespace up {

#ifndef UP_TC2_POLY_PAIRS
#define UP_TC2_POLY_PAIRS 4
#endif
#ifndef UP_TC2_DIAG
#define UP_TC2_DIAG 0  // dev timing only: 1 = epilogue skips the math, 3 = one K-step MMA per subtile
#endif

// ---- cluster / cta_group::2 PTX helpers ----------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

// Arrive on a (possibly remote) mbarrier of the cluster.  Default semantics (release at CTA
// scope), as CUTLASS's ClusterBarrier::arrive: the ordering that matters -- this warp's
// tcgen05.ld before the leader's next MMA into the region -- comes from
// tcgen05.wait::ld + tcgen05.fence::before_thread_sync; a cluster-scope release would also
// wait for the warp's outstanding global stores (measured: 2.4x slower scorer).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// TMA tile load into this CTA's shared memory, completing on the LEADER's mbarrier
// (cluster address).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t smem_dst, const CUtensorMap* map, uint32_t bar_cluster,
                                                 int32_t x, int32_t y, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

__device__ __forceinline__ void mma_bf16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Arrive on the mbarrier at this shared offset in BOTH CTAs of the pair once every
// previously issued tcgen05 op of this thread completes.
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

template <int D>
struct Tc2Cfg {
    static constexpr int HPC = 4;                 // q-heads of one kv-head per CTA pair
    static constexpr int SLOTS = 2;               // heads per CTA
    static constexpr int KC = D / 64;             // 128-byte K-chunks per row
    static constexpr int QSUB = 128 * 128;        // [128 rows x 64 bf16] Q tile
    static constexpr int HK = 64;                 // keys per CTA per 128-key subtile
    static constexpr int KSUB = HK * 128;         // [64 keys x 64 bf16] K tile
    static constexpr int Q_BYTES = SLOTS * KC * QSUB;
    static constexpr int K_STAGE = KC * KSUB;
    static constexpr int R_RESERVE = 2 * (kTc2MaxRequests + 1) * 4;
    static constexpr int BUDGET = 232448 - 1024 - 512 - R_RESERVE;
    static constexpr int KST = (BUDGET - Q_BYTES) / K_STAGE > 8 ? 8 : (BUDGET - Q_BYTES) / K_STAGE;
    static constexpr int NREG = 4;                // TMEM regions of 128 columns (jobs round-robin)
    static constexpr int CH = 4;                  // subtiles per chunk (slot 0 then slot 1 over it)
    static constexpr int NBAR = 2 + 2 * KST + 2 * NREG;
    static constexpr int THREADS = 64 + 512;
    static constexpr int NP = UP_TC2_POLY_PAIRS;
    static int smem(int R) { return Q_BYTES + KST * K_STAGE + NBAR * 8 + 64 + 1024 + 2 * (R + 1) * 4; }
    static_assert(KST >= 2 * CH, "K ring: a chunk in use while the next one loads");
};

template <int D>
__global__ void __launch_bounds__(576, 1)
score_tc2_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                 const ScoreTcParams p) {
    pdl_wait();
    pdl_trigger();
    using C = Tc2Cfg<D>;
    constexpr int HPC = C::HPC, NPAR = 4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sq = smem;
    uint8_t* sk = smem + C::Q_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sk + C::KST * C::K_STAGE);
    uint64_t* q_full = bars + 0;                      // leader: Q of both CTAs landed
    uint64_t* q_empty = bars + 1;                     // both: the item's MMAs are done with Q
    uint64_t* k_full = bars + 2;                      // leader: both halves of stage s landed
    uint64_t* k_empty = bars + 2 + C::KST;            // both: stage s consumed
    uint64_t* t_full = bars + 2 + 2 * C::KST;         // both: region r holds a finished S tile
    uint64_t* t_empty = bars + 2 + 2 * C::KST + C::NREG;  // leader: both CTAs drained region r
    uint32_t* misc = reinterpret_cast<uint32_t*>(bars + C::NBAR);  // [0] tmem base, [1] plan ok
    int32_t* s_cu_units = reinterpret_cast<int32_t*>(misc + 16);
    int32_t* s_cu_blocks = s_cu_units + (p.num_requests + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int R = p.num_requests;
    const int G = p.block_size_g;
    const int unit_keys = p.unit_keys;

    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int s = 0; s < C::KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < C::NREG; ++s) { mbar_init(&t_full[s], 1); mbar_init(&t_empty[s], 8); }  // 4 warps x 2 CTAs
        fence_barrier_init();
        prefetch_tensormap(&qmap);
        prefetch_tensormap(&kmap);
    }
    if (warp == 1) tmem_alloc_pair(misc, 512);
    if (warp == 2) {
        // Plan from cu_seqlens (PackedBatch::validate, scheduler.cpp:33-48); both CTAs of
        // the pair compute the same plan.
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
    cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
    tc_fence_after();
    const uint32_t tmem_base = misc[0];
    if (blockIdx.x == 0) {
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
    P.grid = gridDim.x >> 1;  // one range per CTA pair
    const int pair = blockIdx.x >> 1;
    const int64_t my_begin = P.U > 0 ? range_begin(P, pair) : 0;
    const int64_t my_end = P.U > 0 ? range_begin(P, pair + 1) : 0;

    // leader-side barrier addresses as seen from either CTA of the pair
    const uint32_t q_full_l = mapa_shared(smem_u32(q_full), 0);
    const uint32_t k_full_l = mapa_shared(smem_u32(k_full), 0);
    const uint32_t t_empty_l = mapa_shared(smem_u32(t_empty), 0);

    if (warp == 0) {
        // ===== TMA producer (both CTAs): own Q heads per item, own half of each K subtile =====
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t qiter = 0;
            const uint64_t k_policy = l2_policy_evict_first();
            const uint64_t q_policy = l2_policy_evict_first();
            for (int64_t pos = my_begin; pos < my_end;) {
                const Item it = make_item(P, pos, my_end);
                pos += it.u1 - it.u0;
                const int seg0 = p.cu_seqlens[it.r];
                const int N = p.cu_seqlens[it.r + 1] - seg0;
                const int neff = min(p.query_window_n, N);
                const int key0 = it.u0 * unit_keys;
                const int key1 = min(it.u1 * unit_keys, N);
                const int nst = (key1 - key0 + 127) / 128;
                const int kv_local = (p.q_head_offset + it.hg * HPC) / p.gqa_group - p.kv_head_offset;
                mbar_wait(q_empty, (qiter & 1) ^ 1);
                ++qiter;
                if (rank == 0) mbar_arrive_expect_tx(q_full, 2 * C::Q_BYTES);
                const int qrow = seg0 + N - neff;
#pragma unroll
                for (int s = 0; s < C::SLOTS; ++s) {
#pragma unroll
                    for (int kc = 0; kc < C::KC; ++kc)
                        tma_load_2d_pair(smem_u32(sq + (s * C::KC + kc) * C::QSUB), &qmap, q_full_l,
                                         (it.hg * HPC + 2 * static_cast<int>(rank) + s) * D + kc * 64, qrow, q_policy);
                }
                for (int t = 0; t < nst; ++t) {
                    mbar_wait(&k_empty[stage], phase ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx(&k_full[stage], 2 * C::K_STAGE);
                    const int krow = seg0 + key0 + t * 128 + static_cast<int>(rank) * C::HK;
#pragma unroll
                    for (int kc = 0; kc < C::KC; ++kc)
                        tma_load_2d_pair(smem_u32(sk + stage * C::K_STAGE + kc * C::KSUB), &kmap, k_full_l + stage * 8,
                                         kv_local * D + kc * 64, krow, k_policy);
                    if (++stage == C::KST) { stage = 0; phase ^= 1; }
                }
            }
            // the leader's last multicast commits have landed here before this CTA exits
            if (qiter > 0) mbar_wait(q_empty, (qiter - 1) & 1);
        }
    } else if (warp == 1) {
        // ===== MMA issuer: the leader's single thread drives both SMs' tensor cores =====
        if (rank == 0 && elect_one()) {
            constexpr uint32_t kIdesc = idesc_bf16_f32(256, 128);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t qiter = 0;
            uint32_t uses[C::NREG] = {0u, 0u, 0u, 0u};  // jobs issued into TMEM region r
            const uint64_t a_base = smem_desc_sw128(smem_u32(sq));
            const uint64_t b_base = smem_desc_sw128(smem_u32(sk));
            const uint32_t t_full0 = smem_u32(t_full), t_empty0 = smem_u32(t_empty);
            const uint32_t k_full0 = smem_u32(k_full), k_empty0 = smem_u32(k_empty);
            for (int64_t pos = my_begin; pos < my_end;) {
                const Item it = make_item(P, pos, my_end);
                pos += it.u1 - it.u0;
                const int N = p.cu_seqlens[it.r + 1] - p.cu_seqlens[it.r];
                const int key1 = min(it.u1 * unit_keys, N);
                const int a_end = it.u0 + (key1 - it.u0 * unit_keys + 127) / 128;  // one past the last subtile
                mbar_wait(q_full, qiter & 1);
                ++qiter;
                tc_fence_after();
                // chunks of the absolute subtile index [4k, 4k+4): head slot 0 over the chunk,
                // then slot 1 over the same K stages (job (s, a) -> TMEM region a % 4)
                for (int a0 = it.u0; a0 < a_end;) {
                    const int a1 = min((a0 & ~(C::CH - 1)) + C::CH, a_end);
#pragma unroll 1
                    for (int s = 0; s < C::SLOTS; ++s) {
                        int st = stage;
                        uint32_t ph = phase;
#pragma unroll 1
                        for (int a = a0; a < a1; ++a) {
                            const uint32_t reg = static_cast<uint32_t>(a) & (C::NREG - 1);
                            const uint32_t use = uses[reg]++;
                            if (s == 0) mbar_wait_u32(k_full0 + st * 8, ph);
                            mbar_wait_u32(t_empty0 + reg * 8, (use & 1) ^ 1);
                            tc_fence_after();
                            const uint64_t b_stage = b_base + static_cast<uint32_t>((st * C::K_STAGE) >> 4);
                            const uint32_t d_tmem = tmem_base + reg * 128;
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk) {
                                const uint32_t aoff = ((s * C::KC + (kk >> 2)) * C::QSUB + (kk & 3) * 32) >> 4;
                                const uint32_t boff = ((kk >> 2) * C::KSUB + (kk & 3) * 32) >> 4;
                                if (UP_TC2_DIAG < 3 || kk == 0)
                                    mma_bf16_ss_pair(d_tmem, a_base + aoff, b_stage + boff, kIdesc, kk > 0 ? 1u : 0u);
                            }
                            mma_commit_pair(t_full0 + reg * 8);
                            if (s == C::SLOTS - 1) mma_commit_pair(k_empty0 + st * 8);  // both heads done with it
                            if (++st == C::KST) { st = 0; ph ^= 1; }
                        }
                        if (s == C::SLOTS - 1) { stage = st; phase = ph; }
                    }
                    a0 = a1;
                }
                mma_commit_pair(smem_u32(q_empty));
            }
        }
    } else {
        // ===== epilogue: warpgroup w drains TMEM region w; thread = query row =====
        // Region w holds the jobs (slot s, subtile a) with a % 4 == w, in the MMA's order
        // (per chunk: slot 0, then slot 1), so between two uses of a region the MMA has three
        // other regions to fill: the refill latency hides behind the other warpgroups' work.
        // Warpgroup w keeps running statistics for both heads of this CTA ("virtual heads"
        // hh * 4 + w: the 128-key subtiles of one head are split over four statistics rows by
        // subtile index mod 4, the layout pair_weights / block_combine read with npar = 4).
        const int etid = threadIdx.x - 64;   // 0..511
        const int w = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int j = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const float sc = p.scale_log2;
        const uint32_t t_full_r = smem_u32(t_full) + w * 8;
        const uint32_t t_empty_r = t_empty_l + w * 8;
        const uint32_t taddr0 = tmem_base + lane_base + w * 128;
        const bool lean = G == 64;
        const int gpb = G >> 5;                             // 32-key groups per block
        const int gshift = G == 32 ? 0 : (G == 64 ? 1 : 2);
        uint32_t use = 0;
        for (int64_t pos = my_begin; pos < my_end;) {
            const Item it = make_item(P, pos, my_end);
            pos += it.u1 - it.u0;
            const int seg0 = p.cu_seqlens[it.r];
            const int N = p.cu_seqlens[it.r + 1] - seg0;
            const int neff = min(p.query_window_n, N);
            const int key0 = it.u0 * unit_keys;
            const int key1 = min(it.u1 * unit_keys, N);
            const int a_end = it.u0 + (key1 - key0 + 127) / 128;
            const bool row_valid = j < neff;
            const int qpos = N - neff + j;  // row j's causal limit (importance.cpp:27)
            const int64_t gb_seg = s_cu_blocks[it.r];
            const int blk0 = key0 / G;
            float* Prow[C::SLOTS];
            float mm[C::SLOTS], ll[C::SLOTS];
#pragma unroll
            for (int s = 0; s < C::SLOTS; ++s) {
                Prow[s] = p.P + (static_cast<int64_t>(it.hg * HPC + 2 * static_cast<int>(rank) + s) * p.max_blocks +
                                 gb_seg) * kRows + j;
                mm[s] = -INFINITY;
                ll[s] = 0.f;
            }
#pragma unroll 1
            for (int a = it.u0 + ((w - it.u0) & 3); a < a_end; a += 4) {
                const int cbase = a * 128;  // key offset of subtile a in the request
#pragma unroll
                for (int s = 0; s < C::SLOTS; ++s, ++use) {
                    float m = mm[s], l = ll[s];
                    float* const prow = Prow[s];
                    mbar_wait_u32(t_full_r, use & 1);
                    tc_fence_after();
                    float gs[4] = {0.f, 0.f, 0.f, 0.f};
                    const bool fast = cbase + 128 <= N - neff + 1 && UP_TC2_DIAG != 1;  // warp-uniform
                    bool redo = !fast && cbase < N && UP_TC2_DIAG != 1;
                    bool done = false;
                    if (fast) {
                        // eight 16-column chunks, the next chunk's TMEM load in flight while
                        // the current one is summed
                        const uint64_t sc2 = pk(sc, sc), m2 = pk(-m, -m);
                        uint32_t va[16], vb[16];
                        uint64_t q[4];
                        tmem_ld16(taddr0, va);
#pragma unroll
                        for (int c = 0; c < 8; c += 2) {
                            tmem_ld_wait();
                            tmem_ld16(taddr0 + c * 16 + 16, vb);
                            pin16(va);
                            const uint64_t s0 = chunk_sum_pk<8, C::NP / 2>(va, sc2, m2);
                            tmem_ld_wait();
                            if (c + 2 < 8) tmem_ld16(taddr0 + c * 16 + 32, va);
                            pin16(vb);
                            q[c >> 1] = add2(s0, chunk_sum_pk<8, C::NP / 2>(vb, sc2, m2));
                        }
#pragma unroll
                        for (int g = 0; g < 4; ++g) gs[g] = lo_f(q[g]) + hi_f(q[g]);
                        redo = !((gs[0] + gs[1]) + (gs[2] + gs[3]) <= 0x1p40f);
                        if (lean && __all_sync(0xffffffffu, !row_valid || !redo)) {
                            // lean path: the subtile is exactly blocks 2a, 2a+1 of the request
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cluster(t_empty_r);
                            const float b0 = gs[0] + gs[1], b1 = gs[2] + gs[3];
                            float* pr = prow + static_cast<int64_t>(2 * a) * kRows;
                            pr[0] = row_valid ? b0 : 0.f;
                            pr[kRows] = row_valid ? b1 : 0.f;
                            l += b0;
                            l += b1;
                            done = true;
                        }
                    }
                    if (!done) {
                        if (redo) {
                            // Generic path: causal tail, ragged segment end, or a rebase of m.
#pragma unroll 1
                            for (int q2 = 0; q2 < 4; ++q2) {
                                const int c0 = cbase + q2 * 32;
                                const int lim = min(qpos - c0, min(31, N - 1 - c0));  // last valid column
                                uint32_t v[32];
                                tmem_ld32(taddr0 + q2 * 32, v);
                                tmem_ld_wait();
                                float g = 0.f;
                                if (lim >= 0) {
                                    float a0 = 0.f, a1 = 0.f;
#pragma unroll
                                    for (int k = 0; k < 32; k += 2) {
                                        const float e0 = ex2_approx(fmaf(__uint_as_float(v[k + 0]), sc, -m));
                                        const float e1 = ex2_approx(fmaf(__uint_as_float(v[k + 1]), sc, -m));
                                        a0 += (k + 0 <= lim) ? e0 : 0.f;
                                        a1 += (k + 1 <= lim) ? e1 : 0.f;
                                    }
                                    g = a0 + a1;
                                }
                                if (!(g <= 0x1p40f)) {
                                    // Rebase: move m to this group's maximum (see score_tc.cu).
                                    float gmax = -INFINITY;
#pragma unroll
                                    for (int k = 0; k < 32; ++k)
                                        if (k <= lim) gmax = fmaxf(gmax, __uint_as_float(v[k]));
                                    const float mnew = fmaxf(m, gmax * sc);
                                    if (m != -INFINITY) {
                                        const float f = ex2_approx(m - mnew);
                                        l *= f;
                                        for (int x = 0; x < q2; ++x) gs[x] *= f;  // groups of this subtile so far
                                        // completed blocks of this virtual head before this subtile
                                        for (int b = blk0; b < (cbase >> (5 + gshift)); ++b)
                                            if ((((b * G) >> 7) & 3) == w) prow[static_cast<int64_t>(b) * kRows] *= f;
                                    }
                                    m = mnew;
                                    g = 0.f;
#pragma unroll
                                    for (int k = 0; k < 32; ++k) {
                                        const float e = ex2_approx(fmaf(__uint_as_float(v[k]), sc, -mnew));
                                        g += (k <= lim) ? e : 0.f;
                                    }
                                }
                                gs[q2] = g;
                            }
                        }
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(t_empty_r);
                        if (cbase < N) {  // warp-uniform: else padding past the segment end
                            float bsum = 0.f;
#pragma unroll
                            for (int q2 = 0; q2 < 4; ++q2) {
                                const int c0 = cbase + q2 * 32;
                                if (c0 >= N) break;  // warp-uniform
                                bsum += gs[q2];
                                const int gi = c0 >> 5;
                                if ((gi & (gpb - 1)) == gpb - 1 || c0 + 32 >= N) {  // block gi >> gshift complete
                                    prow[static_cast<int64_t>(gi >> gshift) * kRows] = row_valid ? bsum : 0.f;
                                    l += bsum;
                                    bsum = 0.f;
                                }
                            }
                        }
                    }
                    mm[s] = m;
                    ll[s] = l;
                }
            }
#pragma unroll
            for (int s = 0; s < C::SLOTS; ++s) {
                const int64_t x = (it.sid * (HPC * NPAR) + (2 * static_cast<int>(rank) + s) * NPAR + w) * kRows + j;
                p.stat_m[x] = row_valid ? mm[s] : -INFINITY;
                p.stat_l[x] = row_valid ? ll[s] : 0.f;
            }
            if (rank == 0)
                for (int uu = it.u0 + etid; uu < it.u1; uu += 512)  // unit = 128-key subtile uu, parity uu % 4
                    p.unit_sid[it.seg_start + uu] = tcw_usid(static_cast<int32_t>(it.sid), uu % 4);
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while its peer may still signal it
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, 512);
    }
}

// Opt-in (UP_TC2=1): measured on B200 at the LLaMA 4x32K layer, this kernel is not faster
// than score_tcw's single-CTA form: the scorer is bound by the
// exp2 epilogue (MUFU + FMA-pipe polynomial, and the board power cap under sustained
// load), not by the MMA's shared-memory reads the CTA pair halves.
bool tc2_enabled() {
    static const bool on = [] {
        const char* s = std::getenv("UP_TC2");
        return s != nullptr && s[0] == '1';
    }();
    return on;
}

bool tc2_supported(int D, int HPC, int G, int R) {
    return tc2_enabled() && D == 128 && HPC == 4 && (G == 32 || G == 64 || G == 128) && R <= kTc2MaxRequests;
}

int tc2_stage_keys() { return Tc2Cfg<128>::HK; }

// CTAs of the launch: an even count of co-resident CTAs (cluster pairs on TPCs).
int tc2_grid(int num_sms) {
    static int grid = 0;
    if (grid == 0) {
        using C = Tc2Cfg<128>;
        cudaFuncSetAttribute(score_tc2_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(num_sms & ~1);
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::smem(kTc2MaxRequests);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, score_tc2_kernel<128>, &cfg) != cudaSuccess || clusters < 1)
            clusters = num_sms / 2;
        grid = 2 * clusters;
    }
    return grid;
}

cudaError_t launch_score_tc2(const CUtensorMap& qm, const CUtensorMap& km, const ScoreTcParams& p, int grid,
                             cudaStream_t stream) {
    using C = Tc2Cfg<128>;
    const int smem = C::smem(p.num_requests);
    if (p.num_requests > kTc2MaxRequests || smem > 232448 || (grid & 1)) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(score_tc2_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_mask() & kPdlScore) ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, score_tc2_kernel<128>, qm, km, p);
}

}  // namespace up
