// score_tcw.cu -- tensor-core block scorer with four epilogue warpgroups for HPC = 4, 2 or
// 1 (virtual) q-heads per kv-head (LLaMA-3.1-8B: D = 128, HPC = 4; Gemma-3 / Qwen3-Next
// full-attention layers: D = 256, HPC = 2; MHA shapes: HPC = 1).  A "head" here is a
// virtual head of 128 query rows: a query tile of a longer window (n > 128, q_tiles) or
// several q-heads' short windows packed together (n <= 64, q_pack) -- see params.cuh.
//
// Same math, work partition and per-item statistics as score_tc.cu (its header restates
// importance.cpp:17-132 as a single pass over K); pair_weights_kernel and
// block_combine_kernel finish the job.  What this kernel changes is the pipeline shape,
// because the exp2 epilogue (MUFU, 16/clk/SM) -- not the tensor core -- bounds the scorer:
//  * 18 warps: warp 0 TMA, warp 1 MMA, warps 2..17 = four epilogue warpgroups, so every
//    SMSP runs four exp2 streams.  Warpgroup wg drains head hh = wg / NPAR and, with
//    HPC = 2 / 1 (NPAR = 2 / 4), only the 64-key subtiles whose parity (position in the
//    request mod NPAR) is wg % NPAR: the warpgroups of a head keep separate running
//    statistics, recorded as separate rows vh = hh * NPAR + par in the item statistics
//    (requires G in {32, 64} so that every block lies inside one subtile);
//  * K is streamed in stages of SK keys (128 x 2 stages at D <= 128, 64 x 3 at D = 256)
//    next to the resident Q of the HPC heads (128 KB), so the kv-head's K tile is read
//    from HBM once for all HPC heads;
//  * every 64-key subtile is one N = 64 MMA per head into a ring of NB = 8 / HPC TMEM
//    regions per head (512 columns in total).
#include "score_common.cuh"

namespace up {

#ifndef UP_TCW_POLY_PAIRS_D128
#define UP_TCW_POLY_PAIRS_D128 4
#endif
#ifndef UP_TCW_POLY_PAIRS_D256
#define UP_TCW_POLY_PAIRS_D256 0
#endif

#ifndef UP_TCW_DIAG
#define UP_TCW_DIAG 0  // dev timing only: 1 = skip the epilogue math, 3 = one K-step MMA per subtile
#endif
#ifndef UP_TCW_SUBN_HPC4
#define UP_TCW_SUBN_HPC4 128
#endif
#ifndef UP_TCW_STAGE_KEYS_D128
#define UP_TCW_STAGE_KEYS_D128 128
#endif

// HPC = 4 fast path: the next 32-column TMEM load is in flight while a group is summed
// (tools/ldpipe_sweep.sh: LLaMA 4x32K scorer 159.9 -> 158.5 us; D = 256 unchanged, so the
// two-group HPC = 2 path keeps the plain sequence).
#ifndef UP_TCW_LD_PIPE
#define UP_TCW_LD_PIPE 1
#endif
#ifndef UP_TCW_LEAN2  // lean path of the parity epilogues (NPAR > 1, 64-key subtiles, G = 64)
#define UP_TCW_LEAN2 1
#endif
#ifndef UP_TCW_LEAN
#define UP_TCW_LEAN 1
#endif

template <int D, int HPC, bool SPLIT = false>
struct TcwCfg {
    // TS: with two q-heads per CTA, Q lives in TMEM (tcgen05.mma A operand from tensor
    // memory): the MMA then reads only K from shared memory, which keeps the D = 256
    // MMA math-bound instead of shared-memory-bound, and frees the 128 KB Q tile.
    // (HPC = 1: one q-head per kv-head -- MHA shapes, or packed query rows -- is TS too: an
    // SS N = 64 MMA would read 6 KB of shared memory per 32 cycles)
    static constexpr bool TS = (HPC == 2 || HPC == 1) && D >= 128;
    static constexpr int SK = TS ? 128 : (D <= 128 ? UP_TCW_STAGE_KEYS_D128 : 64);  // keys per K stage
    // keys per MMA / TMEM region (UP_TCW_SUBN_HPC4 = 128: one N = 128 region per head)
    static constexpr int SUBN = HPC == 4 ? UP_TCW_SUBN_HPC4 : 64;
    static constexpr int NG = SUBN / 32;          // 32-column groups per subtile
    static constexpr int SPS = SK / SUBN;         // subtiles per K stage
    // epilogue warpgroups per head = statistics rows per head; SPLIT (HPC = 4): two, one per
    // 64-key half of every subtile
    static constexpr int NPAR = SPLIT ? 2 : 4 / HPC;
    static constexpr int NB = (512 - (TS ? HPC * D / 2 : 0)) / (HPC * SUBN);  // TMEM regions per head
    static constexpr int KC = D / 64;             // 128-byte K-chunks per row
    static constexpr int QSUB = 128 * 128;        // [128 rows x 64 bf16] Q tile
    static constexpr int KSUB = SK * 128;         // [SK keys x 64 bf16] K tile
    static constexpr int Q_BYTES = TS ? 0 : HPC * KC * QSUB;
    static constexpr int Q_COLS = TS ? HPC * D / 2 : 0;   // TMEM columns of the resident Q
    static constexpr int K_STAGE = KC * KSUB;
    static constexpr int R_RESERVE = 2 * (kTcwMaxRequests + 1) * 4;
    static constexpr int BUDGET = 232448 - 1024 - 512 - R_RESERVE;
    static constexpr int KST = (BUDGET - Q_BYTES) / K_STAGE > 8 ? 8 : (BUDGET - Q_BYTES) / K_STAGE;
    static constexpr int NREG = HPC * NB;
    static constexpr int NBAR = 2 + 2 * KST + 2 * NREG;
    static constexpr int THREADS = 64 + 512;
    static constexpr int NP = D <= 128 ? UP_TCW_POLY_PAIRS_D128 : UP_TCW_POLY_PAIRS_D256;
    static int smem(int R) { return Q_BYTES + KST * K_STAGE + NBAR * 8 + 64 + 1024 + 2 * (R + 1) * 4; }
    static_assert(KST >= 2, "K ring too small");
    static_assert(!SPLIT || (HPC == 4 && SUBN == 128 && NB == 1), "SPLIT drains one 128-column region per head");
};

// Parity of the NPAR > 1 epilogues.  Subtile u of the CTA (the counter the MMA warp's TMEM
// ring runs on) goes to warpgroup (u >> ushift) % NPAR: one 64-key subtile per parity unit,
// or pairs of them when a block spans two (G = 128, ushift = 1), so that every block belongs
// to one warpgroup.  Counting in the CTA's own sequence -- not by key position -- keeps a
// warpgroup's consecutive waits on the ring at most NPAR (pairs: 2 NPAR - 1) subtiles apart,
// within the NB regions one mbarrier parity can tell apart, whatever items the CTA walks
// (a key-position parity lets a warpgroup skip whole short items and then wait on a region
// two phases ahead).  The parity of each 128-key unit's first subtile travels to
// block_combine in the top bits of unit_sid (tcw_usid); block_combine adds the block's
// offset in the unit at par_shift granularity.
__host__ __device__ constexpr int tcw_par_shift(int G) { return G > 64 ? 7 : 6; }
__host__ __device__ constexpr int tcw_ushift(int G) { return G > 64 ? 1 : 0; }

// Rebase (cold): rescale the partials this thread already wrote for the item -- blocks
// [g0, g1) in parity units of this warpgroup (subtile index u0 + (g G - key0) / 64).
static __device__ __noinline__ void rescale_rows_par(float* prow, int g0, int g1, int G, int npar, int par,
                                                     float f, int key0, uint32_t u0) {
    const int us = tcw_ushift(G);
    for (int g = g0; g < g1; ++g)
        if (((u0 + static_cast<uint32_t>((g * G - key0) >> 6)) >> us) % npar == static_cast<uint32_t>(par))
            prow[static_cast<int64_t>(g) * kRows] *= f;
}

#ifndef UP_TCW_FIRST_REF  // dev A/B: 0 = an item's first subtile tries the fast path and rebases
#define UP_TCW_FIRST_REF 1
#endif
// First reference m of a row: the maximum of the group's valid columns (k <= lim), scaled
// -- what the overflow rebase from m = -inf produced, without the wasted first pass.
static __device__ __forceinline__ float first_ref(const uint32_t (&v)[32], int lim, float sc) {
    float gmax = -INFINITY;
#pragma unroll
    for (int k = 0; k < 32; ++k)
        if (k <= lim) gmax = fmaxf(gmax, __uint_as_float(v[k]));
    return fmaxf(-INFINITY, gmax * sc);
}

// UP_SCORE_DEBUG phase clocks (second region of the debug buffer): slot k of this CTA
#define TCW_PHASE(k)                                                                   \
    if (p.dbg != nullptr) {                                                            \
        unsigned long long t_;                                                         \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
        if (p.dbg[4 * 4096 + blockIdx.x * 4 + (k)] == 0ull) p.dbg[4 * 4096 + blockIdx.x * 4 + (k)] = t_; \
    }

template <int D, int HPC, bool SPLIT>
__global__ void __launch_bounds__(576, 1)
score_tcw_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                 const ScoreTcParams p) {
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    using C = TcwCfg<D, HPC, SPLIT>;
    constexpr int NPAR = C::NPAR, NB = C::NB;
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
    uint32_t* misc = reinterpret_cast<uint32_t*>(bars + C::NBAR);  // [0] tmem base, [1] plan ok
    int32_t* s_cu_units = reinterpret_cast<int32_t*>(misc + 16);
    int32_t* s_cu_blocks = s_cu_units + (p.num_requests + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int R = p.num_requests;
    const int G = p.block_size_g;
    const int unit_keys = p.unit_keys;
    unsigned long long t_start = 0;
    if (p.dbg != nullptr && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    if (warp == 0 && lane == 0) {
        mbar_init(q_full, C::TS ? 16 : 1);  // TS: every epilogue warp stores its Q slice
        mbar_init(q_empty, 1);
        for (int s = 0; s < C::KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        // a region is released by the warps that drain it: one warpgroup, or two with SPLIT
        for (int s = 0; s < C::NREG; ++s) { mbar_init(&t_full[s], 1); mbar_init(&t_empty[s], SPLIT ? 8 : 4); }
        fence_barrier_init();
        prefetch_tensormap(&qmap);
        prefetch_tensormap(&kmap);
    }
    if (warp == 1) tmem_alloc(misc, 512);
    // Barrier init, tensor-map prefetch and the TMEM allocation overlap the predecessor's
    // tail (PDL); everything from the plan on reads its outputs.
    pdl_wait();
    if (warp == 2) {
        // Plan from cu_seqlens (PackedBatch::validate, scheduler.cpp:33-48).
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
        // ===== TMA producer: Q of the HPC heads once per item, K in 64-key stages =====
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t qiter = 0;
            const uint64_t k_policy = l2_policy_evict_first();
            for (int64_t pos = my_begin; pos < my_end;) {
                const Item it = make_item(P, pos, my_end);
                pos += it.u1 - it.u0;
                const int seg0 = p.cu_seqlens[it.r];
                const int N = p.cu_seqlens[it.r + 1] - seg0;
                const int neff = min(p.query_window_n, N);
                const int key0 = it.u0 * unit_keys;
                const int key1 = min(it.u1 * unit_keys, N);
                const int nst = (key1 - key0 + C::SK - 1) / C::SK;
                const int Tt = p.q_tiles;
                const int kv_local = (p.q_head_offset + it.hg * HPC * p.q_pack / Tt) / p.gqa_group - p.kv_head_offset;
                if (!C::TS) {
                    mbar_wait(q_empty, (qiter & 1) ^ 1);
                    ++qiter;
                    mbar_arrive_expect_tx(q_full, C::Q_BYTES);
                    const int qrow = seg0 + N - neff;
#pragma unroll
                    for (int hh = 0; hh < HPC; ++hh) {
                        const int v = it.hg * HPC + hh;  // virtual head = q-head * Tt + query tile
                        const int h = v / Tt;
#pragma unroll
                        for (int kc = 0; kc < C::KC; ++kc)
                            tma_load_2d(sq + (hh * C::KC + kc) * C::QSUB, &qmap, q_full, h * D + kc * 64,
                                        qrow + (v - h * Tt) * kRows);
                    }
                }
                for (int t = 0; t < nst; ++t) {
                    mbar_wait(&k_empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&k_full[stage], C::K_STAGE);
                    const int krow = seg0 + key0 + t * C::SK;
#pragma unroll
                    for (int kc = 0; kc < C::KC; ++kc)
                        tma_load_2d_hint(sk + stage * C::K_STAGE + kc * C::KSUB, &kmap, &k_full[stage],
                                         kv_local * D + kc * 64, krow, k_policy);
                    if (++stage == C::KST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (one thread): per 64-key subtile, one N = 64 MMA per head =====
        // Descriptors = a per-CTA base plus compile-time offsets (the 14-bit address field
        // cannot carry into the other fields).
        if (elect_one()) {
            constexpr uint32_t kIdesc = idesc_bf16_f32(128, C::SUBN);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t qiter = 0;
            uint32_t u = 0;  // 64-key subtile counter (selects the TMEM region of every head)
            const uint64_t a_base = smem_desc_sw128(smem_u32(sq));
            const uint64_t b_base = smem_desc_sw128(smem_u32(sk));
            for (int64_t pos = my_begin; pos < my_end;) {
                const Item it = make_item(P, pos, my_end);
                pos += it.u1 - it.u0;
                const int N = p.cu_seqlens[it.r + 1] - p.cu_seqlens[it.r];
                const int key0 = it.u0 * unit_keys;
                const int key1 = min(it.u1 * unit_keys, N);
                const int nst = (key1 - key0 + C::SK - 1) / C::SK;
                mbar_wait(q_full, qiter & 1);
                ++qiter;
                tc_fence_after();
                TCW_PHASE(0)
                for (int t = 0; t < nst; ++t) {
                    mbar_wait(&k_full[stage], phase);
                    tc_fence_after();
                    const uint64_t b_stage = b_base + static_cast<uint32_t>((stage * C::K_STAGE) >> 4);
#pragma unroll
                    for (int s = 0; s < C::SPS; ++s, ++u) {
#pragma unroll
                        for (int hh = 0; hh < HPC; ++hh) {
                            const uint32_t reg = hh * NB + u % NB;
                            mbar_wait(&t_empty[reg], ((u / NB) & 1) ^ 1);
                            tc_fence_after();
                            const uint32_t d_tmem = tmem_base + C::Q_COLS + reg * C::SUBN;
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk) {
                                const uint32_t aoff = ((hh * C::KC + (kk >> 2)) * C::QSUB + (kk & 3) * 32) >> 4;
                                // subtile s = rows s*SUBN.. of the stage: SUBN/8 swizzle atoms further
                                const uint32_t boff = ((kk >> 2) * C::KSUB + (kk & 3) * 32 + s * C::SUBN * 128) >> 4;
                                if (UP_TCW_DIAG != 3 || kk == 0) {
                                    if (C::TS)  // A = head hh's Q columns [kk*8, kk*8+8) in TMEM
                                        mma_bf16_ts(d_tmem, tmem_base + hh * (D / 2) + kk * 8, b_stage + boff, kIdesc,
                                                    kk > 0 ? 1u : 0u);
                                    else
                                        mma_bf16_ss(d_tmem, a_base + aoff, b_stage + boff, kIdesc, kk > 0 ? 1u : 0u);
                                }
                            }
                            mma_commit(&t_full[reg]);
                        }
                    }
                    mma_commit(&k_empty[stage]);
                    if (++stage == C::KST) { stage = 0; phase ^= 1; }
                }
                mma_commit(q_empty);
            }
        }
    } else if constexpr (SPLIT) {
        // ===== SPLIT epilogue (HPC = 4, G in {32, 64}): warpgroup wg drains column half
        // c = wg & 1 of every 128-key subtile for the two heads hp = wg >> 1 and hp + 2, so
        // every region is drained by two warpgroups and every warpgroup alternates between two
        // regions: while it sums one head's half, the MMA warp refills the other head's
        // region, and a region is always full again before its drainers come back (with one
        // region per head and one warpgroup per region, each drain was followed by a wait on
        // the tensor pipe).  Statistics rows per (head, half): virtual head hh * 2 + c -- the
        // parity pair_weights / block_combine take at 64-key granularity (par_shift 6).
        const int etid = threadIdx.x - 64;   // 0..511
        const int wg = (warp - 2) >> 2;
        const int c = wg & 1;
        const int hp = wg >> 1;
        const int quarter = warp & 3;        // TMEM lane quarter this warp may access
        const int j = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const float sc = p.scale_log2;
        const uint32_t tfull_addr = smem_u32(t_full), tempty_addr = smem_u32(t_empty);
        const int gshift = G == 64 ? 6 : 5;  // log2 G
        uint32_t u = 0;
        for (int64_t pos = my_begin; pos < my_end;) {
            const Item it = make_item(P, pos, my_end);
            pos += it.u1 - it.u0;
            const int seg0 = p.cu_seqlens[it.r];
            const int N = p.cu_seqlens[it.r + 1] - seg0;
            const int neff = min(p.query_window_n, N);
            const int key0 = it.u0 * unit_keys;
            const int key1 = min(it.u1 * unit_keys, N);
            const int nsub = (key1 - key0 + C::SK - 1) / C::SK * C::SPS;  // as issued by the MMA warp
            const int64_t gb_seg = s_cu_blocks[it.r];
            const int blk0 = key0 >> gshift;
            float* Prow[2];
            float m[2], l[2];
            bool valid2[2];
            int qpos2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int v = it.hg * HPC + hp + 2 * e;
                const int jr = (v % p.q_tiles) * kRows + j;  // window row of this virtual head's row j
                valid2[e] = jr < neff;
                qpos2[e] = N - neff + jr;  // its causal limit (importance.cpp:27)
                Prow[e] = p.P + (static_cast<int64_t>(v) * p.max_blocks + gb_seg) * kRows + j;
                m[e] = -INFINITY;
                l[e] = 0.f;
            }
#pragma unroll 1
            for (int t = 0; t < nsub; ++t, ++u) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int reg = hp + 2 * e;  // NB = 1: region = head
                    const int cb = key0 + t * C::SUBN + 64 * c;  // this warpgroup's 64 keys
                    const bool row_valid = valid2[e];
                    const int qpos = qpos2[e];
                    mbar_wait_u32(tfull_addr + reg * 8, u & 1);
                    tc_fence_after();
                    if (warp == 2 && lane == 0) TCW_PHASE(1)
                    const uint32_t taddr = tmem_base + lane_base + reg * C::SUBN + 64 * c;
                    float gs0 = 0.f, gs1 = 0.f;
                    bool redo;
                    if (cb + 64 <= N - neff + 1 && !(UP_TCW_FIRST_REF && __any_sync(0xffffffffu, row_valid && m[e] == -INFINITY))) {
                        // whole half inside the segment and left of every row's causal limit
                        // (and a reference m set: the item's first half goes the generic way)
                        uint32_t va[32], vb[32];
                        tmem_ld32(taddr, va);
                        tmem_ld_wait();
                        tmem_ld32(taddr + 32, vb);
                        gs0 = group_sum_pk<C::NP>(va, pk(sc, sc), pk(-m[e], -m[e]));
                        tmem_ld_wait();
                        gs1 = group_sum_pk<C::NP>(vb, pk(sc, sc), pk(-m[e], -m[e]));
                        // rows past n_eff carry no statistics: never a reason to rebase
                        redo = !__all_sync(0xffffffffu, !row_valid || gs0 + gs1 <= 0x1p40f);
                    } else {
                        redo = cb < N;
                    }
                    if (redo) {
                        // Generic path: causal tail, ragged segment end, or a rebase of m.
#pragma unroll 1
                        for (int q2 = 0; q2 < 2; ++q2) {
                            const int c0 = cb + q2 * 32;
                            const int lim = min(qpos - c0, min(31, N - 1 - c0));  // last valid column
                            uint32_t v[32];
                            tmem_ld32(taddr + q2 * 32, v);
                            tmem_ld_wait();
                            float gs = 0.f;
                            if (UP_TCW_FIRST_REF && lim >= 0 && m[e] == -INFINITY) m[e] = first_ref(v, lim, sc);
                            if (lim >= 0) {
                                float a0 = 0.f, a1 = 0.f;
#pragma unroll
                                for (int k = 0; k < 32; k += 2) {
                                    const float e0 = ex2_approx(fmaf(__uint_as_float(v[k + 0]), sc, -m[e]));
                                    const float e1 = ex2_approx(fmaf(__uint_as_float(v[k + 1]), sc, -m[e]));
                                    a0 += (k + 0 <= lim) ? e0 : 0.f;
                                    a1 += (k + 1 <= lim) ? e1 : 0.f;
                                }
                                gs = a0 + a1;
                            }
                            if (!(gs <= 0x1p40f)) {
                                // Rebase: move m to this group's maximum (see score_tc.cu).
                                float gmax = -INFINITY;
#pragma unroll
                                for (int k = 0; k < 32; ++k)
                                    if (k <= lim) gmax = fmaxf(gmax, __uint_as_float(v[k]));
                                const float mnew = fmaxf(m[e], gmax * sc);
                                if (m[e] != -INFINITY) {
                                    const float f = ex2_approx(m[e] - mnew);
                                    l[e] *= f;
                                    gs0 *= f;  // the half's first group when q2 = 1
                                    // blocks of this half already written for the item
                                    rescale_rows_par(Prow[e], blk0, cb >> gshift, G, 2, c, f, key0, 0u);  // parity = key half
                                }
                                m[e] = mnew;
                                gs = 0.f;
#pragma unroll
                                for (int k = 0; k < 32; ++k) {
                                    const float x = ex2_approx(fmaf(__uint_as_float(v[k]), sc, -mnew));
                                    gs += (k <= lim) ? x : 0.f;
                                }
                            }
                            if (q2 == 0) gs0 = gs;
                            else gs1 = gs;
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_u32(tempty_addr + reg * 8);
                    if (cb >= N) continue;  // warp-uniform: padding past the segment end
                    const int b = cb >> gshift;
                    if (G == 64) {
                        Prow[e][static_cast<int64_t>(b) * kRows] = row_valid ? gs0 + gs1 : 0.f;
                    } else {
                        Prow[e][static_cast<int64_t>(b) * kRows] = row_valid ? gs0 : 0.f;
                        if (cb + 32 < N) Prow[e][static_cast<int64_t>(b + 1) * kRows] = row_valid ? gs1 : 0.f;
                    }
                    l[e] += gs0 + gs1;
                }
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t x = (it.sid * (HPC * 2) + (hp + 2 * e) * 2 + c) * kRows + j;
                p.stat_m[x] = valid2[e] ? m[e] : -INFINITY;
                p.stat_l[x] = valid2[e] ? l[e] : 0.f;
            }
            for (int uu = it.u0 + etid; uu < it.u1; uu += 512) p.unit_sid[it.seg_start + uu] = static_cast<int32_t>(it.sid);
            if (warp == 2 && lane == 0) TCW_PHASE(2)
        }
    } else {
        // ===== epilogue: warpgroup wg -> head hh, subtile parity par; thread = query row =====
        const int etid = threadIdx.x - 64;   // 0..511
        const int wg = (warp - 2) >> 2;
        const int hh = wg / NPAR;
        const int par = wg % NPAR;
        const int vh = hh * NPAR + par;      // virtual head of the item statistics
        const int quarter = warp & 3;        // TMEM lane quarter this warp may access
        const int j = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const float sc = p.scale_log2;
        // Lean path (HPC = 4, G = 64: every 128-key subtile is exactly two blocks): barrier
        // addresses held in registers, static block bookkeeping, no per-group branches.
        const uint32_t tfull_addr = smem_u32(t_full), tempty_addr = smem_u32(t_empty);
        const bool lean = NPAR == 1 && C::NG == 4 && G == 64 && UP_TCW_DIAG == 0 && UP_TCW_LEAN;
        // parity epilogues (HPC 2 / 1): every 64-key subtile is one G = 64 block
        const bool lean2 = NPAR > 1 && C::NG == 2 && G == 64 && UP_TCW_DIAG == 0 && UP_TCW_LEAN2;
        uint32_t u = 0;
        uint32_t qiter = 0;
        for (int64_t pos = my_begin; pos < my_end;) {
            const Item it = make_item(P, pos, my_end);
            pos += it.u1 - it.u0;
            const int seg0 = p.cu_seqlens[it.r];
            const int N = p.cu_seqlens[it.r + 1] - seg0;
            const int neff = min(p.query_window_n, N);
            const int key0 = it.u0 * unit_keys;
            const int key1 = min(it.u1 * unit_keys, N);
            const int nsub = (key1 - key0 + C::SK - 1) / C::SK * C::SPS;  // as issued by the MMA warp
            const int vhead = it.hg * HPC + hh;                  // virtual head (q-head * Tt + tile)
            // window row of this row, and (packing) which q-head of the virtual head it is
            const int npad = kRows / p.q_pack;
            const int jr = p.q_pack > 1 ? j % npad : (vhead % p.q_tiles) * kRows + j;
            const int qhead = p.q_pack > 1 ? vhead * p.q_pack + j / npad : vhead / p.q_tiles;
            const bool row_valid = jr < neff;
            const int qpos = N - neff + jr;  // row jr's causal limit (importance.cpp:27)
            const int64_t gb_seg = s_cu_blocks[it.r];
            const int blk0 = key0 / G;
            float* Prow = p.P + (static_cast<int64_t>(vhead) * p.max_blocks + gb_seg) * kRows + j;
            if (C::TS) {
                // Q of this item into TMEM: warpgroup (hh, par) stores its half of head hh's
                // D/2 columns (column c = bf16 elements 2c, 2c+1 of row j; zero rows past
                // n_eff), once the previous item's MMAs have completed (q_empty).
                mbar_wait(q_empty, (qiter & 1) ^ 1);
                ++qiter;
                tc_fence_after();
                constexpr int COLS = D / 2 / NPAR;  // 64 at D = 256, 32 at D = 128
                const __nv_bfloat16* qsrc = p.q + static_cast<int64_t>(seg0 + N - neff + jr) * p.q_row_stride +
                                            static_cast<int64_t>(qhead) * D + par * COLS * 2;
                if constexpr (COLS >= 32) {
#pragma unroll
                    for (int c0 = 0; c0 < COLS; c0 += 32) {
                        uint32_t v[32];
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            uint4 w = make_uint4(0u, 0u, 0u, 0u);
                            if (row_valid) w = __ldg(reinterpret_cast<const uint4*>(qsrc + c0 * 2) + x);
                            v[4 * x + 0] = w.x; v[4 * x + 1] = w.y; v[4 * x + 2] = w.z; v[4 * x + 3] = w.w;
                        }
                        tmem_st32(tmem_base + lane_base + hh * (D / 2) + par * COLS + c0, v);
                    }
                } else {  // HPC = 1 at D = 128: four warpgroups, 16 columns each
                    static_assert(COLS == 16, "TS Q slice");
                    uint32_t v[16];
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        uint4 w = make_uint4(0u, 0u, 0u, 0u);
                        if (row_valid) w = __ldg(reinterpret_cast<const uint4*>(qsrc) + x);
                        v[4 * x + 0] = w.x; v[4 * x + 1] = w.y; v[4 * x + 2] = w.z; v[4 * x + 3] = w.w;
                    }
                    tmem_st16(tmem_base + lane_base + hh * (D / 2) + par * COLS, v);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(q_full);
            }
            float m = -INFINITY, l = 0.f, bsum = 0.f;
            // block bookkeeping: NPAR = 1 walks every group in order (counters, any G that
            // is a multiple of 32); NPAR > 1 sees its parity units only (G = 32, 64, 128: shifts)
            const int gpb = G >> 5;
            const int gshift = G == 128 ? 2 : (G == 64 ? 1 : 0);
            const int ushift = tcw_ushift(G);
            const uint32_t u_item0 = u;  // the CTA's subtile counter at this item's first subtile
            int gib = 0, blk = blk0;
            // This warpgroup's subtiles only (parity of the CTA's subtile counter, see
            // tcw_par_shift): the first one, then every NPAR-th (pairs: t, t + 1, then
            // 2 NPAR - 1 on) -- walking and skipping the others cost the NPAR = 4 epilogue
            // a loop round with a reconvergence point per foreign subtile.
            // (at D = 256 the strided walk's extra live state costs more spills than the
            // skips it saves: there the loop visits every subtile and skips; measured MHA
            // -5.5%, GQA-2 D=128 -6.3%, Gemma / Qwen D=256 +2-3% when strided)
            constexpr bool kStride = NPAR > 1 && D <= 128;
            int t = 0;
            if (kStride) {
                while (t < 2 * NPAR && (((u_item0 + t) >> ushift) % NPAR) != static_cast<uint32_t>(par)) ++t;
                u = u_item0 + t;
            }
            // step to this warpgroup's next subtile from subtile u
            auto next_step = [&](uint32_t uu) -> int {
                return !kStride ? 1 : (ushift == 0 ? NPAR : ((uu & 1u) ? 2 * NPAR - 1 : 1));
            };

#pragma unroll 1
            for (int st = next_step(u); t < nsub; t += st, u += st, st = next_step(u)) {
                if (!kStride && NPAR > 1 && ((u >> ushift) % NPAR) != static_cast<uint32_t>(par)) continue;
                const int cbase = key0 + t * C::SUBN;
                const uint32_t reg = hh * NB + u % NB;
                if constexpr (NPAR == 1 && C::NG == 4) {
                    // Lean fast path: the whole subtile inside the segment and left of every
                    // row's causal limit (warp-uniform), blocks [blk, blk+2) complete here.
                    if (lean && cbase + C::SUBN <= N - neff + 1 && !(UP_TCW_FIRST_REF && __any_sync(0xffffffffu, row_valid && m == -INFINITY))) {
                        mbar_wait_u32(tfull_addr + reg * 8, (u / NB) & 1);
                        tc_fence_after();
                        const uint32_t taddr = tmem_base + lane_base + C::Q_COLS + reg * C::SUBN;
                        uint32_t va[32], vb[32];
                        tmem_ld32(taddr, va);
                        tmem_ld_wait();
                        tmem_ld32(taddr + 32, vb);
                        const float g0 = group_sum_pk<C::NP>(va, pk(sc, sc), pk(-m, -m));
                        tmem_ld_wait();
                        tmem_ld32(taddr + 64, va);
                        const float g1 = group_sum_pk<C::NP>(vb, pk(sc, sc), pk(-m, -m));
                        tmem_ld_wait();
                        tmem_ld32(taddr + 96, vb);
                        const float g2 = group_sum_pk<C::NP>(va, pk(sc, sc), pk(-m, -m));
                        tmem_ld_wait();
                        const float g3 = group_sum_pk<C::NP>(vb, pk(sc, sc), pk(-m, -m));
                        const float b0 = g0 + g1, b1 = g2 + g3;
                        // rows past n_eff carry no statistics: never a reason to leave the lean path
                        if (__all_sync(0xffffffffu, !row_valid || b0 + b1 <= 0x1p40f)) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_u32(tempty_addr + reg * 8);
                            Prow[static_cast<int64_t>(blk) * kRows] = row_valid ? b0 : 0.f;
                            Prow[static_cast<int64_t>(blk + 1) * kRows] = row_valid ? b1 : 0.f;
                            l += b0;
                            l += b1;
                            blk += 2;
                            continue;
                        }
                        // some row must rebase: the general path below redoes this subtile
                        // (its wait returns at once, the region is still held)
                    }
                }
                if constexpr (NPAR > 1 && C::NG == 2) {
                    // Lean path: the subtile (= block cbase / 64) inside the segment and left of
                    // every row's causal limit, a reference m set -- two group sums, one vote;
                    // the same sums the fast path forms ((0 + g0) + g1 = g0 + g1).
                    if (lean2 && cbase + C::SUBN <= N - neff + 1 &&
                        !__any_sync(0xffffffffu, row_valid && m == -INFINITY)) {
                        mbar_wait_u32(tfull_addr + reg * 8, (u / NB) & 1);
                        tc_fence_after();
                        const uint32_t taddr = tmem_base + lane_base + C::Q_COLS + reg * C::SUBN;
                        uint32_t va[32], vb[32];
                        tmem_ld32(taddr, va);
                        tmem_ld_wait();
                        tmem_ld32(taddr + 32, vb);
                        const float g0 = group_sum_pk<C::NP>(va, pk(sc, sc), pk(-m, -m));
                        tmem_ld_wait();
                        const float g1 = group_sum_pk<C::NP>(vb, pk(sc, sc), pk(-m, -m));
                        const float b0 = g0 + g1;
                        if (__all_sync(0xffffffffu, !row_valid || b0 <= 0x1p40f)) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_u32(tempty_addr + reg * 8);
                            Prow[static_cast<int64_t>(cbase >> 6) * kRows] = row_valid ? b0 : 0.f;
                            l += b0;
                            continue;
                        }
                        // some row must rebase: the general path redoes the subtile
                    }
                }
                mbar_wait(&t_full[reg], (u / NB) & 1);
                tc_fence_after();
                if (warp == 2 && lane == 0) TCW_PHASE(1)
                const uint32_t taddr = tmem_base + lane_base + C::Q_COLS + reg * C::SUBN;
                // Fast path (warp-uniform): all 64 keys inside the segment and left of every
                // row's causal limit -> two packed group sums and one overflow check.  The
                // region goes back to the MMA warp after the check, so the generic path can
                // re-read it.
                // (an item's first subtile has no reference m yet: the generic path sets it
                // from the first group's maximum instead of overflowing and rebasing)
                const bool fast = cbase + C::SUBN <= N - neff + 1 && UP_TCW_DIAG != 1 &&
                                  !(UP_TCW_FIRST_REF && __any_sync(0xffffffffu, row_valid && m == -INFINITY));
                float gs0 = 0.f, gs1 = 0.f, gs2 = 0.f, gs3 = 0.f;
                bool redo = !fast && cbase < N && UP_TCW_DIAG != 1;
                if (fast) {
                    if constexpr (UP_TCW_LD_PIPE && C::NG == 4) {
                        // the next group's TMEM load is in flight while this group is summed
                        uint32_t va[32], vb[32];
                        tmem_ld32(taddr, va);
                        tmem_ld_wait();
                        tmem_ld32(taddr + 32, vb);
                        gs0 = group_sum_pk<C::NP>(va, pk(sc, sc), pk(-m, -m));
                        tmem_ld_wait();
                        tmem_ld32(taddr + 64, va);
                        gs1 = group_sum_pk<C::NP>(vb, pk(sc, sc), pk(-m, -m));
                        tmem_ld_wait();
                        tmem_ld32(taddr + 96, vb);
                        gs2 = group_sum_pk<C::NP>(va, pk(sc, sc), pk(-m, -m));
                        tmem_ld_wait();
                        gs3 = group_sum_pk<C::NP>(vb, pk(sc, sc), pk(-m, -m));
                    } else {
                        uint32_t v[32];
                        tmem_ld32(taddr, v);
                        tmem_ld_wait();
                        gs0 = group_sum_pk<C::NP>(v, pk(sc, sc), pk(-m, -m));
                        tmem_ld32(taddr + 32, v);
                        tmem_ld_wait();
                        gs1 = group_sum_pk<C::NP>(v, pk(sc, sc), pk(-m, -m));
                        if (C::NG == 4) {
                            tmem_ld32(taddr + 64, v);
                            tmem_ld_wait();
                            gs2 = group_sum_pk<C::NP>(v, pk(sc, sc), pk(-m, -m));
                            tmem_ld32(taddr + 96, v);
                            tmem_ld_wait();
                            gs3 = group_sum_pk<C::NP>(v, pk(sc, sc), pk(-m, -m));
                        }
                    }
                    redo = !((gs0 + gs1) + (gs2 + gs3) <= 0x1p40f);
                }
                if (redo) {
                    // Generic path: causal tail, ragged segment end, or a rebase of m.
#pragma unroll 1
                    for (int q2 = 0; q2 < C::NG; ++q2) {
                        const int c0 = cbase + q2 * 32;
                        const int lim = min(qpos - c0, min(31, N - 1 - c0));  // last valid column
                        uint32_t v[32];
                        tmem_ld32(taddr + q2 * 32, v);
                        tmem_ld_wait();
                        float gs = 0.f;
                        if (UP_TCW_FIRST_REF && lim >= 0 && m == -INFINITY) m = first_ref(v, lim, sc);
                        if (lim >= 0) {
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
                        if (!(gs <= 0x1p40f)) {
                            // Rebase: move m to this group's maximum (see score_tc.cu).
                            float gmax = -INFINITY;
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (k <= lim) gmax = fmaxf(gmax, __uint_as_float(v[k]));
                            const float mnew = fmaxf(m, gmax * sc);
                            if (m != -INFINITY) {
                                const float f = ex2_approx(m - mnew);
                                l *= f;
                                bsum *= f;
                                // groups of this subtile before q2 are not yet folded into bsum
                                gs0 *= f;
                                gs1 *= f;
                                gs2 *= f;
                                rescale_rows_par(Prow, blk0, NPAR == 1 ? blk : cbase >> (5 + gshift), G, NPAR,
                                                 par, f, key0, u_item0);
                            }
                            m = mnew;
                            gs = 0.f;
#pragma unroll
                            for (int k = 0; k < 32; ++k) {
                                const float e = ex2_approx(fmaf(__uint_as_float(v[k]), sc, -mnew));
                                gs += (k <= lim) ? e : 0.f;
                            }
                        }
                        if (q2 == 0) gs0 = gs;
                        else if (q2 == 1) gs1 = gs;
                        else if (q2 == 2) gs2 = gs;
                        else gs3 = gs;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&t_empty[reg]);
                if (cbase >= N) continue;  // warp-uniform: padding subtile past the segment end
#pragma unroll
                for (int q2 = 0; q2 < C::NG; ++q2) {
                    const int c0 = cbase + q2 * 32;
                    if (c0 >= N) break;  // warp-uniform
                    bsum += q2 == 0 ? gs0 : (q2 == 1 ? gs1 : (q2 == 2 ? gs2 : gs3));
                    bool done;
                    int b;
                    if (NPAR == 1) {
                        done = ++gib == gpb || c0 + 32 >= N;
                        b = blk;
                    } else {
                        const int gi = c0 >> 5;
                        done = (gi & (gpb - 1)) == gpb - 1 || c0 + 32 >= N;
                        b = gi >> gshift;
                    }
                    if (done) {  // block b complete
                        Prow[static_cast<int64_t>(b) * kRows] = row_valid ? bsum : 0.f;
                        l += bsum;
                        bsum = 0.f;
                        gib = 0;
                        ++blk;
                    }
                }
            }
            if (kStride) u = u_item0 + nsub;  // the CTA counter past this item (every warpgroup)
            {
                const int64_t x = (it.sid * (HPC * NPAR) + vh) * kRows + j;
                p.stat_m[x] = row_valid ? m : -INFINITY;
                p.stat_l[x] = row_valid ? l : 0.f;
            }
            {
                constexpr int spu = kTileKeys / C::SUBN;  // subtiles per 128-key unit
                for (int uu = it.u0 + etid; uu < it.u1; uu += 512) {
                    const uint32_t par0 = NPAR > 1 ? ((u_item0 + (uu - it.u0) * spu) >> ushift) % NPAR : 0u;
                    p.unit_sid[it.seg_start + uu] = tcw_usid(static_cast<int32_t>(it.sid), static_cast<int>(par0));
                }
            }
            if (warp == 2 && lane == 0) TCW_PHASE(2)
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
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.dbg[blockIdx.x * 4 + 3] = smid;
    }
}

template <int D, int HPC, bool SPLIT = false>
static cudaError_t launch_tcw(const CUtensorMap& qm, const CUtensorMap& km, const ScoreTcParams& p, int grid,
                              cudaStream_t stream) {
    using C = TcwCfg<D, HPC, SPLIT>;
    const int smem = C::smem(p.num_requests);
    if (p.num_requests > kTcwMaxRequests || smem > 232448) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(score_tcw_kernel<D, HPC, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e != cudaSuccess) return e;
    return launch_k(kPdlScore, score_tcw_kernel<D, HPC, SPLIT>, grid, C::THREADS, smem, stream, qm, km, p);
}

// SPLIT epilogue for four q-heads per kv-head when every block lies inside a 64-key half,
// chosen for small launches (at most ~4 128-key units per CTA under the capacity: the
// latency-bound C1-class batches, LLaMA 1x4K scorer stage 30.4 -> 29.4 us).  On large
// launches the one-warpgroup-per-head epilogue is 1.4% faster (LLaMA 4x32K 157.9 vs
// 160.1 us): there the idle warpgroup's MUFU share goes to the other three.
// UP_TCW_SPLIT=0/1 forces either epilogue (A/B timing).
bool tcw_split(int D, int HPC, int G, int64_t max_tokens, int nhg, int grid) {
    static const int force = [] {
        const char* s = std::getenv("UP_TCW_SPLIT");
        return s == nullptr ? -1 : (s[0] == '0' ? 0 : 1);
    }();
    if (!(HPC == 4 && (D == 64 || D == 128) && (G == 32 || G == 64))) return false;
    if (force >= 0) return force == 1;
    return (max_tokens / kTileKeys + 1) * nhg <= 4LL * grid;
}

int tcw_par_shift_for(int G) { return tcw_par_shift(G); }

// statistics rows per head the tail kernels must merge
int tcw_npar(int D, int HPC, int G, int64_t max_tokens, int nhg, int grid) {
    return tcw_split(D, HPC, G, max_tokens, nhg, grid) ? 2 : 4 / HPC;
}

// Keys per K stage (the K tensor map's box rows).
int tcw_stage_keys(int D) { return D <= 128 ? TcwCfg<128, 4>::SK : TcwCfg<256, 2>::SK; }

// Shapes this kernel serves: HPC = 4 at D in {64, 128}, HPC = 2 at D in {64, 128, 256}; with HPC = 2 the
// block size must be 32 or 64 (blocks inside one 64-key subtile).
bool tcw_supported(int D, int HPC, int G, int R) {
    if (R > kTcwMaxRequests || G % 32 != 0) return false;
    if (HPC == 4) return D == 64 || D == 128;
    // G = 128 pairs subtiles per parity unit: a warpgroup's waits on the TMEM ring are then
    // up to 2 NPAR - 1 subtiles apart, which needs NB >= 2 NPAR - 1 regions per head
    // (HPC 2 at D <= 128: NB 3-4; HPC 1 at D = 128: NB 7; not D = 256, where TS Q leaves 2 / 6)
    if (HPC == 2) return (D == 64 || D == 128 || D == 256) && (G == 32 || G == 64 || (G == 128 && D <= 128));
#ifndef UP_NO_TCW_HPC1  // dev A/B: MHA shapes back on score_tc
    if (HPC == 1) return (D == 128 || D == 256) && (G == 32 || G == 64 || (G == 128 && D == 128));  // TS, four parity warpgroups
#endif
    return false;
}

cudaError_t launch_score_tcw(int D, int HPC, const CUtensorMap& qm, const CUtensorMap& km, const ScoreTcParams& p,
                             int grid, cudaStream_t stream) {
    if (tcw_split(D, HPC, p.block_size_g, p.max_tokens, p.num_hgroups, grid)) {
        if (D == 64) return launch_tcw<64, 4, true>(qm, km, p, grid, stream);
        return launch_tcw<128, 4, true>(qm, km, p, grid, stream);
    }
    if (D == 64 && HPC == 4) return launch_tcw<64, 4>(qm, km, p, grid, stream);
    if (D == 64 && HPC == 2) return launch_tcw<64, 2>(qm, km, p, grid, stream);
    if (D == 128 && HPC == 4) return launch_tcw<128, 4>(qm, km, p, grid, stream);
    if (D == 128 && HPC == 2) return launch_tcw<128, 2>(qm, km, p, grid, stream);
    if (D == 256 && HPC == 2) return launch_tcw<256, 2>(qm, km, p, grid, stream);
    if (D == 128 && HPC == 1) return launch_tcw<128, 1>(qm, km, p, grid, stream);
    if (D == 256 && HPC == 1) return launch_tcw<256, 1>(qm, km, p, grid, stream);
    return cudaErrorInvalidValue;
}

}  // namespace up
