// attention.cu -- the drop layer's attention readout over the retained rows (SURVEY §8f
// row 1): attention_readout (model.cpp:215-263) as prefill_layer_step calls it after the
// selection (propagation.cpp:195-205) -- every retained query row attends to the retained
// keys of its segment whose logical position lies in (pos_q - window, pos_q], softmax of
// q·k/sqrt(D) over v.  The compacted rows come straight from up_compact (positions strictly
// increasing per segment), so the visible keys of a row are one contiguous index range
// [lo, hi) found by binary search over the positions.
//
// One CTA per (128-row query tile, q-head), six warps:
//   warp 0     TMA producer: Q tile once, then K tiles (3-stage ring) and V tiles (2-stage)
//   warp 1     MMA issuer (one elected thread): S_j = Q·K_j^T (ss, into TMEM S[j&1]);
//              O += P_j·V_j (ts: P from TMEM, V as an MN-major smem operand)
//   warps 2-5  softmax: one TMEM lane = one query row per thread; online softmax with a lazy
//              reference (O and l are rescaled only when the row max grows by > 2^8), P
//              written to TMEM as bf16 pairs, final O / l stored as bf16
// TMEM (512 columns): S0, S1 (BN columns each), O (D columns), P0, P1 (BN/2 columns each);
// BN = 128 keys per tile for D <= 128, 64 for D = 256.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "params.cuh"

namespace up {

template <int D>
struct AttnCfg {
    // D=256: 64-key tiles; Q resident in TMEM (the S MMA reads A from tensor memory, so it
    // streams only K from smem: with A in smem an M=128, N=64 MMA needs 6 KB per 32 cycles,
    // above the 128 B/clk smem port); P_j is written over the columns of S_j.  TMEM:
    // S0 [0,64), S1 [64,128), O [128,384), Q [384,512).  The freed smem holds 4 K + 3 V stages.
    static constexpr int BM = 128, BN = D > 128 ? 64 : 128;
    static constexpr int NCH = D / 64;                    // 64-element (128-byte) column boxes
    static constexpr int KBOX = BN * 128;                 // one box of a K/V tile
    static constexpr int KV_STAGE = NCH * KBOX;
    static constexpr int KST = 4, VST = 3;
    static constexpr int NBAR = 1 + 2 * KST + 2 * VST + 2 + 2 + 2;
    static constexpr int THREADS = 192;
    static constexpr uint32_t S_COL = 0, O_COL = 2 * BN, Q_COL = 2 * BN + D;
    static_assert(Q_COL + D / 2 <= 512, "TMEM columns");
    static constexpr int smem() { return 1024 + (KST + VST) * KV_STAGE + NBAR * 8 + 64; }
    static_assert(smem() <= 232448 - 1024, "shared memory");
};

// K / V ring depths of the two-tile kernel (D <= 128)
#ifndef UP_ATTN2_KST
#define UP_ATTN2_KST 2
#endif
#ifndef UP_ATTN2_VST
#define UP_ATTN2_VST 2
#endif

// Of every 16 element pairs of a full tile, this many take exp2 on the FMA pipe
// (tools/attn_sweep.sh, tools/attn2_sweep.sh on B200: 1 is best at D = 128, 0 at D = 256).
#ifdef UP_ATTN_POLY_PAIRS
template <int D> constexpr int kAttnPolyPairs = UP_ATTN_POLY_PAIRS;
#else
template <int D> constexpr int kAttnPolyPairs = D > 128 ? 0 : 1;
#endif

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// Rows [r0, rows) of a K/V stage ([nch boxes][rows][128 B], swizzle permutes 16-byte chunks
// within a row only) -> 0.  Rows past the batch's last row hold whatever the caller's buffer
// holds there; their keys are masked (P = 0), but 0 * NaN in the PV MMA would still poison
// O, so the V rows of a tile that runs past the batch are cleared before the MMA reads them.
__device__ __forceinline__ void zero_stage_rows(uint8_t* stage, int nch, int box_bytes, int r0, int rows, int tid,
                                                int nthreads) {
    const int per_box = (rows - r0) * 8;  // 16-byte chunks
    for (int x = tid; x < nch * per_box; x += nthreads) {
        const int c = x / per_box, rem = x - c * per_box;
        reinterpret_cast<uint4*>(stage + c * box_bytes + (r0 + rem / 8) * 128)[rem % 8] = make_uint4(0, 0, 0, 0);
    }
}

// first index i in [b, e) with pos[i] > x (upper_bound) / >= x (lower_bound)
__device__ __forceinline__ int64_t upper_pos(const int64_t* pos, int64_t b, int64_t e, int64_t x) {
    while (b < e) {
        const int64_t m = (b + e) >> 1;
        if (pos[m] <= x) b = m + 1; else e = m;
    }
    return b;
}
__device__ __forceinline__ int64_t lower_pos(const int64_t* pos, int64_t b, int64_t e, int64_t x) {
    while (b < e) {
        const int64_t m = (b + e) >> 1;
        if (pos[m] < x) b = m + 1; else e = m;
    }
    return b;
}

template <int D>
__global__ void __launch_bounds__(192, 1)
attention_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                 const __grid_constant__ CUtensorMap vmap, const AttnParams p) {
    using C = AttnCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sk = smem;
    uint8_t* sv = sk + C::KST * C::KV_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sv + C::VST * C::KV_STAGE);
    uint64_t* q_full = bars;  // the four softmax warps have stored their Q rows in TMEM
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + C::KST;
    uint64_t* v_full = k_empty + C::KST;
    uint64_t* v_empty = v_full + C::VST;
    uint64_t* s_full = v_empty + C::VST;
    uint64_t* p_full = s_full + 2;
    uint64_t* pv_done = p_full + 2;
    int64_t* plan = reinterpret_cast<int64_t*>(bars + C::NBAR);  // q0, seg_begin, seg_end, k_begin, k_end
    uint32_t* misc = reinterpret_cast<uint32_t*>(plan + 5);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int H = p.num_q_heads;
    const int h = blockIdx.x % H;
    const int trev = blockIdx.x / H;

    if (threadIdx.x == 0) {
        // Tile of this CTA: tiles are numbered over the segments, last tile first (the causal
        // tail tiles carry the most keys; scheduling them first evens out the wave).
        const int R = p.num_requests;
        int total = 0;
        for (int r = 0; r < R; ++r) total += (p.cu_seqlens[r + 1] - p.cu_seqlens[r] + C::BM - 1) / C::BM;
        int64_t q0 = -1, sb = 0, se = 0, kb = 0, ke = 0;
        const bool bad = p.cu_seqlens[R] > p.max_tokens;  // malformed batch: no rows touched
        if (bad && blockIdx.x == 0) raise_error(p.err, kErrBadSeqlens);
        if (trev < total && !bad) {
            int t = total - 1 - trev;
            for (int r = 0; r < R; ++r) {
                const int n = p.cu_seqlens[r + 1] - p.cu_seqlens[r];
                const int nt = (n + C::BM - 1) / C::BM;
                if (t < nt) {
                    sb = p.cu_seqlens[r];
                    se = p.cu_seqlens[r + 1];
                    q0 = sb + static_cast<int64_t>(t) * C::BM;
                    break;
                }
                t -= nt;
            }
            const int64_t qlast = (q0 + C::BM < se ? q0 + C::BM : se) - 1;
            ke = p.window > 0 ? upper_pos(p.positions, sb, se, p.positions[qlast]) : qlast + 1;
            kb = p.window > 0 ? lower_pos(p.positions, sb, se, p.positions[q0] - p.window + 1) : sb;
        }
        plan[0] = q0;
        plan[1] = sb;
        plan[2] = se;
        plan[3] = kb;
        plan[4] = ke;
        mbar_init(q_full, 4);
        for (int s = 0; s < C::KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < C::VST; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&s_full[s], 1); mbar_init(&p_full[s], 4); mbar_init(&pv_done[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const int64_t q0 = plan[0];
    if (q0 < 0) return;  // beyond the batch's tiles (the grid is sized for the capacity)
    const int64_t seg_begin = plan[1], seg_end = plan[2], k_begin = plan[3], k_end = plan[4];
    const int nt = static_cast<int>((k_end - k_begin + C::BN - 1) / C::BN);
    const int qh = p.q_head_offset + h;
    const int kvh = qh / p.gqa_group - p.kv_head_offset;

    if (warp == 1) tmem_alloc(misc, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];

    if (warp == 0) {
        if (lane == 0) {
            prefetch_tensormap(&qmap);
            prefetch_tensormap(&kmap);
            prefetch_tensormap(&vmap);
            for (int j = 0; j < nt; ++j) {
                const int32_t row = static_cast<int32_t>(k_begin + static_cast<int64_t>(j) * C::BN);
                const int ks = j % C::KST;
                if (j >= C::KST) mbar_wait(&k_empty[ks], ((j / C::KST) - 1) & 1);
                mbar_arrive_expect_tx(&k_full[ks], C::KV_STAGE);
                for (int c = 0; c < C::NCH; ++c)
                    tma_load_2d(sk + ks * C::KV_STAGE + c * C::KBOX, &kmap, &k_full[ks], kvh * D + c * 64, row);
                const int vs = j % C::VST;
                if (j >= C::VST) mbar_wait(&v_empty[vs], ((j / C::VST) - 1) & 1);
                mbar_arrive_expect_tx(&v_full[vs], C::KV_STAGE);
                for (int c = 0; c < C::NCH; ++c)
                    tma_load_2d(sv + vs * C::KV_STAGE + c * C::KBOX, &vmap, &v_full[vs], kvh * D + c * 64, row);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t kIdescS = idesc_bf16_f32(128, C::BN);
            constexpr uint32_t kIdescO = idesc_bf16_f32(128, D) | (1u << 16);  // B (V) MN-major
            const uint64_t k_base = smem_desc_sw128(smem_u32(sk));
            const uint64_t v_base = smem_desc_sw128_mn(smem_u32(sv), C::KBOX, 1024);
            mbar_wait(q_full, 0);
            tc_fence_after();
            auto issue_s = [&](int j) {
                const int ks = j % C::KST;
                mbar_wait(&k_full[ks], (j / C::KST) & 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + C::S_COL + (j & 1) * C::BN;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {  // A = Q columns [kk*8, kk*8+8) in TMEM
                    const uint32_t koff = (kk & 3) * 32;
                    mma_bf16_ts(d_tmem, tmem + C::Q_COL + kk * 8,
                                k_base + ((ks * C::KV_STAGE + (kk >> 2) * C::KBOX + koff) >> 4), kIdescS,
                                kk > 0 ? 1u : 0u);
                }
                mma_commit(&k_empty[ks]);
                mma_commit(&s_full[j & 1]);
            };
            issue_s(0);
            if (nt > 1) issue_s(1);
            for (int j = 0; j < nt; ++j) {
                mbar_wait(&p_full[j & 1], (j >> 1) & 1);
                const int vs = j % C::VST;
                mbar_wait(&v_full[vs], (j / C::VST) & 1);
                tc_fence_after();
                const uint32_t a_tmem = tmem + C::S_COL + (j & 1) * C::BN;  // P_j over S_j
#pragma unroll
                for (int kk = 0; kk < C::BN / 16; ++kk)  // 16 keys = two 8-row swizzle atoms
                    mma_bf16_ts(tmem + C::O_COL, a_tmem + kk * 8,
                                v_base + ((vs * C::KV_STAGE + kk * 2048) >> 4), kIdescO,
                                (j > 0 || kk > 0) ? 1u : 0u);
                mma_commit(&v_empty[vs]);
                mma_commit(&pv_done[j & 1]);
                if (j + 2 < nt) issue_s(j + 2);
            }
        }
    } else {
        // softmax warps: TMEM lane quarter = warp % 4
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const int64_t qi = q0 + r;
        const bool valid = qi < seg_end;
        int64_t lo = 0, hi = 0;
        if (valid) {
            const int64_t qp = p.positions[qi];
            // strictly increasing positions: without a window the keys are [seg_begin, qi]
            hi = p.window > 0 ? upper_pos(p.positions, seg_begin, seg_end, qp) : qi + 1;
            lo = p.window > 0 ? lower_pos(p.positions, seg_begin, seg_end, qp - p.window + 1) : seg_begin;
            if (lo >= hi) raise_error(p.err, kErrNoVisibleKey);
        }
        {
            // this row of Q into TMEM (column c = bf16 elements 2c, 2c+1; zero past the segment)
            const __nv_bfloat16* qsrc = p.q + qi * p.q_row_stride + static_cast<int64_t>(h) * D;
#pragma unroll
            for (int c0 = 0; c0 < D / 2; c0 += 32) {
                uint32_t v[32];
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    uint4 w = make_uint4(0u, 0u, 0u, 0u);
                    if (valid) w = __ldg(reinterpret_cast<const uint4*>(qsrc + c0 * 2) + x);
                    v[4 * x + 0] = w.x; v[4 * x + 1] = w.y; v[4 * x + 2] = w.z; v[4 * x + 3] = w.w;
                }
                tmem_st32(tmem + lane_base + C::Q_COL + c0, v);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(q_full);
        }
        const float c = p.scale_log2;
        const int64_t total_rows = p.cu_seqlens[p.num_requests];
        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < nt; ++j) {
            const int64_t kb = k_begin + static_cast<int64_t>(j) * C::BN;
            const int vis0 = static_cast<int>(lo - kb < 0 ? 0 : (lo - kb > C::BN ? C::BN : lo - kb));
            const int vis1 = static_cast<int>(hi - kb < 0 ? 0 : (hi - kb > C::BN ? C::BN : hi - kb));
            // warp-uniform: the two P paths below store with tcgen05.st (.sync.aligned)
            const bool full = __all_sync(0xffffffffu, vis0 == 0 && vis1 == C::BN);
            mbar_wait(&s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            const uint32_t s_addr = tmem + lane_base + C::S_COL + (j & 1) * C::BN;
            uint32_t s[C::BN];
#pragma unroll
            for (int q = 0; q < C::BN / 32; ++q)
                tmem_ld32(s_addr + q * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[q * 32]));
            tmem_ld_wait();
            float mx = -INFINITY;
            if (full) {  // four independent three-input max chains
                float a[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int i = 0; i < C::BN; i += 8)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        a[u] = fmax3(a[u], __uint_as_float(s[i + 2 * u]), __uint_as_float(s[i + 2 * u + 1]));
                mx = fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
            } else {
#pragma unroll
                for (int i = 0; i < C::BN; ++i)
                    if (i >= vis0 && i < vis1) mx = fmaxf(mx, __uint_as_float(s[i]));
            }
            mx *= c;
            // lazy rescale: keep the reference unless the max grew by more than 2^8.  The
            // decision is per row, the O rescale warp-wide (tcgen05.ld/st are .sync.aligned).
            const bool grow = mx > m_run + 8.f;
            float alpha = 1.f;
            if (grow) {
                alpha = m_run == -INFINITY ? 0.f : ex2_approx(m_run - mx);
                l_run *= alpha;
                m_run = mx;
            }
            if (j > 0 && __any_sync(0xffffffffu, grow)) {
                // O holds PV_0..PV_{j-1}: wait for the last one, then scale
                mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int q = 0; q < D / 32; ++q) {
                    uint32_t o[32];
                    tmem_ld32(tmem + lane_base + C::O_COL + q * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tmem_st32(tmem + lane_base + C::O_COL + q * 32, o);
                }
            }
            // P_j goes over S_j (all of S_j is in registers); S_j was issued after PV_{j-2},
            // so the MMA pipe already consumed P_{j-2} from these columns
            const float mref = m_run == -INFINITY ? 0.f : m_run;
            float lsum = 0.f;
            const uint32_t p_addr = s_addr;
            if (full) {
                // packed FFMA2 arguments; of every 16 pairs kAttnPolyPairs take 2^x on the FMA
                // pipe (exp2_poly2) instead of MUFU.EX2, which alone would need as many cycles
                // per tile as the two MMAs; packed FADD2 row sums
                const uint64_t c2 = pk(c, c), m2 = pk(-mref, -mref);
                uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
                for (int q = 0; q < C::BN / 32; ++q) {
                    uint32_t pk16[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int e0 = q * 32 + 2 * i;
                        const uint64_t x = fma2(static_cast<uint64_t>(s[e0]) | (static_cast<uint64_t>(s[e0 + 1]) << 32),
                                                c2, m2);
                        const uint64_t e = i < 16 - kAttnPolyPairs<D> ? pk(ex2_approx(lo_f(x)), ex2_approx(hi_f(x)))
                                                                   : exp2_poly2(x);
                        if (q == 0 && i == 0) acc0 = e;
                        else if (q == 0 && i == 1) acc1 = e;
                        else if (i & 1) acc1 = add2(acc1, e);
                        else acc0 = add2(acc0, e);
                        pk16[i] = pack_bf16(lo_f(e), hi_f(e));
                    }
                    tmem_st16(p_addr + q * 16, pk16);
                }
                const uint64_t a2 = add2(acc0, acc1);
                lsum = lo_f(a2) + hi_f(a2);
            } else {
#pragma unroll
            for (int q = 0; q < C::BN / 32; ++q) {
                uint32_t pk16[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int e0 = q * 32 + 2 * i, e1 = e0 + 1;
                    float p0 = ex2_approx(fmaf(__uint_as_float(s[e0]), c, -mref));
                    float p1 = ex2_approx(fmaf(__uint_as_float(s[e1]), c, -mref));
                    if (!full) {
                        if (e0 < vis0 || e0 >= vis1) p0 = 0.f;
                        if (e1 < vis0 || e1 >= vis1) p1 = 0.f;
                    }
                    lsum += p0 + p1;
                    pk16[i] = pack_bf16(p0, p1);
                }
                tmem_st16(p_addr + q * 16, pk16);
            }
            }
            l_run += lsum;
            if (kb + C::BN > total_rows) {  // V rows past the batch -> 0 before PV_j reads them
                const int vs = j % C::VST;
                mbar_wait(&v_full[vs], (j / C::VST) & 1);
                zero_stage_rows(sv + vs * C::KV_STAGE, C::NCH, C::KBOX,
                                static_cast<int>(total_rows - kb > 0 ? total_rows - kb : 0), C::BN, threadIdx.x - 64, 128);
                fence_proxy_async_smem();
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[j & 1]);
        }
        // epilogue: O / l -> bf16
        if (nt > 0) {
            mbar_wait(&pv_done[(nt - 1) & 1], ((nt - 1) >> 1) & 1);
            tc_fence_after();
        }
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        __nv_bfloat16* orow = p.out + qi * p.out_row_stride + static_cast<int64_t>(h) * D;
#pragma unroll
        for (int q = 0; q < D / 32; ++q) {
            uint32_t o[32];
            tmem_ld32(tmem + lane_base + C::O_COL + q * 32, o);
            tmem_ld_wait();
            if (valid) {
                uint4 w[4];
                uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    wp[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
                uint4* dst = reinterpret_cast<uint4*>(orow + q * 32);
#pragma unroll
                for (int i = 0; i < 4; ++i) dst[i] = w[i];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------------------
// D <= 128: persistent, one CTA per SM; each CTA takes work items = (pair of 128-row query
// tiles of one segment, q-head), heaviest first.  Twelve warps:
//   warp 0       TMA producer: Q0, Q1 per item (after the item before released them), then
//                K_j / V_j (128 keys, 2-stage rings running across items) shared by both tiles
//   warp 1       MMA issuer: S_i,j = Q_i·K_j^T into TMEM S_i; O_i += P_i,j·V_j with P_i,j read
//                from the S_i columns it overwrote (ts).  Issue order S0,0 S1,0 | PV0,j S0,j+1
//                PV1,j S1,j+1 | ...: tcgen05.mma of one thread execute in issue order, so
//                S_i,j+1 overwrites S_i only after PV_i,j consumed P_i,j, and while one
//                softmax warpgroup works on its tile the tensor pipe runs the other tile's
//                PV and S (two softmax warps per SMSP hide each other's latency).  The next
//                item's first S MMAs overlap this item's epilogue.
//   warp 2       scheduler: takes items from a global counter (heaviest first), plans them
//                into a 2-deep smem ring
//   warp 3       idle
//   warps 4-7    softmax of tile 0, warps 8-11 softmax of tile 1 (TMEM lane = query row)
// TMEM: S0 [0,128), S1 [128,256), O0 [256, 256+D), O1 [256+D, 256+2D).
template <int D>
struct Attn2Cfg {
    static constexpr int BM = 128, BN = 128;
    static constexpr int NCH = D / 64;
    static constexpr int BOX = 128 * 128;                 // 128 rows x 128 bytes
    static constexpr int Q_BYTES = NCH * BOX;             // one query tile
    static constexpr int KV_STAGE = NCH * BOX;
    static constexpr int KST = UP_ATTN2_KST, VST = UP_ATTN2_VST;
    static constexpr int PLANS = 2;                       // work-item ring depth
    static constexpr int NBAR = 2 + 2 * KST + 2 * VST + 2 + 4 + 2 + 2 * PLANS;
    static constexpr int THREADS = 384;
    static constexpr uint32_t S_COL = 0, O_COL = 2 * BN;
    static_assert(O_COL + 2 * D <= 512, "TMEM columns");
    static constexpr int smem() { return 1024 + 2 * Q_BYTES + (KST + VST) * KV_STAGE + NBAR * 8 + 64 + PLANS * 48; }
    static_assert(smem() <= 232448 - 1024, "shared memory");
};

// Work item = (pair of 128-row query tiles of one segment, q-head).  Pairs are numbered
// over the segments with the last pair of the last segment first (the causal tail pairs
// carry the most keys), the heads of one pair consecutive (they share K/V in L2); CTAs
// take items from a global counter, so the heavy ones go first and the tail balances.
struct PairPlan {
    int64_t q0, seg_begin, seg_end, k_begin;
    int32_t nt;  // 128-key tiles; -1 = no more work
    int32_t h;   // local q-head
};

__device__ __forceinline__ int total_pairs(const AttnParams& p) {
    int total = 0;
    for (int r = 0; r < p.num_requests; ++r) total += (p.cu_seqlens[r + 1] - p.cu_seqlens[r] + 255) / 256;
    return total;
}

__device__ PairPlan pair_plan(const AttnParams& p, int trev, int total) {
    PairPlan pl{0, 0, 0, 0, 0, 0};
    int t = total - 1 - trev;
    for (int r = 0; r < p.num_requests; ++r) {
        const int n = p.cu_seqlens[r + 1] - p.cu_seqlens[r];
        const int np = (n + 255) / 256;
        if (t < np) {
            pl.seg_begin = p.cu_seqlens[r];
            pl.seg_end = p.cu_seqlens[r + 1];
            pl.q0 = pl.seg_begin + static_cast<int64_t>(t) * 256;
            break;
        }
        t -= np;
    }
    const int64_t qlast = (pl.q0 + 256 < pl.seg_end ? pl.q0 + 256 : pl.seg_end) - 1;
    // positions strictly increase within a segment, so without a window the visible keys
    // of row i are exactly [seg_begin, i]: no search
    const int64_t ke = p.window > 0 ? upper_pos(p.positions, pl.seg_begin, pl.seg_end, p.positions[qlast]) : qlast + 1;
    pl.k_begin = p.window > 0 ? lower_pos(p.positions, pl.seg_begin, pl.seg_end, p.positions[pl.q0] - p.window + 1)
                              : pl.seg_begin;
    pl.nt = static_cast<int32_t>((ke - pl.k_begin + 127) / 128);
    return pl;
}

template <int D>
__global__ void __launch_bounds__(384, 1)
attention2q_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                   const __grid_constant__ CUtensorMap vmap, const AttnParams p) {
    using C = Attn2Cfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sq = smem;                                   // Q0 | Q1
    uint8_t* sk = sq + 2 * C::Q_BYTES;
    uint8_t* sv = sk + C::KST * C::KV_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sv + C::VST * C::KV_STAGE);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;
    uint64_t* k_empty = k_full + C::KST;
    uint64_t* v_full = k_empty + C::KST;
    uint64_t* v_empty = v_full + C::VST;
    uint64_t* s_full = v_empty + C::VST;                  // [tile]
    uint64_t* p_full = s_full + 2;                        // [tile][key half]
    uint64_t* o_done = p_full + 4;                        // [tile]
    uint64_t* plan_full = o_done + 2;                     // [PLANS]
    uint64_t* plan_empty = plan_full + C::PLANS;          // [PLANS]
    PairPlan* plans = reinterpret_cast<PairPlan*>(bars + C::NBAR);
    uint32_t* misc = reinterpret_cast<uint32_t*>(plans + C::PLANS);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int H = p.num_q_heads;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int s = 0; s < C::KST; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < C::VST; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&s_full[s], 1); mbar_init(&o_done[s], 1); }
        for (int s = 0; s < 4; ++s) mbar_init(&p_full[s], 4);
        // a plan is read by the TMA warp, the MMA warp and the eight softmax warps
        for (int s = 0; s < C::PLANS; ++s) { mbar_init(&plan_full[s], 1); mbar_init(&plan_empty[s], 10); }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(misc, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];
    // next work item of this CTA (written by the scheduler warp), read by a whole warp
    auto take_plan = [&](int it) {
        const int slot = it % C::PLANS;
        mbar_wait(&plan_full[slot], (it / C::PLANS) & 1);
        const PairPlan pl = plans[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&plan_empty[slot]);
        return pl;
    };

    if (warp == 0) {
        if (lane == 0) {
            prefetch_tensormap(&qmap);
            prefetch_tensormap(&kmap);
            prefetch_tensormap(&vmap);
        }
        uint32_t kv = 0;  // K/V tiles loaded so far (ring position)
        for (int it = 0;; ++it) {
            const PairPlan pl = take_plan(it);
            if (pl.nt < 0) break;
            const int h = pl.h;
            const int kvh = (p.q_head_offset + h) / p.gqa_group - p.kv_head_offset;
            if (lane == 0) {
                if (it > 0) mbar_wait(q_empty, (it - 1) & 1);  // last S MMAs of the previous item done
                mbar_arrive_expect_tx(q_full, 2 * C::Q_BYTES);
                for (int t = 0; t < 2; ++t)
                    for (int c = 0; c < C::NCH; ++c)
                        tma_load_2d(sq + t * C::Q_BYTES + c * C::BOX, &qmap, q_full, h * D + c * 64,
                                    static_cast<int32_t>(pl.q0 + t * C::BM));
                for (int j = 0; j < pl.nt; ++j, ++kv) {
                    const int32_t row = static_cast<int32_t>(pl.k_begin + static_cast<int64_t>(j) * C::BN);
                    const uint32_t ks = kv % C::KST;
                    if (kv >= C::KST) mbar_wait(&k_empty[ks], ((kv / C::KST) - 1) & 1);
                    mbar_arrive_expect_tx(&k_full[ks], C::KV_STAGE);
                    for (int c = 0; c < C::NCH; ++c)
                        tma_load_2d(sk + ks * C::KV_STAGE + c * C::BOX, &kmap, &k_full[ks], kvh * D + c * 64, row);
                    const uint32_t vs = kv % C::VST;
                    if (kv >= C::VST) mbar_wait(&v_empty[vs], ((kv / C::VST) - 1) & 1);
                    mbar_arrive_expect_tx(&v_full[vs], C::KV_STAGE);
                    for (int c = 0; c < C::NCH; ++c)
                        tma_load_2d(sv + vs * C::KV_STAGE + c * C::BOX, &vmap, &v_full[vs], kvh * D + c * 64, row);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t kIdescS = idesc_bf16_f32(128, C::BN);
        constexpr uint32_t kIdescO = idesc_bf16_f32(128, D) | (1u << 16);  // B (V) MN-major
        const uint64_t q_base = smem_desc_sw128(smem_u32(sq));
        const uint64_t k_base = smem_desc_sw128(smem_u32(sk));
        const uint64_t v_base = smem_desc_sw128_mn(smem_u32(sv), C::BOX, 1024);
        auto issue_s = [&](int t, uint32_t kvi) {  // S_t = Q_t K^T from ring slot kvi
            const uint32_t ks = kvi % C::KST;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t off = ((kk >> 2) * C::BOX + (kk & 3) * 32) >> 4;
                mma_bf16_ss(tmem + C::S_COL + t * C::BN, q_base + ((t * C::Q_BYTES) >> 4) + off,
                            k_base + ((ks * C::KV_STAGE) >> 4) + off, kIdescS, kk > 0 ? 1u : 0u);
            }
            mma_commit(&s_full[t]);
        };
        // O_t += P_t V (P over S_t), one 64-key half at a time: the half's MMAs go out as
        // soon as the softmax has stored that half of P
        auto issue_pv = [&](int t, uint32_t kvi, bool first, uint32_t ph) {
            const uint32_t vs = kvi % C::VST;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                mbar_wait(&p_full[t * 2 + hf], ph);
                tc_fence_after();
#pragma unroll
                for (int kk = hf * (C::BN / 32); kk < (hf + 1) * (C::BN / 32); ++kk)  // 16 keys = 8 P columns
                    mma_bf16_ts(tmem + C::O_COL + t * D, tmem + C::S_COL + t * C::BN + kk * 8,
                                v_base + ((vs * C::KV_STAGE + kk * 2048) >> 4), kIdescO,
                                (!first || kk > 0) ? 1u : 0u);
            }
        };
        uint32_t kv = 0, js = 0;  // K/V ring position, S/P phases (tiles so far, per query tile)
        for (int it = 0;; ++it) {
            const PairPlan pl = take_plan(it);
            if (pl.nt < 0) break;
            const int nt = pl.nt;
            if (lane == 0) {
                mbar_wait(q_full, it & 1);
                mbar_wait(&k_full[kv % C::KST], (kv / C::KST) & 1);
                tc_fence_after();
                issue_s(0, kv);
                issue_s(1, kv);
                if (nt == 1) mma_commit(q_empty);
                mma_commit(&k_empty[kv % C::KST]);
                for (int j = 0; j < nt; ++j) {
                    const uint32_t kj = kv + j;
                    const bool more = j + 1 < nt;
                    mbar_wait(&v_full[kj % C::VST], (kj / C::VST) & 1);
                    issue_pv(0, kj, j == 0, (js + j) & 1);
                    if (!more) mma_commit(&o_done[0]);
                    if (more) {
                        mbar_wait(&k_full[(kj + 1) % C::KST], ((kj + 1) / C::KST) & 1);
                        tc_fence_after();
                        issue_s(0, kj + 1);
                    }
                    issue_pv(1, kj, j == 0, (js + j) & 1);
                    mma_commit(&v_empty[kj % C::VST]);
                    if (!more) mma_commit(&o_done[1]);
                    if (more) {
                        issue_s(1, kj + 1);
                        if (j + 2 == nt) mma_commit(q_empty);  // the item's last S MMAs
                        mma_commit(&k_empty[(kj + 1) % C::KST]);
                    }
                }
            }
            kv += nt;
            js += nt;
        }
    } else if (warp == 2) {
        // scheduler: items are handed out dynamically (global counter in the workspace's
        // error region, bytes [128, 136), returned to 0 by the last CTA), planned one
        // ahead of the consumers
        if (lane == 0) {
            uint32_t* ctr = p.err + 32;
            const bool bad = p.cu_seqlens[p.num_requests] > p.max_tokens;  // malformed: no items
            if (bad && blockIdx.x == 0) raise_error(p.err, kErrBadSeqlens);
            const int total = bad ? 0 : total_pairs(p);
            const int items = total * H;
            for (int it = 0;; ++it) {
                const int slot = it % C::PLANS;
                if (it >= C::PLANS) mbar_wait(&plan_empty[slot], ((it / C::PLANS) - 1) & 1);
                const int item = static_cast<int>(atomicAdd(ctr, 1u));
                PairPlan pl{0, 0, 0, 0, -1, 0};
                if (item < items) {
                    pl = pair_plan(p, item / H, total);
                    pl.h = item % H;
                }
                plans[slot] = pl;
                mbar_arrive(&plan_full[slot]);
                if (item >= items) break;
            }
            __threadfence();
            if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every CTA has taken its last item
                atomicExch(ctr, 0u);
                atomicExch(ctr + 1, 0u);
            }
        }
    } else if (warp >= 4) {
        const int t = (warp - 4) >> 2;       // query tile of this warpgroup
        const int quarter = warp & 3;        // TMEM lane quarter
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t s_addr = tmem + lane_base + C::S_COL + t * C::BN;
        const uint32_t o_addr = tmem + lane_base + C::O_COL + t * D;
        const float c = p.scale_log2;
        const int64_t total_rows = p.cu_seqlens[p.num_requests];
        uint32_t js = 0;
        for (int it = 0;; ++it) {
            const PairPlan pl = take_plan(it);
            if (pl.nt < 0) break;
            const int h = pl.h;
            const int nt = pl.nt;
            const int64_t qi = pl.q0 + t * C::BM + r;
            const bool valid = qi < pl.seg_end;
            int64_t lo = 0, hi = 0;
            if (valid) {
                if (p.window > 0) {
                    const int64_t qp = p.positions[qi];
                    hi = upper_pos(p.positions, pl.seg_begin, pl.seg_end, qp);
                    lo = lower_pos(p.positions, pl.seg_begin, pl.seg_end, qp - p.window + 1);
                } else {  // strictly increasing positions: keys [seg_begin, qi]
                    hi = qi + 1;
                    lo = pl.seg_begin;
                }
                if (lo >= hi) raise_error(p.err, kErrNoVisibleKey);
            }
            float m_run = -INFINITY, l_run = 0.f;
            for (int j = 0; j < nt; ++j) {
                const int64_t kb = pl.k_begin + static_cast<int64_t>(j) * C::BN;
                const int vis0 = static_cast<int>(lo - kb < 0 ? 0 : (lo - kb > C::BN ? C::BN : lo - kb));
                const int vis1 = static_cast<int>(hi - kb < 0 ? 0 : (hi - kb > C::BN ? C::BN : hi - kb));
                // warp-uniform: the P stores below are tcgen05.st (.sync.aligned)
                const bool full = __all_sync(0xffffffffu, vis0 == 0 && vis1 == C::BN);
                mbar_wait(&s_full[t], (js + j) & 1);
                tc_fence_after();
                // two passes over S_t in 64-column halves (keeps the row out of registers:
                // the 384-thread CTA has 168 registers per thread): max, then exp2 -> P.
                // P half hf lands in columns [32hf, 32hf+32), which only half 0 occupies and
                // which is already in registers when it is overwritten.
                constexpr int HALF = 64;
                float mx = -INFINITY;
#pragma unroll
                for (int hf = 0; hf < C::BN / HALF; ++hf) {
                    uint32_t s[HALF];
#pragma unroll
                    for (int q = 0; q < HALF / 32; ++q)
                        tmem_ld32(s_addr + hf * HALF + q * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[q * 32]));
                    tmem_ld_wait();
                    if (full) {
                        float a[4] = {mx, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                        for (int i = 0; i < HALF; i += 8)
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                a[u] = fmax3(a[u], __uint_as_float(s[i + 2 * u]), __uint_as_float(s[i + 2 * u + 1]));
                        mx = fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
                    } else {
#pragma unroll
                        for (int i = 0; i < HALF; ++i) {
                            const int e = hf * HALF + i;
                            if (e >= vis0 && e < vis1) mx = fmaxf(mx, __uint_as_float(s[i]));
                        }
                    }
                }
                mx *= c;
                // lazy rescale (reference moves only when the row max grows by > 2^8).  O_t
                // is idle here: PV_t,j-1 completed before S_t,j (issue order) signalled.
                const bool grow = mx > m_run + 8.f;
                float alpha = 1.f;
                if (grow) {
                    alpha = m_run == -INFINITY ? 0.f : ex2_approx(m_run - mx);
                    l_run *= alpha;
                    m_run = mx;
                }
                if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
                    for (int q = 0; q < D / 32; ++q) {
                        uint32_t o[32];
                        tmem_ld32(o_addr + q * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                        tmem_st32(o_addr + q * 32, o);
                    }
                }
                const float mref = m_run == -INFINITY ? 0.f : m_run;
                if (t == 0 && kb + C::BN > total_rows) {  // V rows past the batch -> 0 before PV0 reads them
                    const uint32_t g = js + j;
                    mbar_wait(&v_full[g % C::VST], (g / C::VST) & 1);
                    zero_stage_rows(sv + (g % C::VST) * C::KV_STAGE, C::NCH, C::BOX,
                                    static_cast<int>(total_rows - kb > 0 ? total_rows - kb : 0), C::BN,
                                    threadIdx.x - 128, 128);
                    fence_proxy_async_smem();
                }
                float lsum = 0.f;
                const uint64_t c2 = pk(c, c), m2 = pk(-mref, -mref);
                uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
                for (int hf = 0; hf < C::BN / HALF; ++hf) {
                    uint32_t s[HALF];
#pragma unroll
                    for (int q = 0; q < HALF / 32; ++q)
                        tmem_ld32(s_addr + hf * HALF + q * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[q * 32]));
                    tmem_ld_wait();
#pragma unroll
                    for (int q = 0; q < HALF / 32; ++q) {
                        uint32_t pk16[16];
                        if (full) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                const int e0 = q * 32 + 2 * i;
                                const uint64_t x = fma2(
                                    static_cast<uint64_t>(s[e0]) | (static_cast<uint64_t>(s[e0 + 1]) << 32), c2, m2);
                                const uint64_t e = i < 16 - kAttnPolyPairs<D>
                                                       ? pk(ex2_approx(lo_f(x)), ex2_approx(hi_f(x)))
                                                       : exp2_poly2(x);
                                if (i & 1) acc1 = add2(acc1, e);
                                else acc0 = add2(acc0, e);
                                pk16[i] = pack_bf16(lo_f(e), hi_f(e));
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < 16; ++i) {
                                const int e0 = hf * HALF + q * 32 + 2 * i, e1 = e0 + 1;
                                float p0 = ex2_approx(fmaf(__uint_as_float(s[q * 32 + 2 * i]), c, -mref));
                                float p1 = ex2_approx(fmaf(__uint_as_float(s[q * 32 + 2 * i + 1]), c, -mref));
                                if (e0 < vis0 || e0 >= vis1) p0 = 0.f;
                                if (e1 < vis0 || e1 >= vis1) p1 = 0.f;
                                lsum += p0 + p1;
                                pk16[i] = pack_bf16(p0, p1);
                            }
                        }
                        tmem_st16(s_addr + hf * 32 + q * 16, pk16);
                    }
                    // this half of P is in TMEM: its PV MMAs may start
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&p_full[t * 2 + hf]);
                }
                {
                    const uint64_t a2 = add2(acc0, acc1);
                    lsum += lo_f(a2) + hi_f(a2);
                }
                l_run += lsum;

            }
            // epilogue: O_t / l -> bf16.  The next item's PV_t,0 (which overwrites O_t) is
            // issued only after this warpgroup's next p_full arrival, i.e. after these loads.
            mbar_wait(&o_done[t], it & 1);
            tc_fence_after();
            const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
            __nv_bfloat16* orow = p.out + qi * p.out_row_stride + static_cast<int64_t>(h) * D;
#pragma unroll
            for (int q = 0; q < D / 32; ++q) {
                uint32_t o[32];
                tmem_ld32(o_addr + q * 32, o);
                tmem_ld_wait();
                if (valid) {
                    uint4 w[4];
                    uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        wp[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
                    uint4* dst = reinterpret_cast<uint4*>(orow + q * 32);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = w[i];
                }
            }
            tc_fence_before();
            js += nt;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int D>
static cudaError_t launch_attn2q(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                                 const AttnParams& p, int grid, cudaStream_t stream) {
    using C = Attn2Cfg<D>;
    const int smem = C::smem();
    cudaError_t e = cudaFuncSetAttribute(attention2q_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_k(0, attention2q_kernel<D>, grid, C::THREADS, smem, stream, qm, km, vm, p);
}

template <int D>
static cudaError_t launch_attn(const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                               const AttnParams& p, int grid, cudaStream_t stream) {
    using C = AttnCfg<D>;
    const int smem = C::smem();
    cudaError_t e = cudaFuncSetAttribute(attention_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_k(0, attention_kernel<D>, grid, C::THREADS, smem, stream, qm, km, vm, p);
}

int attention_kv_box_rows(int D) { return D > 128 ? AttnCfg<256>::BN : AttnCfg<128>::BN; }

bool attention_supported(int D) { return D == 64 || D == 128 || D == 256; }

// query rows per CTA: 256 (two tiles) for D <= 128, 128 for D = 256
int attention_rows_per_cta(int D) { return D > 128 ? 128 : 256; }

cudaError_t launch_attention(int D, const CUtensorMap& qm, const CUtensorMap& km, const CUtensorMap& vm,
                             const AttnParams& p, int grid, cudaStream_t stream) {
    if (D == 64) return launch_attn2q<64>(qm, km, vm, p, grid, stream);
    if (D == 128) return launch_attn2q<128>(qm, km, vm, p, grid, stream);
    if (D == 256) return launch_attn<256>(qm, km, vm, p, grid, stream);
    return cudaErrorInvalidValue;
}

}  // namespace up
