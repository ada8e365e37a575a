// select.cu -- per-request top-p keep mask (sm_100a), bit-exact with the reference.
//
// One CTA per request (selection.cpp:51-122):
//   1. validate block scores (finite, >= 0; :61-66) and total them (double);
//   2. zero mass -> keep-all with the degenerate flag (:73-76);
//   3. pack (phi(s) << 32 | ~g, :27-34) and bitonic-sort the words descending in shared
//      memory (ties: lower block index first);
//   4. parallel double prefix sum of the decoded scores in sorted order, k* = first rank
//      with cum / total >= double(p) (:80-93).  The reference sums sequentially; a
//      parallel sum agrees with it to a few ulps, so the decision is taken in parallel
//      only when every ratio near the crossing clears p by a proven error margin;
//      otherwise one thread replays the reference's exact sequential sums (bit-exact by
//      construction: same IEEE double adds in the same order, correctly rounded division);
//   5. expand blocks to tokens, force sinks (i < A) and the query window (i >= N - n_eff)
//      (expand_mask, :36-49), apply the optional no-readmission veto (restrict_selection,
//      propagation.cpp:116-136) and compute retained count and covered mass (:108-120).
#include <cstdlib>
#include <float.h>

#include <cub/block/block_radix_sort.cuh>

#include "params.cuh"

namespace up {

constexpr int kSelThreads = 512;
#ifndef UP_SELECT_RADIX_BITS
#define UP_SELECT_RADIX_BITS 4  // bits per radix-sort pass
#endif

__device__ __forceinline__ uint32_t phi_encode_dev(float x) {
    if (x == 0.0f) x = 0.0f;  // -0 -> +0
    const uint32_t bits = __float_as_uint(x);
    return x >= 0.0f ? (bits ^ 0x80000000u) : (bits ^ 0xFFFFFFFFu);
}

__device__ __forceinline__ float phi_decode_dev(uint32_t bits) {
    return __uint_as_float((bits & 0x80000000u) ? (bits ^ 0x80000000u) : (bits ^ 0xFFFFFFFFu));
}

__device__ __forceinline__ float key_score(uint64_t w) {
    return phi_decode_dev(static_cast<uint32_t>(w >> 32));
}

template <typename T>
__device__ T block_sum(T v, T* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    T t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? scratch[threadIdx.x] : T(0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) scratch[0] = t;
    }
    __syncthreads();
    t = scratch[0];
    __syncthreads();
    return t;
}

// Exclusive prefix sum of one double per thread across the CTA.
__device__ double block_exclusive_scan(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = threadIdx.x < (blockDim.x >> 5) ? scratch[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        scratch[threadIdx.x] = w;  // inclusive warp totals
    }
    __syncthreads();
    const double warp_base = warp > 0 ? scratch[warp - 1] : 0.0;
    const double r = warp_base + x - v;
    __syncthreads();
    return r;
}

#define SEL_STAMP(k)                                                      \
    if (p.dbg != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {       \
        unsigned long long c_;                                            \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_));                \
        p.dbg[k] = c_;                                                    \
    }

// expand_mask (selection.cpp:36-49) of one request by its own select CTA, for small
// capacities (kSmallExpandTokens) where the grid-wide expand_kernel's launch costs more than
// the CTA's N_r byte stores.  Same decisions as expand_kernel; reads the block decisions this
// CTA just published (the caller synchronises the CTA first).
constexpr int64_t kSmallExpandTokens = 8192;

// blk: the CTA's block decisions in shared memory, or null = every block kept.
__device__ void expand_request(const SelectParams& p, int seg0, int N, int neff, bool enabled, const uint8_t* blk) {
    const int64_t A = p.sink_count_a;
    const int G = p.block_size_g;
    uint8_t* keep = p.keep + seg0;
    // 16 tokens per thread step with one 16-byte store; the unaligned head and the tail bytewise
    const int head = min(N, static_cast<int>((16 - (reinterpret_cast<uintptr_t>(keep) & 15)) & 15));
    auto tok = [&](int li) -> uint32_t {
        if (!enabled) return 1u;
        uint32_t k = (blk == nullptr || blk[li / G] != 0 || li < A || li >= N - neff) ? 1u : 0u;
        if (k && p.veto != nullptr && p.veto[seg0 + li]) k = 0u;
        return k;
    };
    for (int li = threadIdx.x; li < head; li += blockDim.x) keep[li] = static_cast<uint8_t>(tok(li));
    const int nvec = (N - head) >> 4;
    const int64_t win0 = N - neff;
    const int nbk = (N + G - 1) / G;
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
        const int l0 = head + 16 * v;
        uint32_t w[4];
        if (enabled && G >= 16 && p.veto == nullptr) {
            // 16 tokens touch at most two blocks: two decisions instead of 16 divisions
            const int b0 = l0 / G;
            const int edge = (b0 + 1) * G;
            const uint32_t k0 = blk == nullptr || blk[b0] != 0;
            const uint32_t k1 = blk == nullptr || blk[min(b0 + 1, nbk - 1)] != 0;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                uint32_t word = 0;
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    const int li = l0 + 4 * x + y;
                    const uint32_t k = (li < edge ? k0 : k1) | (li < A ? 1u : 0u) | (li >= win0 ? 1u : 0u);
                    word |= k << (8 * y);
                }
                w[x] = word;
            }
        } else {
#pragma unroll
            for (int x = 0; x < 4; ++x)
                w[x] = tok(l0 + 4 * x) | (tok(l0 + 4 * x + 1) << 8) | (tok(l0 + 4 * x + 2) << 16) | (tok(l0 + 4 * x + 3) << 24);
        }
        *reinterpret_cast<uint4*>(keep + l0) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    for (int li = head + 16 * nvec + threadIdx.x; li < N; li += blockDim.x) keep[li] = static_cast<uint8_t>(tok(li));
}

// Per-request epilogue shared by both select kernels: blk[] (smem) holds the block
// decisions and sc[] the block scores.  Publishes the decisions for the expand kernel and
// computes retained count / covered mass (selection.cpp:98-120): analytically per block
// without a veto (a block keeps all tokens, or only the forced sinks [0, A) and query
// window [N - n_eff, N)), per token with the veto (restrict_selection,
// propagation.cpp:116-136).
__device__ void finish_request(const SelectParams& p, int r, int seg0, int N, int nb, int neff,
                               const uint8_t* blk, const float* sc, int kstar, bool degenerate,
                               double total, double* red_d, int* red_i) {
    const int tid = threadIdx.x;
    const int G = p.block_size_g;
    const int64_t A = p.sink_count_a;
    const int64_t win0 = N - neff;
    uint8_t* out_blk = p.blk_keep + p.cu_blocks[r];
    int retained = 0;
    double covered = 0.0;
    for (int g = tid; g < nb; g += blockDim.x) {
        out_blk[g] = blk[g];
        const int64_t b0 = static_cast<int64_t>(g) * G;
        const int size = min(G, N - g * G);
        int kept;
        if (p.veto == nullptr) {
            kept = size;
            if (!blk[g]) {
                const int64_t b1 = b0 + size;
                const int64_t sink_end = b1 < A ? b1 : A;
                const int64_t win_beg = b0 > win0 ? b0 : win0;
                const int64_t sink = sink_end > b0 ? sink_end - b0 : 0;
                const int64_t win = b1 > win_beg ? b1 - win_beg : 0;
                const int64_t both = sink_end > win_beg ? sink_end - win_beg : 0;
                kept = static_cast<int>(sink + win - both);
            }
        } else {
            kept = 0;
            for (int x = 0; x < size; ++x) {
                const int64_t i = b0 + x;
                const bool k = (blk[g] != 0 || i < A || i >= win0) && !p.veto[seg0 + i];
                kept += k ? 1 : 0;
            }
        }
        retained += kept;
        // covered_mass attribution (selection.cpp:108-120): s_g * kept_g / |g| -- the ratio
        // is exactly 1 or 0 for whole blocks, so only partially kept blocks divide
        const double frac = kept == size ? 1.0 : (kept == 0 ? 0.0 : static_cast<double>(kept) / static_cast<double>(size));
        covered += static_cast<double>(sc[g]) * frac;
    }
    SEL_STAMP(6)
    if (p.fuse_expand) expand_request(p, seg0, N, neff, true, blk);  // blk: complete in smem (caller synced)
    SEL_STAMP(7)
    retained = block_sum<int>(retained, red_i);
    covered = block_sum<double>(covered, red_d);
    SEL_STAMP(8)
    if (tid == 0) {
        p.cutoff_rank[r] = kstar;
        if (p.retained_count) p.retained_count[r] = retained;
        // Degenerate selections report 1.0 with or without a veto (selection.cpp:104-106,
        // propagation.cpp:135: restrict_selection also falls back to 1.0 at zero mass).
        if (p.covered_mass) p.covered_mass[r] = degenerate ? 1.0 : covered / total;
        if (p.degenerate) p.degenerate[r] = degenerate ? 1 : 0;
    }
}

// Error / pass-through requests: every block kept, stats of a keep-all selection.
__device__ void keep_all_request(const SelectParams& p, int r, int N, int nb, int64_t cutoff) {
    uint8_t* out_blk = p.blk_keep + p.cu_blocks[r];
    for (int g = threadIdx.x; g < nb; g += blockDim.x) out_blk[g] = 1;
    if (threadIdx.x == 0) {
        p.cutoff_rank[r] = cutoff;
        if (p.retained_count) p.retained_count[r] = N;
        if (p.covered_mass) p.covered_mass[r] = 1.0;
        if (p.degenerate) p.degenerate[r] = 0;
    }
    if (p.fuse_expand) {
        __syncthreads();
        const int seg0 = p.cu_seqlens[r];
        const bool enabled = p.drop_enabled == nullptr || p.drop_enabled[r] != 0;
        expand_request(p, seg0, N, min(p.query_window_n, N), enabled, nullptr);
    }
}

// The reference's exact sequential sums (selection.cpp:61-67, :84-93) replayed by one
// thread over the sorted order; returns k*.  Bit-exact by construction.
// KeyAt: rank q -> phi key of the q-th largest block.
template <class KeyAt>
__device__ int exact_crossing_t(const float* sc, int nb, KeyAt key_at, double p_d) {
    // Both loops are serial dependency chains of double adds; the loads and float->double
    // conversions of 8 terms are issued ahead of the adds, so only the add latency remains.
    constexpr int U = 8;
    double tot = 0.0;
    int g = 0;
    for (; g + U <= nb; g += U) {
        double x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = static_cast<double>(sc[g + u]);
#pragma unroll
        for (int u = 0; u < U; ++u) tot += x[u];
    }
    for (; g < nb; ++g) tot += sc[g];
    // Below lo the reference's test fl(c / tot) >= p is false for certain (c / tot < p by a
    // relative 1e-12, far above the rounding of either side), so the double division only
    // runs near the crossing.
    const double lo = p_d * tot * (1.0 - 1e-12);
    double c = 0.0;
    int q = 0;
    for (; q + U <= nb; q += U) {
        double x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = static_cast<double>(phi_decode_dev(key_at(q + u)));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c += x[u];
            if (c >= lo && c / tot >= p_d) return q + u + 1;
        }
    }
    for (; q < nb; ++q) {
        c += static_cast<double>(phi_decode_dev(key_at(q)));
        if (c >= lo && c / tot >= p_d) return q + 1;
    }
    return nb;
}

__device__ int exact_crossing(const float* sc, int nb, const uint32_t* skey, double p_d) {
    return exact_crossing_t(sc, nb, [skey](int q) { return skey[q]; }, p_d);
}


// Guard (see file header): the sequential ratio is monotone in the rank and within delta
// of the parallel one; accept the parallel crossing only when it clears p by delta.
__device__ __forceinline__ bool crossing_certain(bool reached, int rc, double ratio_c, double ratio_prev,
                                                 double p_d, int nb) {
    const double delta = (4.0 * nb + 256.0) * DBL_EPSILON;
    bool certain = reached ? (ratio_c - p_d > delta) : (p_d - ratio_c > delta);
    if (reached && rc >= 1) certain = certain && (p_d - ratio_prev > delta);
    return certain;
}

// The radix select serves the small class (<= 512 blocks per request, 128 threads): LLaMA
// 1x4K 11.8 -> 11.1 us, 4 x 2 blocks 8.2 -> 5.7 us, 4 x 512 blocks even (13.4 / 13.6).  In
// the 512-thread class (<= 2048 blocks) the CUB sort stays: there the select measured slower
// (1 x 2048 blocks 19.0 vs 20.0 us, the 64-request stream 36.3 vs 41.0 us).
// -DUP_SELECT_ALWAYS_SORT: always sort (A/B timing).
// Requests of <= kSelBruteBlocks blocks (C1: 64) rank every block directly (2o in
// select_radix_kernel).  -DUP_SELECT_BRUTE=0: radix select for them too (A/B).
constexpr int kSelBruteBlocks = 128;
#ifndef UP_SELECT_BRUTE
#define UP_SELECT_BRUTE 1
#endif
#ifndef UP_SELECT_RADIX_MAX_THREADS
#define UP_SELECT_RADIX_MAX_THREADS 128
#endif
template <int THREADS>
__device__ __forceinline__ bool use_radix_select() {
#ifdef UP_SELECT_ALWAYS_SORT
    return false;
#else
    return THREADS <= UP_SELECT_RADIX_MAX_THREADS;
#endif
}

// ---- radix select of the crossing rank (no sort) ------------------------------------
// The sorted order is needed only up to the crossing: k* = count(keys > K*) + t, where K*
// is the key of rank k* and t its rank inside the tie group of equal keys (ascending block
// index, PackedScore's ~g).  K* is found MSB-first, 4 bits at a time, below the prefix all
// keys share (block AND / OR): per level every thread bins its candidate keys into 16
// register buckets (count, double mass), a warp reduce-scatter and a fixed-order sum over
// the warps give the level's histogram -- no atomics, so clustered scores (many keys in one
// bucket) cost nothing extra, and the sums are deterministic -- and one warp scans the 16
// buckets descending for the one where the mass above plus the bucket's reaches p * total.
// Ends early when the bucket holds one key.  The masses are summed in another order than
// the reference's sequential sum, so the result is accepted under the same error guard as
// the parallel scan (crossing_certain); otherwise the caller sorts and replays exactly.
struct RadixSel {
    double wmass[32][16];  // per-warp bucket masses of the level
    int wcnt[32][16];
    uint32_t and_all[32], or_all[32];
    uint32_t key;
    int bucket;            // crossing digit of the level, -1 = p never reached
    int bcount;            // keys in the crossing bucket
    int cabove;            // keys strictly above the bucket
    double above;          // their mass
    double all;            // mass of every candidate at the first level
};

// Sum of 16 per-lane values across the warp: lane l ends with bucket (l >> 1) & 15.
template <typename T>
__device__ __forceinline__ T warp_reduce_scatter16(T (&v)[16]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // 16 -> 8 values (lane bit 4 picks the half kept)
        const bool hi = lane & 16;
        const T send = hi ? v[j] : v[j + 8];
        const T keep = hi ? v[j + 8] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // 8 -> 4 (bit 3)
        const bool hi = lane & 8;
        const T send = hi ? v[j] : v[j + 4];
        const T keep = hi ? v[j + 4] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // 4 -> 2 (bit 2)
        const bool hi = lane & 4;
        const T send = hi ? v[j] : v[j + 2];
        const T keep = hi ? v[j + 2] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    {  // 2 -> 1 (bit 1)
        const bool hi = lane & 2;
        const T send = hi ? v[0] : v[1];
        const T keep = hi ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

template <int THREADS, int ITEMS>
__device__ bool radix_crossing(const uint32_t (&key)[ITEMS], const float (&dec)[ITEMS], double total,
                               double p_d, int nb, RadixSel& rs, int& kstar, uint32_t& kkey, int& tkeep) {
    constexpr int WARPS = THREADS / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double target = p_d * total;
    // common prefix of every valid key (key 0 = padding)
    uint32_t a = 0xFFFFFFFFu, o = 0u;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
        if (key[i] != 0u) { a &= key[i]; o |= key[i]; }
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) {
        a &= __shfl_xor_sync(0xffffffffu, a, x);
        o |= __shfl_xor_sync(0xffffffffu, o, x);
    }
    if (lane == 0) { rs.and_all[warp] = a; rs.or_all[warp] = o; }
    __syncthreads();
    a = 0xFFFFFFFFu;
    o = 0u;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) { a &= rs.and_all[w]; o |= rs.or_all[w]; }
    const uint32_t diff = a ^ o;
    int shift = diff == 0u ? 0 : 32 - __clz(diff);  // bits [0, shift) still undecided
    uint32_t pmask = shift == 32 ? 0u : ~((1u << shift) - 1u);
    uint32_t prefix = a & pmask;
    double above = 0.0;
    int cabove = 0;
    int bcount = nb;     // all keys equal (shift = 0): one tie group
    bool first = true;
#pragma unroll 1
    while (shift > 0) {
        const int dshift = shift > 4 ? shift - 4 : 0;
        const uint32_t dmask = (1u << (shift - dshift)) - 1u;
        double m[16];
        int c[16];
#pragma unroll
        for (int b = 0; b < 16; ++b) { m[b] = 0.0; c[b] = 0; }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const bool cand = key[i] != 0u && (key[i] & pmask) == prefix;
            const uint32_t d = (key[i] >> dshift) & dmask;
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                const bool hit = cand && d == static_cast<uint32_t>(b);
                m[b] += hit ? static_cast<double>(dec[i]) : 0.0;
                c[b] += hit ? 1 : 0;
            }
        }
        const double ms = warp_reduce_scatter16<double>(m);
        const int cs = warp_reduce_scatter16<int>(c);
        if ((lane & 1) == 0) { rs.wmass[warp][lane >> 1] = ms; rs.wcnt[warp][lane >> 1] = cs; }
        __syncthreads();
        if (tid < 32) {
            // lane l < 16 owns digit 15 - l (descending); fixed-order sum over the warps
            double bm = 0.0;
            int bc = 0;
            if (lane < 16) {
#pragma unroll 4
                for (int w = 0; w < WARPS; ++w) { bm += rs.wmass[w][15 - lane]; bc += rs.wcnt[w][15 - lane]; }
            }
            double mi = bm;
            int ci = bc;
#pragma unroll
            for (int x = 1; x < 16; x <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, mi, x);
                const int z = __shfl_up_sync(0xffffffffu, ci, x);
                if (lane >= x) { mi += y; ci += z; }
            }
            const unsigned hits = __ballot_sync(0xffffffffu, lane < 16 && above + mi >= target);
            if (first && lane == 15) rs.all = mi;  // every candidate: the whole mass
            if (hits == 0u) {
                if (lane == 0) rs.bucket = -1;
            } else if (lane == __ffs(hits) - 1) {
                rs.bucket = 15 - lane;
                rs.bcount = bc;
                rs.cabove = cabove + ci - bc;
                rs.above = above + mi - bm;
            }
        }
        __syncthreads();
        const int b = rs.bucket;
        if (b < 0) {  // the whole mass stays below p * total (within rounding): not reached
            if (!first) return false;  // rounding disagreed with the level above: sort
            bcount = 0;
            break;
        }
        above = rs.above;
        cabove = rs.cabove;
        bcount = rs.bcount;
        prefix |= static_cast<uint32_t>(b) << dshift;
        pmask |= dmask << dshift;
        shift = dshift;
        first = false;
        if (bcount == 1 && shift > 0) {  // one key left: it is K*
            __syncthreads();
#pragma unroll
            for (int i = 0; i < ITEMS; ++i)
                if (key[i] != 0u && (key[i] & pmask) == prefix) rs.key = key[i];
            __syncthreads();
            prefix = rs.key;
            shift = 0;
        }
        __syncthreads();  // rs.* read by every thread before the next level rewrites it
    }
    const bool reached = bcount > 0;
    double ratio_c, ratio_prev = -1.0;
    int rc;
    if (reached) {
        const double sv = static_cast<double>(phi_decode_dev(prefix));
        if (!(sv > 0.0)) return false;  // zero-mass crossing: only rounding can get here
        // smallest t in [1, bcount] with above + t * s >= target (t * s is exact in double)
        const double tt = ceil((target - above) / sv);
        const int t = tt < 1.0 ? 1 : (tt > static_cast<double>(bcount) ? bcount : static_cast<int>(tt));
        kstar = cabove + t;
        kkey = prefix;
        tkeep = t;
        rc = kstar - 1;
        ratio_c = (above + static_cast<double>(t) * sv) / total;
        ratio_prev = (above + static_cast<double>(t - 1) * sv) / total;
    } else {
        kstar = nb;
        kkey = 0u;  // every valid key is above
        tkeep = 0;
        rc = nb - 1;
        ratio_c = rs.all / total;
    }
    return crossing_certain(reached, rc, ratio_c, ratio_prev, p_d, nb);
}

// ---- CUB radix-sort variant (nb <= THREADS * ITEMS) ---------------------------------
template <int THREADS, int ITEMS, bool RADIX = (THREADS <= UP_SELECT_RADIX_MAX_THREADS)>
__global__ void __launch_bounds__(THREADS)
select_radix_kernel(const SelectParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    if (!cta_batch_valid(p.cu_seqlens, gridDim.x, p.max_tokens)) {  // malformed batch (grid = R)
        if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(p.err, kErrBadSeqlens);
        return;
    }
    using Sort = cub::BlockRadixSort<uint32_t, THREADS, ITEMS, int32_t, UP_SELECT_RADIX_BITS>;
    constexpr int CAP = THREADS * ITEMS;
    __shared__ union {
        RadixSel sel;
        typename Sort::TempStorage sort;
        struct { uint32_t key[CAP]; int32_t val[CAP]; } sorted;  // fallback replay only
    } u;
    __shared__ float sc[CAP];
    __shared__ uint8_t blk[CAP];
    __shared__ double red_d[32];
    __shared__ int red_i[32];
    __shared__ int s_kstar;
    __shared__ double s_ratio[2];

    const int r = blockIdx.x;
    SEL_STAMP(0)
    const int tid = threadIdx.x;
    const int seg0 = p.cu_seqlens[r];
    const int N = p.cu_seqlens[r + 1] - seg0;
    const int G = p.block_size_g;
    const int nb = (N + G - 1) / G;
    if (nb <= p.nb_lo || nb > p.nb_hi) return;  // another size class's launch owns it
    const int neff = min(p.query_window_n, N);
    const bool enabled = p.drop_enabled == nullptr || p.drop_enabled[r] != 0;
    if (!enabled) { keep_all_request(p, r, N, nb, -1); return; }
    if (nb > CAP) {
        if (tid == 0) raise_error(p.err, kErrTooManyBlocks);
        keep_all_request(p, r, N, nb, -1);
        return;
    }
    const float* bs = p.block_scores + p.cu_blocks[r];

    // 1. validate, total, keys (blocked: thread t owns blocks t*ITEMS .. +ITEMS-1).
    uint32_t key[ITEMS];
    int32_t val[ITEMS];
    bool bad = false;
    double tsum = 0.0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int g = tid * ITEMS + i;
        if (g < nb) {
            const float s = bs[g];
            if (!(s >= 0.0f) || !isfinite(s)) bad = true;
            sc[g] = s;
            tsum += s;
            key[i] = phi_encode_dev(s);  // >= 0x80000000 for every valid score
            val[i] = g;
        } else {
            key[i] = 0;                   // padding sorts last
            val[i] = -1;
        }
    }
    bad = __syncthreads_or(bad);
    if (bad) {
        if (tid == 0) raise_error(p.err, kErrBadScore);
        keep_all_request(p, r, N, nb, -1);
        return;
    }
    const double total = block_sum<double>(tsum, red_d);
    const bool degenerate = !(total > 0.0);
    int kstar = nb;
    if (degenerate) {
        for (int g = tid; g < nb; g += THREADS) blk[g] = 1;
    } else {
        SEL_STAMP(1)
        const double p_d = static_cast<double>(p.top_p);
        // 2o. <= 128 blocks: every block's rank in the sorted order (descending phi, ties by
        //     ascending block index) and its inclusive mass by a pass over all blocks -- one
        //     block per thread, no sort, no histogram levels -- under the same
        //     crossing_certain guard (the masses are summed in block order).
        if (RADIX && use_radix_select<128>() && nb <= kSelBruteBlocks && THREADS >= kSelBruteBlocks && UP_SELECT_BRUTE) {
            uint32_t* s_key = reinterpret_cast<uint32_t*>(&u.sel);
#pragma unroll
            for (int i = 0; i < ITEMS; ++i)
                if (val[i] >= 0) s_key[val[i]] = key[i];
            if (tid == 0) { s_kstar = nb + 1; s_ratio[0] = -1.0; s_ratio[1] = -1.0; }
            __syncthreads();
            int rank = 0;
            double cum = 0.0;
            if (tid < nb) {
                const uint32_t kg = s_key[tid];
                for (int j = 0; j < nb; ++j) {
                    const uint32_t kj = s_key[j];
                    const bool before = kj > kg || (kj == kg && j < tid);
                    rank += before ? 1 : 0;
                    if (before || j == tid) cum += static_cast<double>(sc[j]);
                }
                if (cum / total >= p_d) atomicMin(&s_kstar, rank + 1);
            }
            __syncthreads();
            const int kpar = s_kstar;
            const bool reached = kpar <= nb;
            const int rc = reached ? kpar - 1 : nb - 1;
            if (tid < nb && rank == rc) s_ratio[0] = cum / total;
            if (tid < nb && rank == rc - 1) s_ratio[1] = cum / total;
            __syncthreads();
            if (crossing_certain(reached, rc, s_ratio[0], s_ratio[1], p_d, nb)) {
                if (tid < nb) blk[tid] = rank < kpar ? 1 : 0;
                __syncthreads();
                SEL_STAMP(4)
                finish_request(p, r, seg0, N, nb, neff, blk, sc, kpar, degenerate, total, red_d, red_i);
                SEL_STAMP(5)
                return;
            }
            __syncthreads();  // s_key (u) is reused below
        }
        // 2a. radix select of the crossing key K* and its rank t inside the tie group
        float dsc[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) dsc[i] = val[i] >= 0 ? phi_decode_dev(key[i]) : 0.0f;
        uint32_t kkey = 0u;
        int tkeep = 0;
        const bool sel_ok = RADIX && use_radix_select<128>() &&
                            radix_crossing<THREADS, ITEMS>(key, dsc, total, p_d, nb, u.sel, kstar, kkey, tkeep);
        __syncthreads();  // u.sel is dead past this point
        if (sel_ok) {
            SEL_STAMP(2)
            // kept = key > K*, or key == K* among the first t of the tie group in block order
            int ties = 0;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) ties += (val[i] >= 0 && key[i] == kkey) ? 1 : 0;
            int rank = static_cast<int>(block_exclusive_scan(static_cast<double>(ties), red_d));
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                if (val[i] < 0) continue;
                bool k = key[i] > kkey;
                if (key[i] == kkey) k = rank++ < tkeep;
                blk[val[i]] = k ? 1 : 0;
            }
            __syncthreads();
            SEL_STAMP(4)
            finish_request(p, r, seg0, N, nb, neff, blk, sc, kstar, degenerate, total, red_d, red_i);
            SEL_STAMP(5)
            return;
        }
        // 2b. stable descending radix sort of phi(s): ties keep ascending block index, the
        //    order of PackedScore's ~g low word (selection.cpp:27-34).
        Sort(u.sort).SortDescending(key, val);
        SEL_STAMP(2)
        // 3. parallel prefix over the thread's ITEMS consecutive ranks.
        float dec[ITEMS];
        double local = 0.0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            dec[i] = val[i] >= 0 ? phi_decode_dev(key[i]) : 0.0f;
            local += static_cast<double>(dec[i]);
        }
        const double base = block_exclusive_scan(local, red_d);
        if (tid == 0) { s_kstar = nb + 1; s_ratio[0] = -1.0; s_ratio[1] = -1.0; }
        __syncthreads();
        double cum = base;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int q = tid * ITEMS + i;
            cum += static_cast<double>(dec[i]);
            if (q < nb && cum / total >= p_d) { atomicMin(&s_kstar, q + 1); break; }
        }
        __syncthreads();
        const int kpar = s_kstar;
        const bool reached = kpar <= nb;
        const int rc = reached ? kpar - 1 : nb - 1;
        cum = base;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int q = tid * ITEMS + i;
            cum += static_cast<double>(dec[i]);
            if (q == rc) s_ratio[0] = cum / total;
            if (q == rc - 1) s_ratio[1] = cum / total;
        }
        __syncthreads();
        if (crossing_certain(reached, rc, s_ratio[0], s_ratio[1], p_d, nb)) {
            kstar = kpar;
        } else {
            __syncthreads();  // u.sort no longer needed
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                u.sorted.key[tid * ITEMS + i] = key[i];
                u.sorted.val[tid * ITEMS + i] = val[i];
            }
            __syncthreads();
            if (tid == 0) s_kstar = exact_crossing(sc, nb, u.sorted.key, p_d);
            __syncthreads();
            kstar = s_kstar;
        }
        SEL_STAMP(3)
        // 4. block decisions.
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int q = tid * ITEMS + i;
            if (val[i] >= 0) blk[val[i]] = q < kstar ? 1 : 0;
        }
    }
    __syncthreads();
    SEL_STAMP(4)
    finish_request(p, r, seg0, N, nb, neff, blk, sc, kstar, degenerate, total, red_d, red_i);
    SEL_STAMP(5)
}

// ---- bitonic variant for large requests (<= kMaxSortBlocks blocks) ------------------
__global__ void __launch_bounds__(kSelThreads)
select_kernel(const SelectParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    if (!cta_batch_valid(p.cu_seqlens, gridDim.x, p.max_tokens)) {  // malformed batch (grid = R)
        if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(p.err, kErrBadSeqlens);
        return;
    }
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ double red_d[32];
    __shared__ int red_i[32];
    __shared__ int s_kstar;
    __shared__ double s_ratio[2];

    const int r = blockIdx.x;
    const int tid = threadIdx.x;
    const int seg0 = p.cu_seqlens[r];
    const int N = p.cu_seqlens[r + 1] - seg0;
    const int G = p.block_size_g;
    const int nb = (N + G - 1) / G;
    if (nb <= p.nb_lo || nb > p.nb_hi) return;  // another size class's launch owns it
    const int neff = min(p.query_window_n, N);
    const bool enabled = p.drop_enabled == nullptr || p.drop_enabled[r] != 0;
    if (!enabled) { keep_all_request(p, r, N, nb, -1); return; }
    if (nb > kMaxSortBlocks) {
        if (tid == 0) raise_error(p.err, kErrTooManyBlocks);
        keep_all_request(p, r, N, nb, -1);
        return;
    }
    int P2 = 1;
    while (P2 < nb) P2 <<= 1;
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
    float* sc = reinterpret_cast<float*>(keys + P2);
    uint8_t* blk = reinterpret_cast<uint8_t*>(sc + nb);
    const float* bs = p.block_scores + p.cu_blocks[r];

    bool bad = false;
    double tsum = 0.0;
    for (int g = tid; g < P2; g += blockDim.x) {
        if (g < nb) {
            const float s = bs[g];
            if (!(s >= 0.0f) || !isfinite(s)) bad = true;
            sc[g] = s;
            tsum += s;
            keys[g] = (static_cast<uint64_t>(phi_encode_dev(s)) << 32) | static_cast<uint64_t>(~static_cast<uint32_t>(g));
            blk[g] = 0;
        } else {
            keys[g] = 0;
        }
    }
    bad = __syncthreads_or(bad);
    if (bad) {
        if (tid == 0) raise_error(p.err, kErrBadScore);
        keep_all_request(p, r, N, nb, -1);
        return;
    }
    const double total = block_sum<double>(tsum, red_d);
    const bool degenerate = !(total > 0.0);
    int kstar = nb;
    if (!degenerate) {
        for (int kk = 2; kk <= P2; kk <<= 1) {
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                for (int i = tid; i < P2; i += blockDim.x) {
                    const int ixj = i ^ jj;
                    if (ixj > i) {
                        const uint64_t a = keys[i], b = keys[ixj];
                        const bool desc = (i & kk) == 0;
                        if (desc ? (a < b) : (a > b)) { keys[i] = b; keys[ixj] = a; }
                    }
                }
                __syncthreads();
            }
        }
        const int per = (P2 + blockDim.x - 1) / blockDim.x;
        const int r0 = tid * per;
        const int r1 = min(r0 + per, nb);
        double local = 0.0;
        for (int q = r0; q < r1; ++q) local += static_cast<double>(key_score(keys[q]));
        const double base = block_exclusive_scan(local, red_d);
        const double p_d = static_cast<double>(p.top_p);
        if (tid == 0) { s_kstar = nb + 1; s_ratio[0] = -1.0; s_ratio[1] = -1.0; }
        __syncthreads();
        double cum = base;
        for (int q = r0; q < r1; ++q) {
            cum += static_cast<double>(key_score(keys[q]));
            if (cum / total >= p_d) { atomicMin(&s_kstar, q + 1); break; }
        }
        __syncthreads();
        const int kpar = s_kstar;
        const bool reached = kpar <= nb;
        const int rc = reached ? kpar - 1 : nb - 1;
        cum = base;
        for (int q = r0; q < r1; ++q) {
            cum += static_cast<double>(key_score(keys[q]));
            if (q == rc) s_ratio[0] = cum / total;
            if (q == rc - 1) s_ratio[1] = cum / total;
        }
        __syncthreads();
        if (crossing_certain(reached, rc, s_ratio[0], s_ratio[1], p_d, nb)) {
            kstar = kpar;
        } else {
            if (tid == 0) {
                double tot = 0.0;
                for (int g = 0; g < nb; ++g) tot += sc[g];
                double c = 0.0;
                int k = nb;
                for (int q = 0; q < nb; ++q) {
                    c += static_cast<double>(key_score(keys[q]));
                    if (c / tot >= p_d) { k = q + 1; break; }
                }
                s_kstar = k;
            }
            __syncthreads();
            kstar = s_kstar;
        }
        for (int q = tid; q < kstar; q += blockDim.x) blk[~static_cast<uint32_t>(keys[q] & 0xFFFFFFFFull)] = 1;
    } else {
        for (int g = tid; g < nb; g += blockDim.x) blk[g] = 1;
    }
    __syncthreads();
    finish_request(p, r, seg0, N, nb, neff, blk, sc, kstar, degenerate, total, red_d, red_i);
}

// ---- token expansion (expand_mask, selection.cpp:36-49), grid-wide -------------------
// keep[i] = block kept | i < A | i >= N - n_eff (segment-relative), minus the veto;
// pass-through segments keep everything.  16 tokens per thread, one 16-byte store.
__global__ void __launch_bounds__(256)
expand_kernel(const SelectParams p, int R) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    if (!cta_batch_valid(p.cu_seqlens, R, p.max_tokens)) {  // malformed batch: nothing written
        if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(p.err, kErrBadSeqlens);
        return;
    }
    __shared__ int red[8];
    const int T = p.cu_seqlens[R];
    const int64_t A = p.sink_count_a;
    const int G = p.block_size_g;
    const bool aligned = (reinterpret_cast<uintptr_t>(p.keep) & 3) == 0;
    // one 1024-token tile per CTA iteration, 4 tokens per thread (one 32-bit store); the
    // tile's kept count goes to tile_counts (the compaction's count pass, done here)
    for (int64_t tile = blockIdx.x; tile * 1024 < T; tile += gridDim.x) {
        const int i0 = static_cast<int>(tile * 1024) + 4 * static_cast<int>(threadIdx.x);
        uint32_t w = 0u;
        if (i0 < T) {
            int r = find_segment(p.cu_seqlens, R, i0);
            int seg0 = p.cu_seqlens[r], seg1 = p.cu_seqlens[r + 1];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int i = i0 + x;
                if (i >= T) break;
                while (i >= seg1) { ++r; seg0 = seg1; seg1 = p.cu_seqlens[r + 1]; }
                uint32_t k = 1;
                if (p.drop_enabled == nullptr || p.drop_enabled[r]) {
                    const int li = i - seg0;
                    const int N = seg1 - seg0;
                    const int neff = min(p.query_window_n, N);
                    k = (p.blk_keep[p.cu_blocks[r] + li / G] != 0 || li < A || li >= N - neff) ? 1u : 0u;
                    if (k && p.veto != nullptr && p.veto[i]) k = 0;
                }
                w |= k << (8 * x);
            }
            if (aligned && i0 + 4 <= T) {
                *reinterpret_cast<uint32_t*>(p.keep + i0) = w;
            } else {
                for (int x = 0; x < 4 && i0 + x < T; ++x) p.keep[i0 + x] = static_cast<uint8_t>(w >> (8 * x));
            }
        }
        if (p.tile_counts != nullptr) {
            int c = __popc(w);  // one bit per kept token (bytes are 0 or 1)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
            __syncthreads();
            if (threadIdx.x == 0) {
                int s = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) s += red[q];
                p.tile_counts[tile] = s;
            }
            __syncthreads();
        }
    }
}

constexpr int kExpandTile = 1024;

size_t select_smem_bytes(int max_blocks_per_request) {
    int P2 = 1;
    while (P2 < max_blocks_per_request) P2 <<= 1;
    return static_cast<size_t>(P2) * 8 + static_cast<size_t>(max_blocks_per_request) * 5 + 16;
}

bool select_fuses_expand(int64_t max_tokens) { return max_tokens <= kSmallExpandTokens; }

// Side stream + fork/join events of the calling thread on the current device: the larger
// size classes run beside the <= 512-block class instead of after it (they own disjoint
// requests).  Stream capture records the fork as graph edges.
struct SelectFork {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static cudaError_t select_fork_for(SelectFork** out) {
    static thread_local SelectFork forks[32];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 32) return cudaErrorInvalidDevice;
    SelectFork& f = forks[dev];
    if (f.side == nullptr) {
        // first use may fall inside a stream capture (torch.cuda.graph: global mode):
        // create the stream and events in relaxed mode
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        cudaThreadExchangeStreamCaptureMode(&mode);
        e = cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (e != cudaSuccess) return e;
    }
    *out = &f;
    return cudaSuccess;
}

cudaError_t launch_select(const SelectParams& p, int R, int max_blocks_per_request, int num_sms,
                          cudaStream_t stream) {
    // One launch per request size class present under the capacity (the sort's cost
    // grows with the CTA's capacity, so small requests must not pay for a large one):
    // <= 512 blocks: 128 x 4 radix select; <= 2048: 512 x 4 sort; larger: the bitonic
    // kernel.  The larger classes run on a side stream beside the first (disjoint
    // requests): c5 (64 requests, 4K-128K) 42.3 -> 31.2 us per event, c2 12.8 -> 11.9 us.
    // Measured and dropped: one launch for every request <= 2048 blocks -- 128 x 16 radix
    // (c5 45.2 us, 4 x 32K 13.3 -> 21.2 us) or 512 x 4 radix (c5 35.6 us, 4 x 32K 17.1 us).
    // UP_SELECT_FORK=0: all classes on the caller's stream (A/B).
    cudaError_t e;
    SelectParams q = p;
    q.nb_lo = 0;
    q.nb_hi = 512;
    {
        static const bool fork_ok = [] {
            const char* s = std::getenv("UP_SELECT_FORK");
            return s == nullptr || s[0] != '0';
        }();
        SelectFork* f = nullptr;
        const bool fork = fork_ok && max_blocks_per_request > 512;
        if (fork) {  // the larger classes on the side stream, after everything enqueued so far
            if ((e = select_fork_for(&f)) != cudaSuccess) return e;
            if ((e = cudaEventRecord(f->fork, stream)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(f->side, f->fork, 0)) != cudaSuccess) return e;
        }
        if ((e = launch_k(kPdlSelect, select_radix_kernel<128, 4>, R, 128, 0, stream, q)) != cudaSuccess) return e;
        cudaStream_t big = fork ? f->side : stream;
        const int fam = fork ? 0 : kPdlSelect;  // no programmatic edge after an event wait
        if (max_blocks_per_request > 512) {
            q.nb_lo = 512;
            q.nb_hi = 2048;
            if ((e = launch_k(fam, select_radix_kernel<512, 4>, R, 512, 0, big, q)) != cudaSuccess) return e;
        }
        if (max_blocks_per_request > 2048) {
            const int cap = max_blocks_per_request < kMaxSortBlocks ? max_blocks_per_request : kMaxSortBlocks;
            const size_t smem = select_smem_bytes(cap);
            e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            q.nb_lo = 2048;
            q.nb_hi = 0x7fffffff;
            if ((e = launch_k(fam, select_kernel, R, kSelThreads, smem, big, q)) != cudaSuccess) return e;
        }
        if (fork) {
            if ((e = cudaEventRecord(f->join, f->side)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(stream, f->join, 0)) != cudaSuccess) return e;
        }
    }
    if (e != cudaSuccess) return e;
    if (p.fuse_expand) return cudaSuccess;  // the select CTAs wrote the token masks
    static_assert(kExpandTile == 1024, "expand tiles = compaction scan tiles");
    int64_t grid = (p.max_tokens + kExpandTile - 1) / kExpandTile;  // one tile per CTA
    if (grid > num_sms * 8) grid = num_sms * 8;
    if (grid < 1) grid = 1;
    return launch_k(kPdlSelect, expand_kernel, static_cast<unsigned>(grid), 256, 0, stream, q, R);
}

// allreduce_scores (tp_sim.cpp:43-47): fp32 sum in ascending shard order from 0.0f.
struct ReduceParams {
    const float* shards[16];
    int32_t tp;
    int64_t count;
    float* out;
};

__global__ void reduce_shards_kernel(const ReduceParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < p.count;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float acc = 0.0f;
        for (int t = 0; t < p.tp; ++t) acc = __fadd_rn(acc, p.shards[t][g]);
        p.out[g] = acc;
    }
}

cudaError_t launch_reduce_shards(const float* const* shards, int tp, int64_t count, float* out,
                                 int num_sms, cudaStream_t stream) {
    ReduceParams p{};
    for (int t = 0; t < tp; ++t) p.shards[t] = shards[t];
    p.tp = tp;
    p.count = count;
    p.out = out;
    int64_t grid = (count + 255) / 256;
    if (grid > num_sms * 4) grid = num_sms * 4;
    if (grid < 1) grid = 1;
    return launch_k(kPdlSelect, reduce_shards_kernel, static_cast<unsigned>(grid), 256, 0, stream, p);
}

}  // namespace up
