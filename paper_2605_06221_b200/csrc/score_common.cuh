// score_common.cuh -- pieces shared by the tcgen05 scorer kernels (score_tc.cu,
// score_tcw.cu): the balanced work partition and the packed exp2 group sums.
#pragma once

#include "params.cuh"

namespace up {


// Segments per launch of score_tcw: its work plan (per-request unit and block prefix sums)
// lives in shared memory, 8 bytes per segment.  4096 segments (32 KB) still leave the K ring
// its 2 (D <= 128, HPC = 4) / 3 (D = 256) stages, so continuous batches with hundreds of
// decode pass-through segments keep the fast scorer; the CTA-pair kernel keeps 256.
constexpr int kTcwMaxRequests = 4096;
constexpr int kTc2MaxRequests = 256;

// ---------------------------------------------------------------- partition
struct Part {
    const int32_t* cu_units;  // smem [R+1]
    int R;
    int nhg;
    int64_t U;
    int grid;
};

struct Item {
    int r, hg;
    int u0, u1;        // unit range inside the pair
    int64_t sid;       // global unit position of the item start (stats id)
    int64_t seg_start; // global unit position of the pair's unit 0
    int units_r;
};

__device__ __forceinline__ int64_t range_begin(const Part& P, int c) {
    return static_cast<int64_t>(c) * P.U / P.grid;
}

// CTA whose range holds global unit position pos: largest c with c*U/grid <= pos.
__device__ __forceinline__ int cta_of(const Part& P, int64_t pos) {
    return static_cast<int>(((pos + 1) * P.grid - 1) / P.U);
}

__device__ __forceinline__ Item make_item(const Part& P, int64_t pos, int64_t end) {
    Item it;
    // request: largest r with cu_units[r]*nhg <= pos (pairs with zero units are skipped)
    int lo = 0, hi = P.R - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (static_cast<int64_t>(P.cu_units[mid]) * P.nhg <= pos) lo = mid; else hi = mid - 1;
    }
    it.r = lo;
    it.units_r = P.cu_units[lo + 1] - P.cu_units[lo];
    const int64_t base = static_cast<int64_t>(P.cu_units[lo]) * P.nhg;
    const int64_t rel = pos - base;
    it.hg = static_cast<int>(rel / it.units_r);
    it.u0 = static_cast<int>(rel - static_cast<int64_t>(it.hg) * it.units_r);
    it.seg_start = base + static_cast<int64_t>(it.hg) * it.units_r;
    const int64_t seg_end = it.seg_start + it.units_r;
    const int64_t stop = end < seg_end ? end : seg_end;
    it.u1 = it.u0 + static_cast<int>(stop - pos);
    it.sid = pos;
    return it;
}

// unit_sid entries: the item id (its first unit's position, < 2^28) in the low 28 bits and,
// for the scorers whose statistics parity is not a function of the key position alone
// (score_tcw, score_tc2), the parity of the unit's first subtile in the top 4 bits.
__host__ __device__ __forceinline__ int32_t tcw_usid(int32_t sid, int par0) {
    return sid | static_cast<int32_t>(static_cast<uint32_t>(par0) << kUsidParShift);
}
__device__ __forceinline__ int64_t usid_item(int32_t v) { return v & ((1 << kUsidParShift) - 1); }
// statistics parity of a block whose first key is `off` parity units into its 128-key unit
__device__ __forceinline__ int usid_par(int32_t v, int off, int npar) {
    return npar > 1 ? static_cast<int>(((static_cast<uint32_t>(v) >> kUsidParShift) + off) % npar) : 0;
}

// ---------------------------------------------------------------- pair statistics
__device__ __forceinline__ void lse_merge(float& M, float& L, float mc, float lc) {
    if (mc == -INFINITY) return;
    if (mc > M) { L = L * ex2_approx(M - mc) + lc; M = mc; }
    else L += lc * ex2_approx(mc - M);
}

// Of the 16 element pairs of a 32-column group, NP evaluate 2^x with the FMA-pipe
// polynomial (exp2_poly2) instead of MUFU.EX2.  Measured on B200: the four-warpgroup
// scorer (score_tcw.cu) is fastest at NP = 3..5 for D = 128 (MUFU-bound) and NP = 0 for
// D = 256; the two-warpgroup kernel is latency- rather than MUFU-limited and uses NP = 0.
#ifndef UP_POLY_PAIRS
#define UP_POLY_PAIRS 0
#endif
constexpr int kPolyPairs = UP_POLY_PAIRS;

// Σ_k 2^(v_k * sc - m) over 32 TMEM values: packed FFMA2 for the exponent argument, MUFU
// ex2 (or the FMA-pipe polynomial for the last NP pairs), two FADD2 chains.
template <int NP = kPolyPairs>
__device__ __forceinline__ float group_sum_pk(const uint32_t* v, uint64_t sc2, uint64_t m2) {
    uint64_t a0 = 0, a1 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const uint64_t x = fma2(static_cast<uint64_t>(v[2 * i]) | (static_cast<uint64_t>(v[2 * i + 1]) << 32), sc2, m2);
        const uint64_t e = i < 16 - NP ? pk(ex2_approx(lo_f(x)), ex2_approx(hi_f(x))) : exp2_poly2(x);
        if (i == 0) a0 = e;
        else if (i == 1) a1 = e;
        else if (i & 1) a1 = add2(a1, e);
        else a0 = add2(a0, e);
    }
    const uint64_t a = add2(a0, a1);
    return lo_f(a) + hi_f(a);
}

// Packed partial Σ 2^(v_k * sc - m) over 2*PAIRS TMEM values (the last NP pairs on the FMA
// pipe): lo/hi halves of the returned pair are the two accumulation chains.
template <int PAIRS, int NP>
__device__ __forceinline__ uint64_t chunk_sum_pk(const uint32_t* v, uint64_t sc2, uint64_t m2) {
    uint64_t a0 = 0, a1 = 0;
#pragma unroll
    for (int i = 0; i < PAIRS; ++i) {
        const uint64_t x = fma2(static_cast<uint64_t>(v[2 * i]) | (static_cast<uint64_t>(v[2 * i + 1]) << 32), sc2, m2);
        const uint64_t e = i < PAIRS - NP ? pk(ex2_approx(lo_f(x)), ex2_approx(hi_f(x))) : exp2_poly2(x);
        if (i == 0) a0 = e;
        else if (i == 1) a1 = e;
        else if (i & 1) a1 = add2(a1, e);
        else a0 = add2(a0, e);
    }
    return add2(a0, a1);
}

// Makes `v` a fresh definition at this point of the program: code using it cannot be
// scheduled above this statement (used to keep a TMEM load of the next chunk in flight
// while the current chunk is summed).
__device__ __forceinline__ void pin16(uint32_t (&v)[16]) {
    asm volatile("" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                 "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]),
                 "+r"(v[14]), "+r"(v[15]));
}

// Cold path of a rebase: rescale the partials this thread already wrote for the item.
static __device__ __noinline__ void rescale_rows(float* prow, int g0, int g1, float f) {
#pragma unroll 4
    for (int g = g0; g < g1; ++g) prow[static_cast<int64_t>(g) * kRows] *= f;
}

}  // namespace up
