// compact.cu -- segmented prefix sum + gather compaction of retained rows (sm_100a).
//
// Restates apply_drop / gather_rows / patch_metadata (propagation.cpp:47-77, :105-112;
// scheduler.cpp:50-90) for a device-resident varlen batch, in three stream-ordered kernels:
//   compact_count_kernel -- retained rows per tile of kCompactTile source rows;
//   compact_index_kernel -- tile offset = Σ earlier tile counts, CTA-wide exclusive scan of
//                           the keep bits -> retained_index[out] = source row, the new
//                           cu_seqlens entries falling in the tile (new_cu[s] = #retained
//                           rows before cu[s]) and the device-resident retained count;
//   compact_copy_kernel  -- persistent grid, warp per output row (uniform work whatever the
//                           keep pattern), every plane copied with 16-byte streaming
//                           loads/stores, a batch of 8 vectors in flight per lane.  Out of
//                           place: the pre-drop buffer keeps the parked rows
//                           (propagation.cpp:64-67).
#include <cstdlib>
#include "params.cuh"

namespace up {

constexpr int kCompactTile = 1024;     // source rows per scan CTA
constexpr int kCompactThreads = 256;   // 4 rows per thread
constexpr int kCopyThreads = 256;

__device__ __forceinline__ bool row_kept(const CompactParams& p, int64_t i, int T) {
    if (i >= T) return false;
    if (p.drop_enabled != nullptr) {
        const int r = find_segment(p.cu_seqlens, p.num_requests, i);
        if (!p.drop_enabled[r]) return true;
    }
    return p.keep[i] != 0;
}

__global__ void __launch_bounds__(kCompactThreads)
compact_count_kernel(const CompactParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    constexpr int PER = kCompactTile / kCompactThreads;
    __shared__ int red[kCompactThreads / 32];
    // a malformed batch (flagged by the scorer / select) counts nothing; the index pass then
    // emits an empty result
    const bool valid = cta_batch_valid(p.cu_seqlens, p.num_requests, p.max_tokens);
    const int T = valid ? p.cu_seqlens[p.num_requests] : 0;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kCompactTile;
    int c = 0;
    if (t0 < T) {
        const int64_t i0 = t0 + threadIdx.x * PER;
#pragma unroll
        for (int q = 0; q < PER; ++q) c += row_kept(p, i0 + q, T) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < kCompactThreads / 32; ++w) s += red[w];
        p.tile_counts[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kCompactThreads)
compact_index_kernel(const CompactParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    constexpr int PER = kCompactTile / kCompactThreads;
    __shared__ int red[kCompactThreads / 32];
    __shared__ int warp_tot[kCompactThreads / 32];
    __shared__ int s_offset;
    // A malformed batch (cu_seqlens not 0-based / strictly increasing / past capacity, flagged
    // by the scorer / select) compacts to an empty result: the keep mask and the tile counts
    // of such a batch are stale, so nothing is derived from them.
    if (!cta_batch_valid(p.cu_seqlens, p.num_requests, p.max_tokens)) {
        if (blockIdx.x == 0) {
            for (int s = threadIdx.x; s <= p.num_requests; s += blockDim.x) p.cu_out[s] = 0;
            if (threadIdx.x == 0 && p.num_out) *p.num_out = 0;
        }
        return;
    }
    const int T = p.cu_seqlens[p.num_requests];
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kCompactTile;
    if (t0 >= T) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    int acc = 0;
    for (int b = tid; b < static_cast<int>(blockIdx.x); b += kCompactThreads) acc += p.tile_counts[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
        int s = 0;
        for (int w = 0; w < kCompactThreads / 32; ++w) s += red[w];
        s_offset = s;
    }

    const int64_t i0 = t0 + tid * PER;
    uint32_t bits = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) bits |= (row_kept(p, i0 + q, T) ? 1u : 0u) << q;
    const int cnt = __popc(bits);
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    int wbase = 0, local_total = 0;
    for (int w = 0; w < kCompactThreads / 32; ++w) {
        if (w < warp) wbase += warp_tot[w];
        local_total += warp_tot[w];
    }
    const int offset = s_offset;
    int pos = offset + wbase + x - cnt;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int64_t i = i0 + q;
        if (i < T) {
            const int s = find_segment(p.cu_seqlens, p.num_requests, i);
            if (p.cu_seqlens[s] == i) p.cu_out[s] = pos;
        }
        if (bits & (1u << q)) {
            p.retained_index[pos] = static_cast<int32_t>(i);
            ++pos;
        }
    }
    if (t0 + kCompactTile >= T && tid == 0) {
        p.cu_out[p.num_requests] = offset + local_total;
        if (p.num_out) *p.num_out = offset + local_total;
    }
}

// One warp copies row src_row of plane pl to row dst_row: 16-byte streaming vectors, a
// batch of 8 in flight per lane (scalar fallbacks for unaligned planes).
// U = 16-byte vectors per lane in flight per step
template <int U = 8>
__device__ __forceinline__ void copy_row_plane(const CompactParams& p, int pl, int64_t src_row, int64_t dst_row,
                                               int lane) {
    {
        const int64_t rb = p.row_bytes[pl];
        const uint8_t* src = p.src[pl] + src_row * p.src_stride[pl];
        uint8_t* dst = p.dst[pl] + dst_row * p.dst_stride[pl];
        const uintptr_t align = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
        if (((rb | static_cast<int64_t>(align)) & 15) == 0) {
            const int4* s = reinterpret_cast<const int4*>(src);
            int4* d = reinterpret_cast<int4*>(dst);
            const int64_t nv = rb >> 4;
            int64_t v = lane;
            for (; v + (U - 1) * 32 < nv; v += U * 32) {
                int4 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) x[u] = __ldcs(s + v + u * 32);
#pragma unroll
                for (int u = 0; u < U; ++u) __stcs(d + v + u * 32, x[u]);
            }
            int4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (v + u * 32 < nv) x[u] = __ldcs(s + v + u * 32);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (v + u * 32 < nv) __stcs(d + v + u * 32, x[u]);
        } else if (((rb | static_cast<int64_t>(align)) & 3) == 0) {
            for (int64_t b = lane * 4; b < rb; b += 32 * 4)
                *reinterpret_cast<uint32_t*>(dst + b) = *reinterpret_cast<const uint32_t*>(src + b);
        } else {
            for (int64_t b = lane; b < rb; b += 32) dst[b] = src[b];
        }
    }
}

// Every plane of a row, one after the other (the large-batch copy: bandwidth-bound).
__device__ __forceinline__ void copy_row_planes(const CompactParams& p, int64_t src_row, int64_t dst_row, int lane) {
#pragma unroll 1
    for (int pl = 0; pl < p.num_planes; ++pl) copy_row_plane(p, pl, src_row, dst_row, lane);
}

// Gather: output row o <- source row retained_index[o] (persistent grid, warp per row).
__global__ void __launch_bounds__(kCopyThreads)
compact_copy_kernel(const CompactParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * kCopyThreads + threadIdx.x) >> 5;
    const int nw = (gridDim.x * kCopyThreads) >> 5;
    const int n = p.cu_out[p.num_requests];
    for (int o = gw; o < n; o += nw) copy_row_planes(p, p.retained_index[o], o, lane);
}

// Scatter, the inverse of the gather: row o of src -> row index[o] of dst, for the first
// *num_out rows (or max_tokens when num_out is null).  Unwinding a drop this way writes the
// current state of every retained row back over its pre-drop row, so the pre-drop buffer
// becomes the reconstituted stream (reconstitute, propagation.cpp:79-100: parked rows keep
// the state they had when dropped).
__global__ void __launch_bounds__(kCopyThreads)
scatter_rows_kernel(const CompactParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * kCopyThreads + threadIdx.x) >> 5;
    const int nw = (gridDim.x * kCopyThreads) >> 5;
    const int64_t n = p.num_out != nullptr ? static_cast<int64_t>(*p.num_out) : p.max_tokens;
    for (int64_t o = gw; o < n; o += nw) {
        const int32_t d = p.retained_index[o];
        if (d < 0) continue;  // row without a destination
        copy_row_planes(p, o, d, lane);
    }
}

// Small capacities (<= kSmallCompactRows source rows, e.g. BASELINE C1's single 4K request):
// the count / index / copy kernels collapse into one launch.  Every CTA scans the whole keep
// mask (a few KB, L2-resident) into its own shared-memory retained index -- CTA 0 also
// publishes retained_index, cu_seqlens_out and num_out -- then copies its share of the
// output rows exactly as compact_copy_kernel does.
constexpr int kSmallCompactRows = 8192;
#ifndef UP_SMALL_COPY_UNROLL  // measured C1: 8 -> 10.2 us, 16 (a whole hidden row per round trip) -> 17.1 us
#define UP_SMALL_COPY_UNROLL 8
#endif

__global__ void __launch_bounds__(kCopyThreads)
compact_small_kernel(const CompactParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    constexpr int PER = 16;  // rows per thread per chunk: one 16-byte load of the keep mask
    constexpr int CHUNK = kCopyThreads * PER;
    extern __shared__ int32_t idx[];  // [max_tokens] (dynamic: the capacity, <= kSmallCompactRows)
    __shared__ int warp_tot[kCopyThreads / 32];
    const bool lead = blockIdx.x == 0;
    if (!cta_batch_valid(p.cu_seqlens, p.num_requests, p.max_tokens)) {  // empty result, as compact_index
        if (lead) {
            for (int s = threadIdx.x; s <= p.num_requests; s += blockDim.x) p.cu_out[s] = 0;
            if (threadIdx.x == 0 && p.num_out) *p.num_out = 0;
        }
        return;
    }
    const int T = p.cu_seqlens[p.num_requests];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int carry = 0;
    for (int base = 0; base < T; base += CHUNK) {
        const int i0 = base + tid * PER;
        uint32_t bits = 0;
        if (p.drop_enabled == nullptr && i0 + PER <= T && (reinterpret_cast<uintptr_t>(p.keep + i0) & 15) == 0) {
            const uint4 w = *reinterpret_cast<const uint4*>(p.keep + i0);  // keep bytes are 0 / 1
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < PER; ++q) bits |= ((ws[q >> 2] >> (8 * (q & 3))) & 1u) << q;
        } else {
#pragma unroll
            for (int q = 0; q < PER; ++q) bits |= (row_kept(p, i0 + q, T) ? 1u : 0u) << q;
        }
        const int cnt = __popc(bits);
        int x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[warp] = x;
        __syncthreads();
        int wbase = 0, chunk_total = 0;
#pragma unroll
        for (int w = 0; w < kCopyThreads / 32; ++w) {
            if (w < warp) wbase += warp_tot[w];
            chunk_total += warp_tot[w];
        }
        int pos = carry + wbase + x - cnt;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int i = i0 + q;
            if (lead && i < T) {
                const int s = find_segment(p.cu_seqlens, p.num_requests, i);
                if (p.cu_seqlens[s] == i) p.cu_out[s] = pos;
            }
            if (bits & (1u << q)) {
                idx[pos] = i;
                if (lead) p.retained_index[pos] = i;
                ++pos;
            }
        }
        carry += chunk_total;
        __syncthreads();  // warp_tot reused by the next chunk
    }
    if (lead && tid == 0) {
        p.cu_out[p.num_requests] = carry;
        if (p.num_out) *p.num_out = carry;
    }
    if (p.num_planes == 0) return;
    // latency-bound: one warp per (row, plane), so a row's planes travel in parallel
    const int gw = (blockIdx.x * kCopyThreads + tid) >> 5;
    const int nw = (gridDim.x * kCopyThreads) >> 5;
    for (int t = gw; t < carry * p.num_planes; t += nw) {
        const int o = t / p.num_planes;
        copy_row_plane<UP_SMALL_COPY_UNROLL>(p, t - o * p.num_planes, idx[o], o, lane);
    }
}

bool compact_is_small(int64_t max_tokens) { return max_tokens <= kSmallCompactRows; }

static int copy_grid(int num_sms, int64_t rows) {
    static int occ = 0;
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, compact_copy_kernel, kCopyThreads, 0);
        if (occ < 1) occ = 1;
    }
    int64_t grid = static_cast<int64_t>(num_sms) * occ;
    const int64_t need = (rows + (kCopyThreads / 32) - 1) / (kCopyThreads / 32);
    if (grid > need) grid = need;
    return static_cast<int>(grid < 1 ? 1 : grid);
}

cudaError_t launch_scatter_rows(const CompactParams& p, int num_sms, cudaStream_t stream) {
    if (p.num_planes == 0 || p.max_tokens == 0) return cudaSuccess;
    return launch_k(kPdlCompact, scatter_rows_kernel, copy_grid(num_sms, p.max_tokens), kCopyThreads, 0, stream, p);
}

// counts_ready: tile_counts already hold the kept rows per kCompactTile tile (written by
// up_select's expand kernel for this keep mask), so the count pass is skipped.
cudaError_t launch_compact(const CompactParams& p, int num_sms, cudaStream_t stream, bool counts_ready) {
    const int64_t tiles = (p.max_tokens + kCompactTile - 1) / kCompactTile;
    cudaError_t e = cudaSuccess;
    if (compact_is_small(p.max_tokens)) {
        static const int per_sm = [] {
            const char* s = std::getenv("UP_SMALL_COMPACT_CTAS_PER_SM");  // dev A/B
            return s == nullptr ? 3 : std::atoi(s);  // C1: 2 / 3 / 4 / 6 / 8 -> 8.8 / 8.4 / 10.0 / 10.2 / 11.8 us
        }();
        int64_t grid = (p.max_tokens * p.num_planes + kCopyThreads / 32 - 1) / (kCopyThreads / 32);  // warp per (row, plane)
        if (grid > per_sm * static_cast<int64_t>(num_sms)) grid = per_sm * static_cast<int64_t>(num_sms);
        return launch_k(kPdlCompact, compact_small_kernel, static_cast<unsigned>(grid < 1 ? 1 : grid), kCopyThreads,
                        sizeof(int32_t) * static_cast<size_t>(p.max_tokens), stream, p);
    }
    if (!counts_ready &&
        (e = launch_k(kPdlCompactScan, compact_count_kernel, static_cast<unsigned>(tiles), kCompactThreads, 0, stream, p)) !=
            cudaSuccess)
        return e;
    if ((e = launch_k(kPdlCompactScan, compact_index_kernel, static_cast<unsigned>(tiles), kCompactThreads, 0, stream, p)) != cudaSuccess)
        return e;
    if (p.num_planes > 0) {
        e = launch_k(kPdlCompact, compact_copy_kernel, copy_grid(num_sms, p.max_tokens), kCopyThreads, 0, stream, p);
    }
    return e;
}

int64_t compact_tiles(int64_t max_tokens) { return (max_tokens + kCompactTile - 1) / kCompactTile; }
int compact_max_planes() { return kMaxPlanes; }

}  // namespace up
