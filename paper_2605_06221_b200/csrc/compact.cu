// compact.cu -- segmented prefix sum + gather compaction of retained rows (sm_100a).
//
// Restates apply_drop / gather_rows / patch_metadata (propagation.cpp:47-77, :105-112;
// scheduler.cpp:50-90) for a device-resident varlen batch:
//   compact_count_kernel   -- kept rows per tile of kCompactTile source rows
//   compact_scatter_kernel -- tile offset = Σ earlier tile counts; CTA-wide exclusive scan of
//                             the keep bits gives each retained row its output slot; writes
//                             retained_index, the new cu_seqlens entries that fall in the
//                             tile (new_cu[s] = #retained rows before cu[s]), and copies the
//                             rows of every plane with 16-byte vector loads/stores, several
//                             in flight per lane (HBM-bound; out of place so the pre-drop
//                             buffer keeps the parked rows, propagation.cpp:64-67).
#include "params.cuh"

namespace up {

constexpr int kCompactTile = 256;      // source rows per CTA
constexpr int kCompactThreads = 256;   // one row per thread

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
    __shared__ int red[kCompactThreads / 32];
    const int T = p.cu_seqlens[p.num_requests];
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kCompactTile;
    int c = 0;
    if (t0 < T) {
        const int64_t i0 = t0 + threadIdx.x * (kCompactTile / kCompactThreads);
#pragma unroll
        for (int q = 0; q < kCompactTile / kCompactThreads; ++q) c += row_kept(p, i0 + q, T) ? 1 : 0;
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

// Copy `bytes` bytes (multiple of 16, 16-byte aligned) with one warp, 8 vectors in flight/lane.
__device__ __forceinline__ void warp_copy_vec(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                              int64_t bytes, int lane) {
    const int64_t nvec = bytes >> 4;
    const int4* s = reinterpret_cast<const int4*>(src);
    int4* d = reinterpret_cast<int4*>(dst);
    int64_t v = lane;
    for (; v + 7 * 32 < nvec; v += 8 * 32) {
        int4 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldcs(s + v + u * 32);
#pragma unroll
        for (int u = 0; u < 8; ++u) __stcs(d + v + u * 32, x[u]);
    }
    for (; v < nvec; v += 32) __stcs(d + v, __ldcs(s + v));
}

__global__ void __launch_bounds__(kCompactThreads)
compact_scatter_kernel(const CompactParams p) {
    constexpr int PER = kCompactTile / kCompactThreads;
    __shared__ int red[kCompactThreads / 32];
    __shared__ int warp_tot[kCompactThreads / 32];
    __shared__ int s_offset;
    __shared__ int s_rows[kCompactTile];  // source rows of this tile's retained rows, in order
    const int T = p.cu_seqlens[p.num_requests];
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kCompactTile;
    if (t0 >= T) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // Offset of this tile: Σ counts of earlier tiles.
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

    // Local exclusive scan of the keep bits (PER consecutive rows per thread).
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
    int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += warp_tot[w];
    int local_total = 0;
    for (int w = 0; w < kCompactThreads / 32; ++w) local_total += warp_tot[w];
    const int excl = wbase + x - cnt;
    const int offset = s_offset;

    int pos = excl;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int64_t i = i0 + q;
        if (i < T) {
            // New cu_seqlens entry for a segment starting at this row.
            const int s = find_segment(p.cu_seqlens, p.num_requests, i);
            if (p.cu_seqlens[s] == i) p.cu_out[s] = offset + pos;
        }
        if (bits & (1u << q)) {
            s_rows[pos] = static_cast<int>(i);
            if (p.retained_index) p.retained_index[offset + pos] = static_cast<int32_t>(i);
            ++pos;
        }
    }
    if (t0 + kCompactTile >= T && tid == 0) {
        p.cu_out[p.num_requests] = offset + local_total;
        if (p.num_out) *p.num_out = offset + local_total;
    }
    __syncthreads();

    // Row copies: warp per (row, plane).
    const int units = local_total * p.num_planes;
    for (int u = warp; u < units; u += kCompactThreads / 32) {
        const int q = u / p.num_planes;
        const int pl = u - q * p.num_planes;
        const int64_t src_row = s_rows[q];
        const int64_t dst_row = offset + q;
        const int64_t rb = p.row_bytes[pl];
        const uint8_t* src = p.src[pl] + src_row * p.src_stride[pl];
        uint8_t* dst = p.dst[pl] + dst_row * p.dst_stride[pl];
        const bool vec = ((rb & 15) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
        if (vec) {
            warp_copy_vec(dst, src, rb, lane);
        } else if ((rb & 7) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7) == 0) {
            for (int64_t b = lane * 8; b < rb; b += 32 * 8)
                *reinterpret_cast<uint64_t*>(dst + b) = *reinterpret_cast<const uint64_t*>(src + b);
        } else if ((rb & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3) == 0) {
            for (int64_t b = lane * 4; b < rb; b += 32 * 4)
                *reinterpret_cast<uint32_t*>(dst + b) = *reinterpret_cast<const uint32_t*>(src + b);
        } else {
            for (int64_t b = lane; b < rb; b += 32) dst[b] = src[b];
        }
    }
}

// Narrow planes (positions: 4 or 8 bytes per row) are copied thread-per-row instead of
// warp-per-row; the scatter kernel handles them too, this keeps the row loop above simple.
cudaError_t launch_compact(const CompactParams& p, cudaStream_t stream) {
    const int64_t tiles = (p.max_tokens + kCompactTile - 1) / kCompactTile;
    compact_count_kernel<<<static_cast<unsigned>(tiles), kCompactThreads, 0, stream>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    compact_scatter_kernel<<<static_cast<unsigned>(tiles), kCompactThreads, 0, stream>>>(p);
    return cudaGetLastError();
}

int64_t compact_tiles(int64_t max_tokens) { return (max_tokens + kCompactTile - 1) / kCompactTile; }
int compact_max_planes() { return kMaxPlanes; }

}  // namespace up
