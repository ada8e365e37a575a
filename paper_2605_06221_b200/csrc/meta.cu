// meta.cu -- per-layer metadata that downstream layers read after a drop (sm_100a):
//
//   slot_mapping_kernel -- Eq. 16 (PagedKVCache::slot_for /
//       recompute_slots_after_drop, kvcache.cpp:67-80, :147-158): for every retained row i
//       of the compacted batch and every downstream layer l,
//           slot[l][i] = block_table[l][r_i][p_i / B] * B + p_i % B
//       with r_i the row's segment (from the compacted cu_seqlens) and p_i its logical
//       position.  Pages are allocated by the caller's block manager; a missing page
//       (negative table entry or page index past the table) raises the sticky
//       AllocationMiss flag and writes slot -1.
//   decode_seqused_kernel -- Eq. 17 (decode_seqused,
//       kvcache.cpp:182-186): seqused[l][r] = (retained length of r after the last drop
//       at a layer < l, else its original length) + decode_appended[r].
#include "params.cuh"

namespace up {

__global__ void __launch_bounds__(256)
slot_mapping_kernel(const SlotMapParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    const int64_t n = p.num_rows != nullptr ? static_cast<int64_t>(*p.num_rows) : p.max_rows;
    const int64_t total = n * p.num_layers;
    for (int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < total;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int l = static_cast<int>(x / n);
        const int64_t i = x - static_cast<int64_t>(l) * n;
        const int r = find_segment(p.cu_seqlens, p.num_requests, i);
        const int64_t pos = p.positions[i];
        const int64_t page = pos / p.block_size;
        int64_t slot = -1;
        if (pos >= 0 && page < p.max_pages) {
            const int32_t phys = p.block_tables[(static_cast<int64_t>(l) * p.num_requests + r) * p.max_pages + page];
            if (phys >= 0) slot = static_cast<int64_t>(phys) * p.block_size + pos % p.block_size;
        }
        if (slot < 0) raise_error(p.err, kErrAllocationMiss);
        p.slots[static_cast<int64_t>(l) * p.slot_stride + i] = slot;
    }
}

__global__ void __launch_bounds__(256)
decode_seqused_kernel(const SequsedParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    const int total = p.num_layers * p.num_requests;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
        const int l = x / p.num_requests;
        const int r = x - l * p.num_requests;
        // DropHistory::last_event_before (kvcache.cpp:32-39): last drop at a layer < l
        int k = -1;
        for (int d = 0; d < p.num_drops; ++d) {
            if (p.drop_layers[d] < l) k = d;
            else break;
        }
        const int32_t* cu = k >= 0 ? p.cu_after[k] : p.cu_orig;
        const int64_t base = cu[r + 1] - cu[r];
        p.seqused[x] = static_cast<int32_t>(base + (p.decode_appended ? p.decode_appended[r] : 0));
    }
}

cudaError_t launch_slot_mapping(const SlotMapParams& p, int num_sms, cudaStream_t stream) {
    int64_t work = p.max_rows * p.num_layers;
    int64_t grid = (work + 255) / 256;
    if (grid > num_sms * 8) grid = num_sms * 8;
    if (grid < 1) grid = 1;
    return launch_k(kPdlMeta, slot_mapping_kernel, static_cast<unsigned>(grid), 256, 0, stream, p);
}

cudaError_t launch_decode_seqused(const SequsedParams& p, cudaStream_t stream) {
    const int total = p.num_layers * p.num_requests;
    const int grid = total > 0 ? (total + 255) / 256 : 1;
    return launch_k(kPdlMeta, decode_seqused_kernel, grid, 256, 0, stream, p);
}

}  // namespace up
