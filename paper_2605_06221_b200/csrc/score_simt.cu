// score_simt.cu -- generic importance scorer on CUDA cores (any n, G, D; token scores).
//
// Used when the tensor-core scorer's envelope does not apply (n > 128, G not a multiple
// of 32, D not in {64, 128, 256}) or when the caller asks for per-token scores
// (ImportanceScores::token_scores, importance.hpp:18-23).  Same math as the reference
// (importance.cpp:17-132) in two passes:
//   simt_row_stats_kernel  -- warp per (request, head, query row): max and denominator of
//                             the row's softmax over keys 0..query position (:45-59)
//   simt_token_kernel      -- warp per key: Σ_h Σ_j exp(s - m) / l / n_eff (:61-66),
//                             accumulated in double
//   simt_block_kernel      -- thread per block: mean of the float token scores (:76-90)
#include <cuda_bf16.h>

#include "params.cuh"

namespace up {

__device__ __forceinline__ float dot_bf16(const __nv_bfloat16* a, const __nv_bfloat16* b, int D) {
    float acc = 0.f;
    for (int c = 0; c < D; ++c) acc = fmaf(__bfloat162float(a[c]), __bfloat162float(b[c]), acc);
    return acc;
}

__device__ __forceinline__ int kv_of(const ScoreSimtParams& p, int h) {
    return (p.q_head_offset + h) / p.gqa_group - p.kv_head_offset;
}

__global__ void simt_row_stats_kernel(const ScoreSimtParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    if (!cta_batch_valid(p.cu_seqlens, p.num_requests, p.max_tokens)) return;  // flagged by the plan
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + warp;
    const int r = blockIdx.y / p.num_heads;
    const int h = blockIdx.y % p.num_heads;
    if (p.drop_enabled != nullptr && !p.drop_enabled[r]) return;
    const int seg0 = p.cu_seqlens[r];
    const int N = p.cu_seqlens[r + 1] - seg0;
    const int neff = min(p.query_window_n, N);
    if (j >= neff) return;
    const int qpos = N - neff + j;
    const __nv_bfloat16* qrow = p.q + static_cast<int64_t>(seg0 + qpos) * p.q_row_stride +
                                static_cast<int64_t>(h) * p.head_dim;
    const int kvh = kv_of(p, h);
    float m = -INFINITY, l = 0.f;
    for (int i = lane; i <= qpos; i += 32) {
        const __nv_bfloat16* krow = p.k + static_cast<int64_t>(seg0 + i) * p.k_row_stride +
                                    static_cast<int64_t>(kvh) * p.head_dim;
        const float s = dot_bf16(qrow, krow, p.head_dim) * p.scale;
        if (s > m) { l = l * expf(m - s) + 1.f; m = s; } else { l += expf(s - m); }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float l2 = __shfl_xor_sync(0xffffffffu, l, o);
        const float mm = fmaxf(m, m2);
        l = (m == -INFINITY ? 0.f : l * expf(m - mm)) + (m2 == -INFINITY ? 0.f : l2 * expf(m2 - mm));
        m = mm;
    }
    if (lane == 0) {
        const int64_t idx = (static_cast<int64_t>(h) * p.num_requests + r) * p.simt_n + j;
        p.row_m[idx] = m;
        p.row_l[idx] = l;
    }
}

// Warp per global token index; lanes stride over (head, query row) pairs.
__global__ void simt_token_kernel(const ScoreSimtParams p, int64_t total_tokens_cap) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    if (!cta_batch_valid(p.cu_seqlens, p.num_requests, p.max_tokens)) return;  // flagged by the plan
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    const int T = p.cu_seqlens[p.num_requests];
    if (t >= T || t >= total_tokens_cap) return;
    const int r = find_segment(p.cu_seqlens, p.num_requests, t);
    if (p.drop_enabled != nullptr && !p.drop_enabled[r]) {
        if (lane == 0 && p.token_scores) p.token_scores[t] = 0.f;
        return;
    }
    const int seg0 = p.cu_seqlens[r];
    const int N = p.cu_seqlens[r + 1] - seg0;
    const int neff = min(p.query_window_n, N);
    const int i = static_cast<int>(t) - seg0;
    double acc = 0.0;
    const int pairs = p.num_heads * neff;
    for (int x = lane; x < pairs; x += 32) {
        const int h = x / neff, j = x - (x / neff) * neff;
        const int qpos = N - neff + j;
        if (i > qpos) continue;
        const __nv_bfloat16* qrow = p.q + static_cast<int64_t>(seg0 + qpos) * p.q_row_stride +
                                    static_cast<int64_t>(h) * p.head_dim;
        const __nv_bfloat16* krow = p.k + static_cast<int64_t>(seg0 + i) * p.k_row_stride +
                                    static_cast<int64_t>(kv_of(p, h)) * p.head_dim;
        const float s = dot_bf16(qrow, krow, p.head_dim) * p.scale;
        const int64_t idx = (static_cast<int64_t>(h) * p.num_requests + r) * p.simt_n + j;
        acc += static_cast<double>(expf(s - p.row_m[idx])) / static_cast<double>(p.row_l[idx]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) p.token_scores[t] = static_cast<float>(acc / static_cast<double>(neff));
}

__global__ void simt_block_kernel(const ScoreSimtParams p) {
    pdl_wait();     // predecessor's outputs are visible past this point
    pdl_trigger();  // let the dependent kernel's CTAs launch while this one runs
    const int R = p.num_requests;
    const int total = p.cu_blocks[R];
    for (int gb = blockIdx.x * blockDim.x + threadIdx.x; gb < total; gb += gridDim.x * blockDim.x) {
        const int r = find_segment(p.cu_blocks, R, gb);
        if (p.drop_enabled != nullptr && !p.drop_enabled[r]) {
            p.block_scores[gb] = 0.f;
            continue;
        }
        const int seg0 = p.cu_seqlens[r];
        const int N = p.cu_seqlens[r + 1] - seg0;
        const int g = gb - p.cu_blocks[r];
        const int b = g * p.block_size_g;
        const int e = min(N, b + p.block_size_g);
        double sum = 0.0;
        for (int i = b; i < e; ++i) sum += p.token_scores[seg0 + i];
        p.block_scores[gb] = static_cast<float>(sum / static_cast<double>(e - b));
    }
}

cudaError_t launch_score_simt(const ScoreSimtParams& p, int64_t max_tokens, int num_sms,
                              cudaStream_t stream) {
    const int rows_per_cta = 8;
    dim3 g1((p.simt_n + rows_per_cta - 1) / rows_per_cta, p.num_requests * p.num_heads);
    cudaError_t e = launch_k(kPdlScore, simt_row_stats_kernel, g1, rows_per_cta * 32, 0, stream, p);
    if (e != cudaSuccess) return e;
    const int64_t g2 = (max_tokens + 7) / 8;
    e = launch_k(kPdlScore, simt_token_kernel, static_cast<unsigned>(g2), 256, 0, stream, p, max_tokens);
    if (e != cudaSuccess) return e;
    return launch_k(kPdlScore, simt_block_kernel, num_sms * 2, 256, 0, stream, p);
}

}  // namespace up
