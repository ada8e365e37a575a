// peer.cu -- the TP score all-reduce (Eq. 15; allreduce_scores,
// tp_sim.cpp:29-49) as ONE kernel over peer memory (NVLink P2P / NVSwitch), instead of an
// NCCL all-gather + a local reduce.  CTA c stores chunk c of this rank's partial into row
// `rank` of every peer's exchange buffer (16-byte-free plain P2P stores), then runs the
// rendezvous of peer.cuh and sums the tp rows of its chunk in ascending rank order --
// bitwise the reference's allreduce_scores, on every rank.  The fused variant (the block
// combine storing straight into the peers) is block_combine_peer_kernel in score_tc.cu.
#include <cuda_runtime.h>

#include "peer.cuh"

namespace up {

__global__ void __launch_bounds__(256) peer_allreduce_kernel(const PeerReduceParams p) {
    pdl_wait();
    const int c = blockIdx.x;
    const int64_t g0 = static_cast<int64_t>(c) * p.chunk < p.count ? static_cast<int64_t>(c) * p.chunk : p.count;
    const int64_t g1 = g0 + p.chunk < p.count ? g0 + p.chunk : p.count;
    __shared__ uint32_t s_epoch;
    if (threadIdx.x == 0) s_epoch = peer_epoch(p);
    __syncthreads();
    const int64_t row = peer_row_offset(p, s_epoch, p.rank);
    for (int t = 0; t < p.tp; ++t) {
        float* dst = p.peer_slots[t] + row;
        for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) dst[g] = p.partial[g];
    }
    peer_publish_and_wait(p, c, s_epoch);
    peer_sum_chunk(p, g0, g1, s_epoch);
    pdl_trigger();
    peer_epoch_advance(p);
}

int peer_grid(int num_sms) { return num_sms < kPeerMaxChunks ? num_sms : kPeerMaxChunks; }

cudaError_t launch_peer_allreduce(const PeerReduceParams& p, int grid, cudaStream_t stream) {
    return launch_k(kPdlSelect, peer_allreduce_kernel, static_cast<unsigned>(grid), 256, 0, stream, p);
}

}  // namespace up
