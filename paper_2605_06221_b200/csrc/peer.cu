// peer.cu -- the TP score all-reduce (Eq. 15; allreduce_scores,
// tp_sim.cpp:29-49) as ONE kernel over peer memory (NVLink P2P / NVSwitch), instead of an
// NCCL all-gather + a local reduce.
//
// Every rank r owns an exchange buffer slots_r = float[tp][capacity] and a flag array
// flags_r = uint32[kPeerMaxChunks] (both zeroed once, mapped into every peer with CUDA IPC).
// CTA c of rank r handles chunk c of the partial block-score vector:
//   1. store partial[chunk c] into row r of every peer's slots (16-byte P2P stores),
//   2. __syncthreads, system fence, flags_t[c] += 1 on every peer t (release),
//   3. wait until its own flags_r[c] reaches (epoch + 1) * tp (acquire): all tp ranks'
//      rows of chunk c have landed in slots_r,
//   4. out[g] = ((0 + slots_r[0][g]) + slots_r[1][g]) + ... in ascending rank order --
//      bitwise the reference's allreduce_scores, on every rank.
// The flags are monotonic counters; each rank keeps a device epoch counter that the last
// CTA of a launch advances, so a captured CUDA graph can replay the reduction.  A CTA only
// waits for the SAME chunk of the other ranks, never for another CTA of its own grid, and
// the grid is one CTA per SM (fixed, so every flag advances by tp per call), so there is
// no intra-GPU deadlock.  A wait that exceeds ~2 s raises kErrPeerTimeout and gives up
// (the sticky device status reports it).
#include <cuda_runtime.h>

#include "common.cuh"
#include "params.cuh"

namespace up {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(256) peer_allreduce_kernel(const PeerReduceParams p) {
    pdl_wait();
    const int c = blockIdx.x;
    const int64_t g0 = static_cast<int64_t>(c) * p.chunk < p.count ? static_cast<int64_t>(c) * p.chunk : p.count;
    const int64_t g1 = g0 + p.chunk < p.count ? g0 + p.chunk : p.count;
    __shared__ uint32_t s_epoch;
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint32_t*>(p.epoch);
    // 1. this rank's chunk into row `rank` of every peer's exchange buffer
    for (int t = 0; t < p.tp; ++t) {
        float* dst = p.peer_slots[t] + static_cast<int64_t>(p.rank) * p.capacity;
        for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) dst[g] = p.partial[g];
    }
    __syncthreads();
    const uint32_t target = (s_epoch + 1u) * static_cast<uint32_t>(p.tp);
    if (threadIdx.x == 0) {
        // 2. publish: the CTA's stores (ordered before by bar.sync) then the flags
        __threadfence_system();
        for (int t = 0; t < p.tp; ++t) atomicAdd_system(p.peer_flags[t] + c, 1u);
        // 3. wait for every rank's row of this chunk
        const long long t0 = clock64();
        while (ld_acquire_sys(p.flags + c) < target) {
            if (clock64() - t0 > (4ll << 30)) {  // ~2 s at 1.9 GHz
                raise_error(p.err, kErrPeerTimeout);
                break;
            }
            __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
    // 4. ascending-rank fp32 sum from 0.0f (tp_sim.cpp:43-47)
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) {
        float acc = 0.0f;
        for (int t = 0; t < p.tp; ++t) acc = __fadd_rn(acc, __ldcg(p.slots + static_cast<int64_t>(t) * p.capacity + g));
        p.out[g] = acc;
    }
    pdl_trigger();
    // the last CTA advances this rank's epoch for the next launch (stream-ordered)
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t done = atomicAdd(p.epoch + 1, 1u);
        if (done == gridDim.x - 1) {
            p.epoch[1] = 0;
            __threadfence();
            atomicAdd(p.epoch, 1u);
        }
    }
}

cudaError_t launch_peer_allreduce(const PeerReduceParams& p, int grid, cudaStream_t stream) {
    return launch_k(kPdlSelect, peer_allreduce_kernel, static_cast<unsigned>(grid), 256, 0, stream, p);
}

}  // namespace up
