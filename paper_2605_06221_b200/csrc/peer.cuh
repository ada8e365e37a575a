// peer.cuh -- device side of the TP rendezvous over peer memory (used by peer.cu's
// stand-alone all-reduce and by the fused combine + all-reduce in score_tc.cu).
//
// Every rank owns an exchange buffer [epoch[2] | flags[kPeerMaxChunks] | slots[2][tp][capacity]]
// mapped into all peers (CUDA IPC).  A launch uses a FIXED grid of peer_grid() CTAs on every
// rank; CTA c owns chunk c of the vector:
//   1. (caller) stores its values of chunk c into row `rank` of bank (epoch & 1) of every
//      peer's slots,
//   2. peer_publish_and_wait: bar.sync, system fence, flags_t[c] += 1 on every peer t, then
//      spin (acquire) until its own flags[c] reaches (epoch + 1) * tp,
//   3. peer_sum_chunk: out[g] = ((0 + slots[0][g]) + slots[1][g]) + ... ascending rank,
//   4. peer_epoch_advance: the last CTA of the launch advances this rank's epoch.
// The flags are monotonic; since every launch bumps every flag once per rank, the targets
// follow from the device epoch alone (CUDA-graph replayable).
// Two banks by epoch parity close the write-after-read window: rank A's launch e+1 may
// store into a peer B while B is still summing launch e (B passed its wait, A finished e
// and moved on) -- but e+1 writes the other bank.  A cannot reach e+2 (the bank B may
// still read) before every peer published for e+1, and a peer publishes for e+1 only
// after its launch e -- including the sum -- completed (stream order + pdl_wait).  A CTA waits only for the
// same chunk of the other ranks, and the grid is co-resident, so no intra-GPU deadlock.
#pragma once
#include "common.cuh"
#include "params.cuh"

namespace up {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Thread 0 of the CTA reads the epoch (before any flag of this launch can move it); the
// caller makes it visible to the CTA (__syncthreads) before any store to a peer.
__device__ __forceinline__ uint32_t peer_epoch(const PeerReduceParams& p) {
    return *reinterpret_cast<volatile uint32_t*>(p.epoch);
}

// Offset of row `row` of the bank this launch uses, in any rank's slots.
__device__ __forceinline__ int64_t peer_row_offset(const PeerReduceParams& p, uint32_t epoch, int row) {
    return (static_cast<int64_t>(epoch & 1u) * p.tp + row) * p.capacity;
}

// All threads: the CTA's stores to the peers are done (program order before the call).
__device__ __forceinline__ void peer_publish_and_wait(const PeerReduceParams& p, int c, uint32_t epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int t = 0; t < p.tp; ++t) atomicAdd_system(p.peer_flags[t] + c, 1u);
        const uint32_t target = (epoch + 1u) * static_cast<uint32_t>(p.tp);
        const long long t0 = clock64();
        while (ld_acquire_sys(p.flags + c) < target) {
            if (clock64() - t0 > (4ll << 30)) {  // ~2 s at 1.9 GHz: a peer never arrived
                raise_error(p.err, kErrPeerTimeout);
                break;
            }
            __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// out[g] for g in [g0, g1): ascending-rank fp32 sum from 0.0f (tp_sim.cpp:43-47).
__device__ __forceinline__ void peer_sum_chunk(const PeerReduceParams& p, int64_t g0, int64_t g1, uint32_t epoch) {
    const float* bank = p.slots + peer_row_offset(p, epoch, 0);
    for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) {
        float acc = 0.0f;
        for (int t = 0; t < p.tp; ++t) acc = __fadd_rn(acc, __ldcg(bank + static_cast<int64_t>(t) * p.capacity + g));
        p.out[g] = acc;
    }
}

__device__ __forceinline__ void peer_epoch_advance(const PeerReduceParams& p) {
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

}  // namespace up
