// ubench_tmem.cu -- TMEM read throughput on sm_100a (dev probe, not product): W warps per
// CTA, one CTA per SM, each warp repeatedly tcgen05.ld.32x32b.x32 (its lane quarter, 32
// columns = 4 KB per warp-instruction) with 1 or 2 loads in flight; prints bytes/clk/SM.
// The scorer's epilogue reads every fp32 S element from TMEM once, so this rate / 4 B is
// an upper bound on its elements per clock, next to MUFU's 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_06221_b200/csrc -o tools/_bin/ubench_tmem tools/ubench_tmem.cu
#include <cstdio>
#include "common.cuh"

using namespace up;

template <int INFLIGHT>
__global__ void k_tmem(float* out, long long* clk, int iters) {
    __shared__ uint32_t s_base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&s_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t base = s_base + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t col0 = static_cast<uint32_t>((warp >> 2) * 32) % 512;
    float acc = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t a[32], b[32];
        tmem_ld32(base + col0, a);
        if (INFLIGHT > 1) tmem_ld32(base + ((col0 + 256) % 512), b);
        tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
            acc += __uint_as_float(a[k]);
            acc1 += __uint_as_float(a[k + 1]);
            acc2 += __uint_as_float(a[k + 2]);
            acc3 += __uint_as_float(a[k + 3]);
        }
        if (INFLIGHT > 1) {
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
                acc += __uint_as_float(b[k]);
                acc1 += __uint_as_float(b[k + 1]);
                acc2 += __uint_as_float(b[k + 2]);
                acc3 += __uint_as_float(b[k + 3]);
            }
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = (acc + acc1) + (acc2 + acc3);
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(s_base, 512);
    }
}

template <int INFLIGHT>
void run(int warps) {
    const int blocks = 148, iters = 4096;
    float* out;
    long long* clk;
    cudaMalloc(&out, blocks * warps * 32 * 4);
    cudaMalloc(&clk, blocks * 8);
    k_tmem<INFLIGHT><<<blocks, warps * 32>>>(out, clk, iters);
    k_tmem<INFLIGHT><<<blocks, warps * 32>>>(out, clk, iters);
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < blocks; ++i) avg += c[i];
    avg /= blocks;
    const double bytes = double(warps) * iters * INFLIGHT * 32 * 32 * 4;  // per CTA
    printf("tcgen05.ld 32x32b.x32, %2d warps, %d in flight: %.1f B/clk/SM = %.1f fp32 elements/clk/SM (%s)\n", warps,
           INFLIGHT, bytes / avg, bytes / avg / 4, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<1>(w);
        run<2>(w);
    }
    return 0;
}
