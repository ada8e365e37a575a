// ubench_ex2.cu -- throughput probe for the scorer's exp2 options on sm_100a (dev tool,
// not part of the product): ex2.approx.ftz.f32, ex2.approx.f16x2, ex2.approx.ftz.bf16x2,
// and the FMA-pipe polynomial.  Prints results per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_ex2 tools/ubench_ex2.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>

constexpr int ITERS = 4096;
constexpr int CH = 8;

__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }

__global__ void k_f32(float* out, float seed, long long* clk) {
    float v[CH];
    for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c) * 1e-6f - 0.5f;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) v[c] = ex2f(v[c]) - 1.5f;
    long long t1 = clock64();
    float s = 0; for (int c = 0; c < CH; ++c) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void k_h2(float* out, float seed, long long* clk) {
    uint32_t v[CH];
    for (int c = 0; c < CH; ++c) { __half2 h = __floats2half2_rn(seed * c * 1e-6f - 0.5f, -0.25f); v[c] = *reinterpret_cast<uint32_t*>(&h); }
    const __half2 k = __floats2half2_rn(-1.5f, -1.5f);
    const uint32_t ku = *reinterpret_cast<const uint32_t*>(&k);
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) { uint32_t y = ex2h2(v[c]); asm volatile("add.f16x2 %0, %1, %2;" : "=r"(v[c]) : "r"(y), "r"(ku)); }
    long long t1 = clock64();
    float s = 0; for (int c = 0; c < CH; ++c) s += __low2float(*reinterpret_cast<__half2*>(&v[c]));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void k_b2(float* out, float seed, long long* clk) {
    uint32_t v[CH];
    for (int c = 0; c < CH; ++c) { __nv_bfloat162 h = __floats2bfloat162_rn(seed * c * 1e-6f - 0.5f, -0.25f); v[c] = *reinterpret_cast<uint32_t*>(&h); }
    const __nv_bfloat162 k = __floats2bfloat162_rn(-1.5f, -1.5f);
    const uint32_t ku = *reinterpret_cast<const uint32_t*>(&k);
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) { uint32_t y = ex2b2(v[c]); asm volatile("add.bf16x2 %0, %1, %2;" : "=r"(v[c]) : "r"(y), "r"(ku)); }
    long long t1 = clock64();
    float s = 0; for (int c = 0; c < CH; ++c) s += __low2float(*reinterpret_cast<__nv_bfloat162*>(&v[c]));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int per_thread_results, int threads) {
    float* out; long long* clk;
    const int blocks = 148;
    cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&clk, blocks * 8);
    kern<<<blocks, threads>>>(out, 1.f, clk);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, 1.f, clk);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long c[148]; cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < blocks; ++i) avg += c[i]; avg /= blocks;
    const double results = double(threads) * ITERS * CH * per_thread_results;
    printf("%-10s threads=%4d  %.2f results/clk/SM (clock64), %.3f ms, %.1f Gresults/s/SM\n", name, threads,
           results / avg, ms, results / (ms * 1e6));
    cudaFree(out); cudaFree(clk);
}

int main() {
    for (int t : {256, 512, 1024}) {
        run("ex2.f32", k_f32, 1, t);
        run("ex2.f16x2", k_h2, 2, t);
        run("ex2.bf16x2", k_b2, 2, t);
    }
    return 0;
}
