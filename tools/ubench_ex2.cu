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

int main_group();
int main(int argc, char**) {
    if (argc > 1) return main_group();
    for (int t : {256, 512, 1024}) {
        run("ex2.f32", k_f32, 1, t);
        run("ex2.f16x2", k_h2, 2, t);
        run("ex2.bf16x2", k_b2, 2, t);
    }
    return 0;
}

// ---- epilogue mix probe: the scorer's group sum (score_common.cuh) on register data ----
#include "../paper_2605_06221_b200/csrc/score_common.cuh"
template <int NP>
__global__ void __launch_bounds__(1024) k_group(float* out, float seed, long long* clk, int iters) {
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(seed * (threadIdx.x + c) * 1e-3f - 2.0f);
    const uint64_t sc2 = up::pk(1.0f, 1.0f);
    float acc = 0.f;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const float mm = -0.5f - static_cast<float>(i) * 1e-6f;  // varies per iteration: no hoisting
        acc += up::group_sum_pk<NP>(v, sc2, up::pk(mm, mm));
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int NP>
void run_group(int threads) {
    float* out; long long* clk;
    const int blocks = 148, iters = 2048;
    cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&clk, blocks * 8);
    k_group<NP><<<blocks, threads>>>(out, 1.f, clk, iters);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_group<NP><<<blocks, threads>>>(out, 1.f, clk, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double elems = double(blocks) * threads * iters * 32;
    printf("group_sum_pk<%d> threads=%d: %.2f elements/clk/SM (%.3f ms)\n", NP, threads,
           elems / (ms * 1e-3 * 1.965e9) / blocks, ms);
    cudaFree(out); cudaFree(clk);
}

int main_group() {
    for (int t : {256, 512, 768, 1024}) { run_group<0>(t); run_group<4>(t); run_group<6>(t); run_group<8>(t); }
    return 0;
}
