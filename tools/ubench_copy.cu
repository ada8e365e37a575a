// ubench_copy.cu -- dev probe: HBM bandwidth of row-gather copies on sm_100a (not product
// code).  Gathers `rows` rows of `rb` bytes (every 4th source row) and reports GB/s
// (read + write) for
//   (1) warp-per-row 16-byte vector copy, 8 vectors in flight per lane (compact.cu style);
//   (2) TMA bulk copies (cp.async.bulk global->smem->global), one thread per CTA driving a
//       ring of smem slots;
//   (3) cudaMemcpyAsync D2D of the same byte count (contiguous), for reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_copy tools/ubench_copy.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_warp(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                              const int* __restrict__ idx, int rows, int64_t rb) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * 256 + threadIdx.x) >> 5, nw = (gridDim.x * 256) >> 5;
    for (int o = gw; o < rows; o += nw) {
        const int4* s = reinterpret_cast<const int4*>(src + int64_t(idx[o]) * rb);
        int4* d = reinterpret_cast<int4*>(dst + int64_t(o) * rb);
        const int64_t nv = rb >> 4;
        for (int64_t v = lane; v < nv; v += 8 * 32) {
            int4 x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (v + u * 32 < nv) x[u] = __ldcs(s + v + u * 32);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (v + u * 32 < nv) __stcs(d + v + u * 32, x[u]);
        }
    }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int SLOTS, int SLOT_BYTES>
__global__ void __launch_bounds__(32) k_bulk(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                             const int* __restrict__ idx, int rows, int rb) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[SLOTS];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < SLOTS; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int per_slot = SLOT_BYTES / rb;  // rows per slot
    constexpr int AHEAD = SLOTS / 2;       // batches whose loads are in flight ahead of the stores
    uint32_t phase[SLOTS] = {};
    // rows of this CTA: contiguous range, in batches of per_slot rows
    const int64_t r0 = int64_t(rows) * blockIdx.x / gridDim.x, r1 = int64_t(rows) * (blockIdx.x + 1) / gridDim.x;
    const int nbat = int((r1 - r0 + per_slot - 1) / per_slot);
    for (int i = 0; i < nbat + AHEAD; ++i) {
        if (i < nbat) {  // loads of batch i into slot i % SLOTS
            const int s = i % SLOTS;
            // the slot's previous store (batch i - SLOTS) must have read its smem: at most
            // SLOTS - AHEAD - 1 newer store groups may still be pending
            if (i >= SLOTS) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(SLOTS - AHEAD - 1) : "memory");
            const int64_t base = r0 + int64_t(i) * per_slot;
            const int n = int(r1 - base < per_slot ? r1 - base : per_slot);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(n * rb) : "memory");
            for (int k = 0; k < n; ++k)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(smem + s * SLOT_BYTES + k * rb)), "l"(src + int64_t(idx[base + k]) * rb), "r"(rb),
                             "r"(su32(&bar[s]))
                             : "memory");
        }
        const int j = i - AHEAD;
        if (j >= 0) {  // store batch j once its loads landed
            const int s = j % SLOTS;
            asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}"
                         ::"r"(su32(&bar[s])), "r"(phase[s]) : "memory");
            phase[s] ^= 1;
            const int64_t base = r0 + int64_t(j) * per_slot;
            const int n = int(r1 - base < per_slot ? r1 - base : per_slot);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(dst + base * rb), "r"(su32(smem + s * SLOT_BYTES)), "r"(n * rb) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int rb = 8192;
    const int rows = 131072 / 4;  // retained rows of a 4x32K batch at rho = 0.25
    const int64_t src_rows = int64_t(rows) * 4;
    uint8_t *src, *dst;
    int* idx;
    cudaMalloc(&src, src_rows * rb);
    cudaMalloc(&dst, int64_t(rows) * rb);
    cudaMalloc(&idx, rows * 4);
    int* h = new int[rows];
    for (int i = 0; i < rows; ++i) h[i] = i * 4 + (i % 3);
    cudaMemcpy(idx, h, rows * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = 2.0 * rows * rb;
    auto report = [&](const char* name, float ms) { printf("%-28s %.1f us  %.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e6)); };
    for (int occ : {4, 8}) {
        for (int it = 0; it < 2; ++it) {
            cudaEventRecord(a);
            k_warp<<<148 * occ, 256>>>(src, dst, idx, rows, rb);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it) report(occ == 4 ? "warp-per-row (4 CTA/SM)" : "warp-per-row (8 CTA/SM)", ms);
        }
    }
    {
        constexpr int SLOTS = 4, SB = 32768;
        cudaFuncSetAttribute(k_bulk<SLOTS, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SLOTS * SB);
        for (int ctas : {148, 296, 592}) {
            for (int it = 0; it < 2; ++it) {
                cudaEventRecord(a);
                k_bulk<SLOTS, SB><<<ctas, 32, SLOTS * SB>>>(src, dst, idx, rows, rb);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                char nm[64];
                snprintf(nm, 64, "TMA bulk 4x32KB (%d CTAs)", ctas);
                if (it) report(nm, ms);
            }
        }
    }
    {
        constexpr int SLOTS = 8, SB = 24576;
        cudaFuncSetAttribute(k_bulk<SLOTS, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SLOTS * SB);
        for (int ctas : {148, 296}) {
            for (int it = 0; it < 2; ++it) {
                cudaEventRecord(a);
                k_bulk<SLOTS, SB><<<ctas, 32, SLOTS * SB>>>(src, dst, idx, rows, rb);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                char nm[64];
                snprintf(nm, 64, "TMA bulk 8x24KB (%d CTAs)", ctas);
                if (it) report(nm, ms);
            }
        }
    }
    for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        cudaMemcpyAsync(dst, src, int64_t(rows) * rb, cudaMemcpyDeviceToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it) report("cudaMemcpy D2D (contiguous)", ms);
    }
    printf("check: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
