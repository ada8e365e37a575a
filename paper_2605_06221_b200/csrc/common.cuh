// common.cuh -- shared device helpers for the sm_100a UniPrefill kernels: workspace
// layout, sticky error flags, and thin inline-PTX wrappers for mbarrier, TMA
// (cp.async.bulk.tensor) and tcgen05 (MMA / TMEM).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

#include "../../include/uniprefill_b200.h"

namespace up {

// ---------------------------------------------------------------- error flags
// Sticky bits OR-ed into workspace word 0 by kernels; read by up_device_status().
enum : uint32_t {
    kErrBadScore = 1u,      // negative / non-finite block score (selection.cpp:62-66)
    kErrBadSeqlens = 2u,    // cu_seqlens not 0-based / strictly increasing / over capacity
    kErrTooManyBlocks = 4u, // a request has more blocks than the on-chip sort holds
    kErrMaskedRow = 8u,     // fully masked query row (importance.cpp:57-59)
    kErrAllocationMiss = 16u,  // slot for a page the block table does not hold (kvcache.cpp:71-78)
    kErrNoVisibleKey = 32u,    // attention row with no visible key (model.cpp:237)
    kErrPeerTimeout = 64u,     // a TP peer's partial scores never arrived (peer.cu)
};

constexpr int kMaxSortBlocks = 16384;  // per-request blocks the select kernel sorts on chip
constexpr int kTileKeys = 128;          // keys per tcgen05 S tile (UMMA N)
constexpr int kUsidParShift = 28;       // unit_sid: item id below, statistics parity above (score_common.cuh)
constexpr int kRows = 128;              // query rows per S tile (UMMA M) -> max n for tcgen05

// Workspace carve-up (byte offsets), identical on host and device.
struct Workspace {
    uint32_t* err;         // [0] sticky error bits
    int32_t* plan;         // [0]=chunk_keys [1]=total_items [2]=num_hgroups
    int32_t* cu_chunks;    // [R+1]
    int32_t* cu_items;     // [R+1]
    float* P;              // [Hq][max_blocks][128]  per-(row, block) partial exp sums
    float* stat_m;         // [Hq][max_chunks][128]  per-(row, chunk) reference max (log2 units)
    float* stat_l;         // [Hq][max_chunks][128]  per-(row, chunk) partial denominator
    float* stat_w;         // [Hq][max_chunks][128]  per-(row, chunk) final weight
    float* simt_m;         // [Hq][R][n]  SIMT path row max
    float* simt_l;         // [Hq][R][n]  SIMT path row denominator
    int32_t* tile_counts;  // [num_compact_tiles]
    int64_t max_blocks;
    int64_t max_chunks;
    int32_t simt_n;
};

__device__ __forceinline__ void raise_error(uint32_t* err, uint32_t bit) { atomicOr(err, bit); }

// ---------------------------------------------------------------- launches (PDL)
// Programmatic dependent launch: every kernel of the path is launched with
// programmatic stream serialization, so the next kernel's CTAs are scheduled while the
// current one drains; each kernel calls pdl_wait() before touching its predecessor's
// outputs (a no-op when launched without the attribute) and pdl_trigger() to let its own
// dependent launch early.  Which kernel families are launched that way is the mask below.
#ifndef UP_PDL_DEFAULT_MASK
#define UP_PDL_DEFAULT_MASK 11  // compaction launches without PDL: measured 7% slower on the 64-request stream
#endif
constexpr int kPdlDefaultMask = UP_PDL_DEFAULT_MASK;
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Kernel families for the PDL policy (UP_PDL_MASK bit per family; default all).
enum PdlFamily : int { kPdlScore = 1, kPdlSelect = 2, kPdlCompact = 4, kPdlMeta = 8, kPdlCompactScan = 16 };

inline int pdl_mask() {
    static const int m = [] {
        const char* s = std::getenv("UP_PDL_MASK");
        return s ? std::atoi(s) : kPdlDefaultMask;
    }();
    return m;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(int family, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_mask() & family) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
        "r"(bytes)
        : "memory");
}

// Variants on a precomputed shared::cta address (hot loops: no per-call address math).
__device__ __forceinline__ void mbar_wait_u32(uint32_t addr, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_u32(uint32_t addr) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(addr)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(phase)
        : "memory");
}

// Generic-proxy shared-memory writes -> visible to the async proxy (TMA, tcgen05.mma).
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 2-D TMA tile load global -> shared, completing on an mbarrier (transaction bytes).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t x, int32_t y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// Same with an L2 cache policy (createpolicy): K tiles are read exactly once, so they are
// loaded evict-first and do not push the scorer's P partials out of L2 before the combine.
__device__ __forceinline__ void tma_load_2d_hint(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                                 int32_t x, int32_t y, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---- tcgen05 -----------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate, single CTA.
__device__ __forceinline__ void mma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]^T: A (M = 128 rows = TMEM lanes, K along 32-bit columns,
// two bf16 per column) read from tensor memory.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Arrive on an mbarrier once every previously issued tcgen05 op of this thread completes.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 32 consecutive 32-bit TMEM columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

// 32 lanes x 16 consecutive 32-bit TMEM columns -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// 32 registers per thread -> 32 lanes x 32 consecutive 32-bit TMEM columns.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// 16 registers per thread -> 32 lanes x 16 consecutive 32-bit TMEM columns.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor for a K-major bf16 operand in the canonical
// SWIZZLE_128B layout written by TMA: 8-row x 128-byte swizzle atoms, atoms of
// consecutive rows 1024 bytes apart (SBO), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);  // start address
    d |= static_cast<uint64_t>(1) << 16;                       // LBO (unused for SW128 K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;               // SBO
    d |= static_cast<uint64_t>(1) << 46;                       // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2) << 61;                       // SWIZZLE_128B
    return d;
}

// Same for an MN-major operand (N contiguous, e.g. V [keys][D] as the B of P·V) in the
// SWIZZLE_128B layout TMA writes for 64-element-wide boxes: 64 N-elements per 128-byte
// row, K rows 128 bytes apart, 8-row atoms SBO bytes apart, 64-wide N chunks LBO apart.
__device__ __forceinline__ uint64_t smem_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// Instruction descriptor: kind::f16, A=B=bf16, D=f32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
    return (1u << 4)                                  // D format f32
           | (1u << 7)                                // A format bf16
           | (1u << 10)                               // B format bf16
           | (static_cast<uint32_t>(N >> 3) << 17)    // N / 8
           | (static_cast<uint32_t>(M >> 4) << 24);   // M / 16
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---- packed fp32 pairs (FFMA2 / FADD2 on sm_100a) ---------------------------------
__device__ __forceinline__ uint64_t pk(float lo, float hi) {
    return static_cast<uint64_t>(__float_as_uint(lo)) | (static_cast<uint64_t>(__float_as_uint(hi)) << 32);
}
__device__ __forceinline__ float lo_f(uint64_t x) { return __uint_as_float(static_cast<uint32_t>(x)); }
__device__ __forceinline__ float hi_f(uint64_t x) { return __uint_as_float(static_cast<uint32_t>(x >> 32)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// 2^x for a pair on the FMA pipe (offloads MUFU): x clamped to [-126, 64]; round-to-
// nearest split x = j + f via the 1.5*2^23 magic number, degree-3 minimax polynomial for
// 2^f on [-0.5, 0.5] (max relative error 7.5e-5), exponent added into the bits.  Values
// below 2^-126 of the reference come out as denormal-small positives (negligible against
// the >= 1 row mass); x >= 40 can only occur when the reference must move (rebase).
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
    const float x0 = fminf(fmaxf(lo_f(x), -126.f), 64.f);
    const float x1 = fminf(fmaxf(hi_f(x), -126.f), 64.f);
    const uint64_t xc = pk(x0, x1);
    const uint64_t t = add2(xc, pk(12582912.f, 12582912.f));     // j + 1.5*2^23
    const uint64_t j = add2(t, pk(-12582912.f, -12582912.f));    // j
    const uint64_t f = fma2(j, pk(-1.f, -1.f), xc);               // x - j in [-0.5, 0.5]
    uint64_t p = fma2(pk(0.05517162704803067f, 0.05517162704803067f), f,
                      pk(0.2426111716750347f, 0.2426111716750347f));
    p = fma2(p, f, pk(0.693260997791971f, 0.693260997791971f));
    p = fma2(p, f, pk(0.9999280708313836f, 0.9999280708313836f));
    // exponent insert per lane (32-bit shift-adds; kept out of a fused 64-bit add with carry)
    uint32_t r0, r1;
    asm("{\n\t.reg .u32 s;\n\t"
        "shl.b32 s, %2, 23;\n\tadd.u32 %0, s, %3;\n\t"
        "shl.b32 s, %4, 23;\n\tadd.u32 %1, s, %5;\n\t}"
        : "=r"(r0), "=r"(r1)
        : "r"(static_cast<uint32_t>(t)), "r"(static_cast<uint32_t>(p)), "r"(static_cast<uint32_t>(t >> 32)),
          "r"(static_cast<uint32_t>(p >> 32)));
    return static_cast<uint64_t>(r0) | (static_cast<uint64_t>(r1) << 32);
}

// Binary search: largest s in [0, R) with cu[s] <= x (cu is non-decreasing, cu[0] = 0).
// PackedBatch::validate (scheduler.cpp:33-48) on the device, plus the capacity bound:
// cu[0] == 0, strictly increasing, cu[R] <= max_tokens.  Every thread of the CTA calls it
// (one __syncthreads_and); kernels that index by segment return early on false so a
// malformed batch never reads or writes past its buffers.
__device__ __forceinline__ bool cta_batch_valid(const int32_t* cu, int R, int64_t max_tokens) {
    bool ok = true;
    for (int r = threadIdx.x; r < R; r += blockDim.x) ok = ok && cu[r + 1] > cu[r];
    if (threadIdx.x == 0) ok = ok && cu[0] == 0 && static_cast<int64_t>(cu[R]) <= max_tokens;
    return __syncthreads_and(ok) != 0;
}

__device__ __forceinline__ int find_segment(const int32_t* cu, int R, int64_t x) {
    int lo = 0, hi = R - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cu[mid] <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

}  // namespace up
