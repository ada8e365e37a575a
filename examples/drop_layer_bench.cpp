// drop_layer_bench.cpp -- the hot path driven from C++ only: the host mirror
// (include/uniprefill_b200.hpp) over the C ABI, no Python anywhere.  What an engine written
// in C++ (the reference's Engine::run_batch, scheduler.cpp:293-332) does at its drop layers:
//
//   for every drop layer:  score_blocks -> top_p_select -> compact_selected   (one CUDA stream)
//
// The layer loop is captured once into a CUDA graph and replayed; prints one JSON line
// with tokens/s over the timed replays.  Synthetic activations ("planted" regime of
// paper_2605_06221_b200/synthetic.py: a per-kv-head direction added to every query and to
// the keys of ~25% of the blocks) are generated on the host once and reused by every layer
// (each set is far larger than the 126 MB L2).
//
//   make -C examples && examples/_build/drop_layer_bench --requests 4 --len 32768 --layers 32
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "uniprefill_b200.hpp"

namespace b2 = uniprefill::b200;

static void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
        std::exit(2);
    }
}

struct Rng {  // splitmix64 + Box-Muller
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
    float normal() {
        const double u1 = uniform() + 1e-300, u2 = uniform();
        return static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2));
    }
};

int main(int argc, char** argv) {
    int R = 4, N = 32768, layers = 32, steps = 5, warmup = 3;
    int Hq = 32, Hkv = 8, D = 128, hidden = 4096;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string a = argv[i];
        const int v = std::atoi(argv[i + 1]);
        if (a == "--requests") R = v;
        else if (a == "--len") N = v;
        else if (a == "--layers") layers = v;
        else if (a == "--steps") steps = v;
        else if (a == "--warmup") warmup = v;
        else if (a == "--q-heads") Hq = v;
        else if (a == "--kv-heads") Hkv = v;
        else if (a == "--head-dim") D = v;
        else if (a == "--hidden") hidden = v;
    }
    const int64_t T = int64_t(R) * N;
    const int group = Hq / Hkv;
    b2::ScoreConfig cfg;  // SPEC defaults: n=128, G=64, A=128, p=0.99
    cfg.validate();

    // ---- synthetic planted activations (host), uploaded once ----
    Rng rng{1234};
    std::vector<float> dir(size_t(Hkv) * D);
    for (auto& x : dir) x = rng.normal();
    const float gamma = 0.8f;
    std::vector<__nv_bfloat16> q(size_t(T) * Hq * D), k(size_t(T) * Hkv * D), v(size_t(T) * Hkv * D),
        hid(size_t(T) * hidden);
    std::vector<int64_t> pos(T);
    std::vector<uint8_t> hot(static_cast<size_t>(T));
    for (int r = 0; r < R; ++r)
        for (int g = 0; g * 64 < N; ++g) {
            const uint8_t h = rng.uniform() < 0.25 ? 1 : 0;
            for (int i = g * 64; i < N && i < (g + 1) * 64; ++i) hot[size_t(r) * N + i] = h;
        }
    for (int64_t t = 0; t < T; ++t) {
        pos[t] = t % N;
        for (int h = 0; h < Hq; ++h)
            for (int d = 0; d < D; ++d)
                q[(size_t(t) * Hq + h) * D + d] = __float2bfloat16(rng.normal() + gamma * dir[size_t(h / group) * D + d]);
        for (int h = 0; h < Hkv; ++h)
            for (int d = 0; d < D; ++d) {
                k[(size_t(t) * Hkv + h) * D + d] =
                    __float2bfloat16(rng.normal() + (hot[t] ? gamma * dir[size_t(h) * D + d] : 0.f));
                v[(size_t(t) * Hkv + h) * D + d] = __float2bfloat16(rng.normal());
            }
        for (int d = 0; d < hidden; d += 8) {  // hidden content does not affect the path
            const float x = rng.normal();
            for (int e = 0; e < 8; ++e) hid[size_t(t) * hidden + d + e] = __float2bfloat16(x);
        }
    }
    std::vector<int32_t> cu(R + 1);
    for (int r = 0; r <= R; ++r) cu[r] = r * N;

    auto upload = [](const void* h, size_t bytes) {
        void* d = nullptr;
        cuda_check(cudaMalloc(&d, bytes), "cudaMalloc");
        cuda_check(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice), "upload");
        return d;
    };
    auto alloc = [](size_t bytes) {
        void* d = nullptr;
        cuda_check(cudaMalloc(&d, bytes), "cudaMalloc");
        return d;
    };
    void* d_q = upload(q.data(), q.size() * 2);
    void* d_k = upload(k.data(), k.size() * 2);
    void* d_v = upload(v.data(), v.size() * 2);
    void* d_h = upload(hid.data(), hid.size() * 2);
    void* d_pos = upload(pos.data(), pos.size() * 8);
    auto* d_cu = static_cast<int32_t*>(upload(cu.data(), cu.size() * 4));

    b2::VarlenBatch batch{R, T, d_cu, nullptr};
    b2::HeadLayout heads{Hq, Hkv, D, group};
    b2::Workspace ws(batch, heads, cfg);
    const up_batch bc = batch.c();
    const up_score_config cc = cfg.c();
    const int64_t nb = up_max_blocks(&bc, &cc);
    auto* d_bs = static_cast<float*>(alloc(nb * 4));
    auto* d_cub = static_cast<int32_t*>(alloc((R + 1) * 4));
    auto* d_keep = static_cast<uint8_t*>(alloc(T));
    auto* d_cut = static_cast<int64_t*>(alloc(R * 8));
    auto* d_cu_out = static_cast<int32_t*>(alloc((R + 1) * 4));
    auto* d_idx = static_cast<int32_t*>(alloc(T * 4));
    auto* d_nout = static_cast<int32_t*>(alloc(4));
    void* o_h = alloc(size_t(T) * hidden * 2);
    void* o_k = alloc(size_t(T) * Hkv * D * 2);
    void* o_v = alloc(size_t(T) * Hkv * D * 2);
    void* o_p = alloc(size_t(T) * 8);
    const std::vector<up_plane> planes = {
        {d_h, o_h, int64_t(hidden) * 2, 0, 0},
        {d_k, o_k, int64_t(Hkv) * D * 2, 0, 0},
        {d_v, o_v, int64_t(Hkv) * D * 2, 0, 0},
        {d_pos, o_p, 8, 0, 0},
    };

    cudaStream_t s;
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    int launches = 0;
    auto layer = [&]() {
        b2::score_blocks(s, batch, heads, cfg, d_q, d_k, d_bs, d_cub, ws);
        launches += up_last_launch_count();
        b2::top_p_select(s, batch, cfg, d_bs, d_cub, d_keep, up_selection_out{d_cut, nullptr, nullptr, nullptr}, ws);
        launches += up_last_launch_count();
        // the keep mask is top_p_select's output on this workspace: its tile counts are reused
        b2::compact_selected(s, batch, d_keep, planes, d_cu_out, d_idx, d_nout, ws);
        launches += up_last_launch_count();
        // block boundary (a LLaMA block = [attention (drop), FFN]): reconstitute the residual
        // stream -- the retained rows' current states back over their pre-drop rows
        // (reconstitute, propagation.cpp:79-100; scheduler.cpp:349-360)
        b2::scatter_rows(s, d_idx, d_nout, T, {up_plane{o_h, d_h, int64_t(hidden) * 2, 0, 0}});
        launches += up_last_launch_count();
    };
    layer();
    b2::check_device(s, ws);  // ContractViolation -> exception
    const int launches_per_layer = launches;

    cudaGraph_t graph;
    cudaGraphExec_t exec;
    cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal), "capture");
    for (int l = 0; l < layers; ++l) layer();
    cuda_check(cudaStreamEndCapture(s, &graph), "end capture");
    cuda_check(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
    for (int i = 0; i < warmup; ++i) cuda_check(cudaGraphLaunch(exec, s), "warmup");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cuda_check(cudaStreamSynchronize(s), "sync");
    cudaEventRecord(e0, s);
    for (int i = 0; i < steps; ++i) cuda_check(cudaGraphLaunch(exec, s), "replay");
    cudaEventRecord(e1, s);
    cuda_check(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    b2::check_device(s, ws);
    int32_t nout = 0;
    cudaMemcpy(&nout, d_nout, 4, cudaMemcpyDeviceToHost);
    const double step_ms = ms / steps;
    std::printf("{\"driver\": \"c++ (uniprefill_b200.hpp)\", \"requests\": %d, \"tokens_per_request\": %d, "
                "\"drop_layers\": %d, \"ms_per_step\": %.4f, \"us_per_layer\": %.2f, \"tokens_per_s\": %.6e, "
                "\"retention_rho\": %.4f, \"launches_per_layer\": %d}\n",
                R, N, layers, step_ms, step_ms * 1e3 / layers, double(T) * layers / (step_ms / 1e3),
                double(nout) / double(T), launches_per_layer);
    return 0;
}
