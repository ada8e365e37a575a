// test_parity.cpp -- C++ parity tests through the host mirror (include/uniprefill_b200.hpp),
// written like the reference's own doctest cases (/root/reference/proj/tests/*.cpp) and
// checked against the UNMODIFIED reference (oracle/_ref/libuniprefill_ref.so, extern "C"
// shim in oracle/ref_shim.cpp).  Built by __graft_entry__.build(); run by
// tests/test_gpu_cpp.py on a GPU.  Test infrastructure only.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "uniprefill_b200.hpp"

extern "C" {
struct RefScoreConfig { int32_t query_window_n, block_size_g, sink_count_a; float top_p; };
struct RefSelectionInfo { int64_t cutoff_rank, retained_count; double retention_ratio, covered_mass; int32_t degenerate_keep_all; };
int ref_top_p_select(const float*, int64_t, const RefScoreConfig*, int64_t, uint8_t*, RefSelectionInfo*);
int ref_score_tokens_heads(const float*, int64_t, const float*, int64_t, int64_t, int, int, int, int, int,
                           const RefScoreConfig*, float*, float*, int32_t*);
int ref_attention_readout(const float*, const int64_t*, int64_t, const float*, const float*, const int64_t*, int64_t,
                          int, int, int, int64_t, float*);
}

namespace b2 = uniprefill::b200;

static int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                                \
    do {                                                                           \
        ++g_checks;                                                                \
        if (!(cond)) {                                                             \
            ++g_failed;                                                            \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                          \
    } while (0)
#define TEST_CASE(name) static void name()

template <class T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    explicit Dev(size_t count) : n(count) { cudaMalloc(&p, sizeof(T) * (count ? count : 1)); }
    Dev(const std::vector<T>& h) : Dev(h.size()) { cudaMemcpy(p, h.data(), sizeof(T) * n, cudaMemcpyHostToDevice); }
    ~Dev() { cudaFree(p); }
    std::vector<T> get(size_t count) const {
        std::vector<T> h(count);
        cudaMemcpy(h.data(), p, sizeof(T) * count, cudaMemcpyDeviceToHost);
        return h;
    }
};

struct GpuSelection {
    std::vector<uint8_t> keep;
    int64_t cutoff;
    double covered;
};

static GpuSelection gpu_select(const std::vector<float>& scores, int64_t N, const b2::ScoreConfig& cfg) {
    Dev<float> bs(scores);
    const int64_t nb = (N + cfg.block_size_g - 1) / cfg.block_size_g;
    Dev<int32_t> cu(std::vector<int32_t>{0, static_cast<int32_t>(N)});
    Dev<int32_t> cub(std::vector<int32_t>{0, static_cast<int32_t>(nb)});
    Dev<uint8_t> keep(N);
    Dev<int64_t> cutoff(1), retained(1);
    Dev<double> covered(1);
    Dev<uint8_t> degen(1);
    b2::VarlenBatch b{1, N, cu.p, nullptr};
    b2::Workspace ws(b, b2::HeadLayout{1, 1, 64}, cfg);
    up_selection_out out{cutoff.p, retained.p, covered.p, degen.p};
    b2::top_p_select(nullptr, b, cfg, bs.p, cub.p, keep.p, out, ws);
    b2::check_device(nullptr, ws);
    return {keep.get(N), cutoff.get(1)[0], covered.get(1)[0]};
}

static GpuSelection ref_select(const std::vector<float>& scores, int64_t N, const b2::ScoreConfig& cfg) {
    RefScoreConfig rc{cfg.query_window_n, cfg.block_size_g, cfg.sink_count_a, cfg.top_p};
    GpuSelection s{std::vector<uint8_t>(N), 0, 0};
    RefSelectionInfo info{};
    ref_top_p_select(scores.data(), static_cast<int64_t>(scores.size()), &rc, N, s.keep.data(), &info);
    s.cutoff = info.cutoff_rank;
    s.covered = info.covered_mass;
    return s;
}

static b2::ScoreConfig plain(float p) {
    b2::ScoreConfig c;
    c.top_p = p;
    c.block_size_g = 1;
    c.sink_count_a = 0;
    c.query_window_n = 1;
    return c;
}

TEST_CASE(top_p_select_worked_example) {  // test_selection.cpp:152-161
    const GpuSelection s = gpu_select({0.5f, 0.3f, 0.15f, 0.05f}, 4, plain(0.9f));
    CHECK(s.cutoff == 3);
    CHECK((s.keep == std::vector<uint8_t>{1, 1, 1, 1}));
}

TEST_CASE(selection_matches_reference_on_random_vectors) {  // test_selection.cpp:201-231
    std::mt19937 rng(21);
    std::uniform_real_distribution<float> U(0.f, 1.f);
    for (int trial = 0; trial < 300; ++trial) {
        const int nb = 1 + static_cast<int>(rng() % 80);
        std::vector<float> s(nb);
        for (auto& x : s) {
            const unsigned kind = rng() % 4;
            x = kind == 0 ? 0.f : kind == 1 ? std::floor(U(rng) * 4.f) * 0.25f
                : kind == 2 ? 1.4e-45f * static_cast<float>(1 + rng() % 5) : U(rng);
        }
        const float p = trial % 3 == 0 ? 1.f : 0.5f + 0.49f * U(rng);
        const GpuSelection g = gpu_select(s, nb, plain(p));
        const GpuSelection r = ref_select(s, nb, plain(p));
        CHECK(g.keep == r.keep);
        CHECK(g.cutoff == r.cutoff);
        CHECK(std::fabs(g.covered - r.covered) <= 1e-12 * std::max(1.0, std::fabs(r.covered)));
    }
}

TEST_CASE(config_errors_throw_config_error) {  // config.cpp:98-103
    bool threw = false;
    try {
        b2::ScoreConfig c;
        c.top_p = 0.f;
        c.validate();
    } catch (const b2::ConfigError&) {
        threw = true;
    }
    CHECK(threw);
}

TEST_CASE(negative_block_scores_are_contract_violations) {  // test_selection.cpp:192-199
    bool threw = false;
    try {
        gpu_select({0.5f, -0.1f}, 2, plain(0.9f));
    } catch (const b2::ContractViolation&) {
        threw = true;
    }
    CHECK(threw);
}

TEST_CASE(score_blocks_within_rtol_of_reference) {  // test_importance.cpp:111-142 style
    const int H = 8, Hkv = 2, D = 128;
    for (int N : {300, 1000, 2048}) {
        std::mt19937 rng(N);
        std::normal_distribution<float> nd(0.f, 1.f);
        std::vector<__nv_bfloat16> q(static_cast<size_t>(N) * H * D), k(static_cast<size_t>(N) * Hkv * D);
        std::vector<float> qf(q.size()), kf(k.size());
        for (size_t i = 0; i < q.size(); ++i) { q[i] = __float2bfloat16(nd(rng)); qf[i] = __bfloat162float(q[i]); }
        for (size_t i = 0; i < k.size(); ++i) { k[i] = __float2bfloat16(nd(rng)); kf[i] = __bfloat162float(k[i]); }
        b2::ScoreConfig cfg;
        const int64_t nb = (N + cfg.block_size_g - 1) / cfg.block_size_g;
        Dev<__nv_bfloat16> dq(q), dk(k);
        Dev<int32_t> cu(std::vector<int32_t>{0, N});
        Dev<float> bs(nb + 2);
        Dev<int32_t> cub(2);
        b2::VarlenBatch b{1, N, cu.p, nullptr};
        b2::HeadLayout h{H, Hkv, D, H / Hkv};
        b2::Workspace ws(b, h, cfg);
        b2::score_blocks(nullptr, b, h, cfg, dq.p, dk.p, bs.p, cub.p, ws);
        b2::check_device(nullptr, ws);
        const std::vector<float> got = bs.get(nb);
        // reference on the same bf16-exact values (MHA view: kv columns replicated)
        std::vector<float> kx(static_cast<size_t>(N) * H * D);
        for (int i = 0; i < N; ++i)
            for (int hh = 0; hh < H; ++hh)
                std::memcpy(&kx[(static_cast<size_t>(i) * H + hh) * D], &kf[(static_cast<size_t>(i) * Hkv + hh / (H / Hkv)) * D],
                            sizeof(float) * D);
        RefScoreConfig rc{cfg.query_window_n, cfg.block_size_g, cfg.sink_count_a, cfg.top_p};
        std::vector<float> want(nb);
        int32_t neff = 0;
        ref_score_tokens_heads(qf.data(), H * D, kx.data(), H * D, N, H, H, D, 0, H, &rc, nullptr, want.data(), &neff);
        for (int64_t g = 0; g < nb; ++g) CHECK(std::fabs(got[g] - want[g]) <= 1e-3f * std::fabs(want[g]) + 1e-9f);
    }
}

TEST_CASE(compaction_keeps_rows_in_position_order) {  // test_propagation.cpp:97-111
    const int rows = 8, cols = 32;
    std::vector<float> st(rows * cols);
    for (int i = 0; i < rows * cols; ++i) st[i] = static_cast<float>(i);
    Dev<float> src(st), dst(rows * cols);
    Dev<uint8_t> keep(std::vector<uint8_t>{1, 1, 0, 0, 0, 0, 1, 1});
    Dev<int32_t> cu(std::vector<int32_t>{0, rows}), cu_out(2), idx(rows), nout(1);
    b2::VarlenBatch b{1, rows, cu.p, nullptr};
    b2::ScoreConfig cfg;
    b2::Workspace ws(b, b2::HeadLayout{1, 1, 64}, cfg);
    b2::compact(nullptr, b, keep.p, {up_plane{src.p, dst.p, cols * 4, 0, 0}}, cu_out.p, idx.p, nout.p, ws);
    b2::check_device(nullptr, ws);
    CHECK((idx.get(4) == std::vector<int32_t>{0, 1, 6, 7}));
    CHECK((cu_out.get(2) == std::vector<int32_t>{0, 4}));
    const std::vector<float> out = dst.get(rows * cols);
    CHECK(std::memcmp(&out[2 * cols], &st[6 * cols], cols * 4) == 0);
}

TEST_CASE(attention_readout_matches_reference) {  // model.cpp:215-263 over retained rows
    const int H = 4, Hkv = 2, D = 128;
    const std::vector<int32_t> lens{300, 1, 129};
    std::vector<int32_t> cuv{0};
    for (int32_t n : lens) cuv.push_back(cuv.back() + n);
    const int T = cuv.back();
    std::mt19937_64 rng(11);
    std::normal_distribution<float> nd(0.f, 1.f);
    std::vector<__nv_bfloat16> q(static_cast<size_t>(T) * H * D), k(static_cast<size_t>(T) * Hkv * D), v(k.size());
    std::vector<float> qf(q.size()), kf(k.size()), vf(v.size());
    for (size_t i = 0; i < q.size(); ++i) { q[i] = __float2bfloat16(nd(rng)); qf[i] = __bfloat162float(q[i]); }
    for (size_t i = 0; i < k.size(); ++i) { k[i] = __float2bfloat16(nd(rng)); kf[i] = __bfloat162float(k[i]); }
    for (size_t i = 0; i < v.size(); ++i) { v[i] = __float2bfloat16(nd(rng)); vf[i] = __bfloat162float(v[i]); }
    std::vector<int64_t> pos(T);  // retained positions: strictly increasing with gaps
    for (size_t r = 0; r < lens.size(); ++r)
        for (int i = cuv[r]; i < cuv[r + 1]; ++i) pos[i] = 3 * (i - cuv[r]) + static_cast<int64_t>(r);
    Dev<__nv_bfloat16> dq(q), dk(k), dv(v), dout(q.size());
    Dev<int64_t> dpos(pos);
    Dev<int32_t> cu(cuv);
    b2::VarlenBatch b{static_cast<int32_t>(lens.size()), T, cu.p, nullptr};
    b2::HeadLayout h{H, Hkv, D, H / Hkv};
    b2::ScoreConfig cfg;
    b2::Workspace ws(b, h, cfg);
    b2::attention_readout(nullptr, b, h, dq.p, dk.p, dv.p, dpos.p, 0, dout.p, 0, ws);
    b2::check_device(nullptr, ws);
    const std::vector<__nv_bfloat16> got = dout.get(q.size());
    for (size_t r = 0; r < lens.size(); ++r) {
        const int b0 = cuv[r], n = lens[r];
        std::vector<float> want(static_cast<size_t>(n) * H * D);
        ref_attention_readout(&qf[static_cast<size_t>(b0) * H * D], &pos[b0], n, &kf[static_cast<size_t>(b0) * Hkv * D],
                              &vf[static_cast<size_t>(b0) * Hkv * D], &pos[b0], n, H, Hkv, D, 0, want.data());
        for (size_t i = 0; i < want.size(); ++i) {  // bf16 P and output: 2e-2 relative
            const float g = __bfloat162float(got[static_cast<size_t>(b0) * H * D + i]);
            CHECK(std::fabs(g - want[i]) <= 2e-2f * (1.f + std::fabs(want[i])));
        }
    }
}

int main() {
    struct { const char* name; void (*fn)(); } cases[] = {
        {"top_p_select worked example", top_p_select_worked_example},
        {"selection matches the reference on random vectors", selection_matches_reference_on_random_vectors},
        {"config errors throw ConfigError", config_errors_throw_config_error},
        {"negative block scores are contract violations", negative_block_scores_are_contract_violations},
        {"score_blocks within rtol 1e-3 of the reference", score_blocks_within_rtol_of_reference},
        {"compaction keeps rows in position order", compaction_keeps_rows_in_position_order},
        {"attention_readout matches the reference", attention_readout_matches_reference},
    };
    for (auto& c : cases) {
        const int before = g_failed;
        c.fn();
        std::printf("[%s] %s\n", g_failed == before ? "ok" : "FAIL", c.name);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed == 0 ? 0 : 1;
}
