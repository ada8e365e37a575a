// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference implementation.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with the
// reference's own sources where they lie (/root/reference/proj/core/src/*.cpp) into
// oracle/_ref/libuniprefill_ref.so.  Nothing of the reference is copied into this repo;
// this file only converts plain arrays to the reference's types, calls its public API
// (core/include/uniprefill/*.hpp) and maps its exceptions to status codes:
//   0 ok, 1 ConfigError, 2 ContractViolation, 9 any other exception.
#include "uniprefill/errors.hpp"
#include "uniprefill/flops.hpp"
#include "uniprefill/model.hpp"
#include "uniprefill/importance.hpp"
#include "uniprefill/propagation.hpp"
#include "uniprefill/kvcache.hpp"
#include "uniprefill/scheduler.hpp"
#include "uniprefill/selection.hpp"
#include "uniprefill/tp_sim.hpp"

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <thread>
#include <vector>

using namespace uniprefill;

namespace {

struct RefScoreConfig {
    int32_t query_window_n;
    int32_t block_size_g;
    int32_t sink_count_a;
    float top_p;
};

ScoreConfig to_cfg(const RefScoreConfig* c) {
    ScoreConfig s;
    s.query_window_n = c->query_window_n;
    s.block_size_g = c->block_size_g;
    s.sink_count_a = c->sink_count_a;
    s.top_p = c->top_p;
    return s;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError&) {
        return 1;
    } catch (const ContractViolation&) {
        return 2;
    } catch (...) {
        return 9;
    }
}

// MHA view of a GQA tensor: kv-head columns replicated H / H_kv times.
Matrix expand_heads(const float* src, int64_t ld, int64_t rows, int heads_in, int heads_out,
                    int head_dim) {
    Matrix m(rows, static_cast<int64_t>(heads_out) * head_dim);
    const int group = heads_out / heads_in;
    for (int64_t r = 0; r < rows; ++r) {
        for (int h = 0; h < heads_out; ++h) {
            std::memcpy(m.row(r) + static_cast<int64_t>(h) * head_dim,
                        src + r * ld + static_cast<int64_t>(h / group) * head_dim,
                        sizeof(float) * static_cast<size_t>(head_dim));
        }
    }
    return m;
}

struct RefSelectionInfo {
    int64_t cutoff_rank;
    int64_t retained_count;
    double retention_ratio;
    double covered_mass;
    int32_t degenerate_keep_all;
};

struct RefModelCfg {
    int32_t num_blocks;
    int32_t sublayers_per_block;
    int32_t hidden_dim;
    int32_t head_dim;
    int32_t num_heads;
    int32_t window_size;
    int32_t ffn_dim;
    const int32_t* layer_pattern;  // pattern_length() SublayerKind values
};

ModelConfig to_model(const RefModelCfg* c) {
    ModelConfig m;
    m.num_blocks = c->num_blocks;
    m.sublayers_per_block = c->sublayers_per_block;
    m.hidden_dim = c->hidden_dim;
    m.head_dim = c->head_dim;
    m.num_heads = c->num_heads;
    m.window_size = c->window_size;
    m.ffn_dim = c->ffn_dim;
    for (int i = 0; i < m.pattern_length(); ++i) m.layer_pattern.push_back(static_cast<SublayerKind>(c->layer_pattern[i]));
    return m;
}

} // namespace

extern "C" {

// attention_readout (model.cpp:215-263) over one segment; GQA k/v ([rows, kv_heads*D]) are
// expanded to the reference's MHA view.  window <= 0: no window.
int ref_attention_readout(const float* q, const int64_t* q_pos, int64_t q_rows, const float* k, const float* v,
                          const int64_t* kv_pos, int64_t kv_rows, int heads, int kv_heads, int head_dim,
                          int64_t window, float* out) {
    return guarded([&] {
        Matrix qm(q_rows, static_cast<int64_t>(heads) * head_dim);
        std::memcpy(qm.data.data(), q, sizeof(float) * qm.data.size());
        const int64_t kld = static_cast<int64_t>(kv_heads) * head_dim;
        const Matrix km = expand_heads(k, kld, kv_rows, kv_heads, heads, head_dim);
        const Matrix vm = expand_heads(v, kld, kv_rows, kv_heads, heads, head_dim);
        const Matrix o = attention_readout(qm, std::span<const int64_t>(q_pos, q_rows), km, vm,
                                           std::span<const int64_t>(kv_pos, kv_rows), heads,
                                           window > 0 ? std::optional<int64_t>(window) : std::nullopt);
        std::memcpy(out, o.data.data(), sizeof(float) * o.data.size());
    });
}

// layer_flops / scoring_flops (flops.cpp:14-39).
int ref_layer_flops(int32_t kind, int64_t tokens, const RefModelCfg* cfg, uint64_t* out) {
    return guarded([&] { *out = layer_flops(static_cast<SublayerKind>(kind), tokens, to_model(cfg)); });
}

int ref_scoring_flops(int64_t effective_n, int64_t num_keys, const RefModelCfg* cfg, uint64_t* out) {
    return guarded([&] { *out = scoring_flops(effective_n, num_keys, to_model(cfg)); });
}

// validate_savings (flops.cpp:58-144) over a dense ledger (every layer at `original`
// tokens) and an accelerated ledger (accel_tokens[l] per layer, drops in order, scoring
// overhead).  u64_out = {dense, accel, scoring, measured, formula, closed_linear_form};
// i32_out = {exact, single_drop, drop_layer, layers_after_drop, linear_form_exact};
// f64_out = {retention_ratio, attention_only_ratio}.
int ref_validate_savings(const RefModelCfg* cfg, int64_t original, const int64_t* accel_tokens,
                         int32_t num_drops, const int32_t* drop_layers, const int64_t* before,
                         const int64_t* after, const double* retention, uint64_t scoring,
                         uint64_t* u64_out, int32_t* i32_out, double* f64_out) {
    return guarded([&] {
        const ModelConfig m = to_model(cfg);
        FlopsLedger dense, accel;
        for (int l = 0; l < m.total_layers(); ++l) {
            const SublayerKind kind = m.layer_pattern[static_cast<size_t>(l % m.pattern_length())];
            dense.add_layer(l, kind, original, m);
            accel.add_layer(l, kind, accel_tokens[l], m);
        }
        for (int32_t d = 0; d < num_drops; ++d) {
            DropRecord r;
            r.layer = drop_layers[d];
            r.tokens_before = before[d];
            r.tokens_after = after[d];
            r.retention_ratio = retention[d];
            accel.add_drop(r);
        }
        accel.add_scoring(scoring);
        const SavingsReport rep = validate_savings(dense, accel, m);
        const uint64_t u[6] = {rep.dense_total, rep.accel_total, rep.scoring_overhead, rep.measured_delta,
                               rep.formula_delta, rep.closed_linear_form};
        std::memcpy(u64_out, u, sizeof(u));
        i32_out[0] = rep.exact_match;
        i32_out[1] = rep.single_drop;
        i32_out[2] = rep.drop_layer;
        i32_out[3] = rep.layers_after_drop;
        i32_out[4] = rep.linear_form_exact;
        f64_out[0] = rep.retention_ratio;
        f64_out[1] = rep.attention_only_ratio;
    });
}


int ref_phi_encode(float x, uint32_t* out) {
    return guarded([&] { *out = phi_encode(x); });
}

float ref_phi_decode(uint32_t bits) { return phi_decode(bits); }

// score_tokens_heads (importance.hpp:42-43) over one request.
int ref_score_tokens_heads(const float* q, int64_t q_ld, const float* k, int64_t k_ld, int64_t N,
                           int num_heads, int num_kv_heads, int head_dim, int head_begin,
                           int head_end, const RefScoreConfig* cfg, float* token_scores,
                           float* block_scores, int32_t* effective_n) {
    return guarded([&] {
        const Matrix qm = expand_heads(q, q_ld, N, num_heads, num_heads, head_dim);
        const Matrix km = expand_heads(k, k_ld, N, num_kv_heads, num_heads, head_dim);
        const ImportanceScores s =
            score_tokens_heads(qm, km, num_heads, head_begin, head_end, to_cfg(cfg));
        if (token_scores) std::memcpy(token_scores, s.token_scores.data(), s.token_scores.size() * 4);
        std::memcpy(block_scores, s.block_scores.data(), s.block_scores.size() * 4);
        if (effective_n) *effective_n = s.effective_n;
    });
}

// sharded_block_scores + allreduce_scores (tp_sim.hpp:25-31).
int ref_sharded_allreduce(const float* q, int64_t q_ld, const float* k, int64_t k_ld, int64_t N,
                          int num_heads, int num_kv_heads, int head_dim, const RefScoreConfig* cfg,
                          int tp_degree, float* shard_out /* tp x nb or NULL */, float* reduced) {
    return guarded([&] {
        const Matrix qm = expand_heads(q, q_ld, N, num_heads, num_heads, head_dim);
        const Matrix km = expand_heads(k, k_ld, N, num_kv_heads, num_heads, head_dim);
        const auto shards = sharded_block_scores(qm, km, num_heads, to_cfg(cfg), tp_degree);
        if (shard_out) {
            size_t off = 0;
            for (const auto& s : shards) {
                std::memcpy(shard_out + off, s.block_scores.data(), s.block_scores.size() * 4);
                off += s.block_scores.size();
            }
        }
        const std::vector<float> r = allreduce_scores(shards);
        std::memcpy(reduced, r.data(), r.size() * 4);
    });
}

// sharded_block_scores + allreduce_scores (tp_sim.cpp:12-49) with the shards scored on up to
// `threads` host threads -- for BASELINE-size parity runs and the timed CPU reference arm.
// Bit-identical to the sequential reference: shard t is score_tokens_heads over its own
// heads only (each head's arithmetic reads only that head's columns, importance.cpp:104-119),
// on a query matrix holding just the last n_eff rows (the only rows score_tokens_heads reads,
// :109-112), and the shards are reduced by the reference's allreduce_scores.  With
// tp_degree == 1 the single shard IS score_tokens (importance.cpp:129-132) and its block
// scores are returned unreduced.  q: the LAST q_rows rows of the request (q_rows >= min(n, N)),
// [q_rows, num_heads*D]; k: [N, num_kv_heads*D].
static std::vector<float> sharded_scores_mt(const float* q, int64_t q_ld, int64_t q_rows, const float* k,
                                            int64_t k_ld, int64_t N, int num_heads, int num_kv_heads,
                                            int head_dim, const ScoreConfig& sc, int tp_degree, int threads,
                                            float* shard_out) {
    if (tp_degree <= 0 || num_heads % tp_degree != 0) throw ConfigError("bad tp_degree");
    const int hps = num_heads / tp_degree;
    const int group = num_heads / num_kv_heads;
    const int64_t neff = std::min<int64_t>(sc.query_window_n, N);
    if (q_rows < neff) throw ContractViolation("need the last n_eff query rows");
    std::vector<ShardScores> shards(static_cast<size_t>(tp_degree));
    std::vector<int> status(static_cast<size_t>(tp_degree), 0);
    auto work = [&](int t) {
        status[static_cast<size_t>(t)] = guarded([&] {
            Matrix qm(neff, static_cast<int64_t>(hps) * head_dim);
            Matrix km(N, static_cast<int64_t>(hps) * head_dim);
            for (int hh = 0; hh < hps; ++hh) {
                const int h = t * hps + hh;
                for (int64_t j = 0; j < neff; ++j)
                    std::memcpy(qm.row(j) + static_cast<int64_t>(hh) * head_dim,
                                q + (q_rows - neff + j) * q_ld + static_cast<int64_t>(h) * head_dim,
                                sizeof(float) * static_cast<size_t>(head_dim));
                for (int64_t i = 0; i < N; ++i)
                    std::memcpy(km.row(i) + static_cast<int64_t>(hh) * head_dim,
                                k + i * k_ld + static_cast<int64_t>(h / group) * head_dim,
                                sizeof(float) * static_cast<size_t>(head_dim));
            }
            const ImportanceScores sc_t = score_tokens_heads(qm, km, hps, 0, hps, sc);
            shards[static_cast<size_t>(t)] = ShardScores{t, sc_t.block_scores};
        });
    };
    const int nt = std::max(1, std::min(threads, tp_degree));
    if (nt == 1) {
        for (int t = 0; t < tp_degree; ++t) work(t);
    } else {
        std::vector<std::thread> pool;
        std::atomic<int> next{0};
        for (int w = 0; w < nt; ++w)
            pool.emplace_back([&] { for (int t = next++; t < tp_degree; t = next++) work(t); });
        for (auto& th : pool) th.join();
    }
    for (int st : status) {
        if (st == 1) throw ConfigError("shard failed");
        if (st != 0) throw ContractViolation("shard failed");
    }
    if (shard_out) {
        size_t off = 0;
        for (const auto& sh : shards) {
            std::memcpy(shard_out + off, sh.block_scores.data(), sh.block_scores.size() * 4);
            off += sh.block_scores.size();
        }
    }
    if (tp_degree == 1) return shards[0].block_scores;
    return allreduce_scores(shards);
}

int ref_sharded_allreduce_mt(const float* q, int64_t q_ld, int64_t q_rows, const float* k, int64_t k_ld,
                             int64_t N, int num_heads, int num_kv_heads, int head_dim, const RefScoreConfig* cfg,
                             int tp_degree, int threads, float* shard_out /* tp x nb or NULL */, float* reduced) {
    return guarded([&] {
        const std::vector<float> r = sharded_scores_mt(q, q_ld, q_rows, k, k_ld, N, num_heads, num_kv_heads,
                                                       head_dim, to_cfg(cfg), tp_degree, threads, shard_out);
        std::memcpy(reduced, r.data(), r.size() * 4);
    });
}

// One unit of the reference's varlen layer loop -- a (request, drop layer) pair at
// scheduler.cpp:293-332, hot path only: score (score_tokens; with tp_degree > 1 the
// reference's TP path sharded_block_scores + allreduce_scores, propagation.cpp:163-170, its
// shards on `threads` host threads), top_p_select (:172), apply_drop on the request's
// TokenStream (scheduler.cpp:318), patch_metadata on its packed segment (:332).  The stream
// and batch are built from `hidden` [N, hidden_cols] before the clock starts; *seconds is the
// hot path's steady_clock time, *retained the rows kept.
int ref_drop_unit(const float* q, int64_t q_ld, int64_t q_rows, const float* k, int64_t k_ld, int64_t N,
                  int num_heads, int num_kv_heads, int head_dim, const float* hidden, int64_t hidden_cols,
                  const RefScoreConfig* cfg, int tp_degree, int threads, int64_t* retained, double* seconds) {
    return guarded([&] {
        const ScoreConfig sc = to_cfg(cfg);
        Matrix prompt(N, hidden_cols);
        std::memcpy(prompt.data.data(), hidden, sizeof(float) * static_cast<size_t>(N * hidden_cols));
        TokenStream stream = TokenStream::from_prompt(prompt);
        DropHistory history;
        history.original_length = N;
        PackedBatch batch;
        batch.tokens = std::move(prompt);
        batch.cu_seqlens = {0, N};
        batch.request_ids = {0};
        batch.phases = {Phase::Prefill};
        const auto t0 = std::chrono::steady_clock::now();
        const std::vector<float> blocks = sharded_scores_mt(q, q_ld, q_rows, k, k_ld, N, num_heads, num_kv_heads,
                                                            head_dim, sc, tp_degree, threads, nullptr);
        std::vector<std::optional<Selection>> sels(1);
        sels[0] = top_p_select(blocks, sc, N);
        apply_drop(stream, *sels[0], 0, history);
        patch_metadata(batch, sels, 0);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        *retained = batch.cu_seqlens.back();
    });
}

// allreduce_scores (tp_sim.hpp:31) on explicit shards.
int ref_allreduce_scores(const float* const* shards, const int32_t* shard_ids, int32_t tp,
                         int64_t length, float* out) {
    return guarded([&] {
        std::vector<ShardScores> v;
        for (int32_t t = 0; t < tp; ++t) {
            v.push_back(ShardScores{shard_ids[t], std::vector<float>(shards[t], shards[t] + length)});
        }
        const std::vector<float> r = allreduce_scores(v);
        std::memcpy(out, r.data(), r.size() * 4);
    });
}

// top_p_select (selection.hpp:53-54).
int ref_top_p_select(const float* block_scores, int64_t num_blocks, const RefScoreConfig* cfg,
                     int64_t num_tokens, uint8_t* keep, RefSelectionInfo* info) {
    return guarded([&] {
        const Selection sel = top_p_select(
            std::span<const float>(block_scores, static_cast<size_t>(num_blocks)), to_cfg(cfg),
            num_tokens);
        std::memcpy(keep, sel.keep_mask.data(), sel.keep_mask.size());
        info->cutoff_rank = sel.cutoff_rank;
        info->retained_count = sel.retained_count();
        info->retention_ratio = sel.retention_ratio;
        info->covered_mass = sel.covered_mass;
        info->degenerate_keep_all = sel.degenerate_keep_all ? 1 : 0;
    });
}

// top_p_select over `count` independent score vectors (vector i = scores[offsets[i] ..
// offsets[i+1]), top_p = top_ps[i], the other knobs from *base); keep masks concatenated
// the same way, cutoff ranks per vector.  Returns the first non-zero status.
int ref_top_p_select_batch(const float* scores, const int64_t* offsets, const float* top_ps, int32_t count,
                           const RefScoreConfig* base, uint8_t* keep, int64_t* cutoff_rank) {
    for (int32_t i = 0; i < count; ++i) {
        RefScoreConfig c = *base;
        c.top_p = top_ps[i];
        const int64_t b = offsets[i], n = offsets[i + 1] - offsets[i];
        RefSelectionInfo info{};
        const int st = ref_top_p_select(scores + b, n, &c, n, keep + b, &info);
        if (st != 0) return st;
        cutoff_rank[i] = info.cutoff_rank;
    }
    return 0;
}

// expand_mask (selection.hpp:46-47).
int ref_expand_mask(const uint8_t* block_mask, int64_t num_blocks, int block_size,
                    int64_t num_tokens, int64_t sink_count, int64_t window_n, uint8_t* keep) {
    return guarded([&] {
        const std::vector<uint8_t> bm(block_mask, block_mask + num_blocks);
        const std::vector<uint8_t> k = expand_mask(bm, block_size, num_tokens, sink_count, window_n);
        std::memcpy(keep, k.data(), k.size());
    });
}

// apply_drop (propagation.hpp:415) on one request's stream; returns compacted rows and
// logical positions, and checks the parked map partitions the sequence.
int ref_apply_drop(const float* states, int64_t rows, int64_t cols, const uint8_t* keep,
                   float* out_states, int64_t* out_positions, int64_t* out_rows) {
    return guarded([&] {
        Matrix prompt(rows, cols);
        std::memcpy(prompt.data.data(), states, sizeof(float) * static_cast<size_t>(rows * cols));
        TokenStream stream = TokenStream::from_prompt(prompt);
        Selection sel;
        sel.keep_mask.assign(keep, keep + rows);
        for (int64_t i = 0; i < rows; ++i) {
            if (keep[i]) sel.retained_indices.push_back(i);
        }
        DropHistory history;
        history.original_length = rows;
        apply_drop(stream, sel, 0, history);
        stream.validate();
        std::memcpy(out_states, stream.active_states.data.data(),
                    sizeof(float) * stream.active_states.data.size());
        std::memcpy(out_positions, stream.logical_positions.data(),
                    sizeof(int64_t) * stream.logical_positions.size());
        *out_rows = stream.active_count();
    });
}

// A sequence of drops with the states transformed between them, then reconstitute
// (propagation.cpp:47-100).  keeps[d] has one entry per row active before drop d;
// after[d] (rows retained by drop d, or NULL) replaces the active states after drop d
// -- standing in for the layers between drops.  Writes the full-length reconstituted
// states and positions.
int ref_reconstitute_sequence(const float* prompt, int64_t rows, int64_t cols, int32_t num_drops,
                              const uint8_t* const* keeps, const float* const* after, float* out_states,
                              int64_t* out_positions) {
    return guarded([&] {
        Matrix m(rows, cols);
        std::memcpy(m.data.data(), prompt, sizeof(float) * static_cast<size_t>(rows * cols));
        TokenStream stream = TokenStream::from_prompt(m);
        DropHistory history;
        history.original_length = rows;
        for (int32_t d = 0; d < num_drops; ++d) {
            const int64_t n = stream.active_count();
            Selection sel;
            sel.keep_mask.assign(keeps[d], keeps[d] + n);
            for (int64_t i = 0; i < n; ++i)
                if (keeps[d][i]) sel.retained_indices.push_back(i);
            apply_drop(stream, sel, d, history);
            if (after != nullptr && after[d] != nullptr)
                std::memcpy(stream.active_states.data.data(), after[d],
                            sizeof(float) * stream.active_states.data.size());
        }
        reconstitute(stream);
        stream.validate();
        std::memcpy(out_states, stream.active_states.data.data(), sizeof(float) * stream.active_states.data.size());
        std::memcpy(out_positions, stream.logical_positions.data(),
                    sizeof(int64_t) * stream.logical_positions.size());
    });
}

// PagedKVCache::recompute_slots_after_drop (kvcache.cpp:147-158) for one request: pages
// for positions [0, prealloc_len) are first allocated layer-interleaved (so physical ids
// differ per layer), then the slots of the retained positions are recomputed (allocating
// any missing page on demand).  Exports the resulting block tables [num_layers][max_pages]
// (-1 = no page) and the slots [num_layers][n_ret].
int ref_recompute_slots(int num_layers, int block_size, int64_t prealloc_len, const int64_t* retained,
                        int64_t n_ret, int64_t max_pages, int32_t* tables, int64_t* slots) {
    return guarded([&] {
        PagedKVCache cache(num_layers, 8, block_size);
        for (int64_t pos = 0; pos < prealloc_len; pos += block_size)
            for (int l = num_layers - 1; l >= 0; --l) cache.ensure_slot(l, 0, pos);
        std::vector<int> layers(static_cast<size_t>(num_layers));
        for (int l = 0; l < num_layers; ++l) layers[static_cast<size_t>(l)] = l;
        const auto out = cache.recompute_slots_after_drop(layers, 0, std::span<const int64_t>(retained, n_ret));
        for (int l = 0; l < num_layers; ++l) {
            for (int64_t i = 0; i < n_ret; ++i) slots[l * n_ret + i] = out[static_cast<size_t>(l)][static_cast<size_t>(i)];
            for (int64_t pg = 0; pg < max_pages; ++pg)
                tables[l * max_pages + pg] = cache.page_allocated(l, 0, pg * block_size)
                                                 ? static_cast<int32_t>(cache.slot_for(l, 0, pg * block_size) / block_size)
                                                 : -1;
        }
    });
}

// decode_seqused (kvcache.cpp:182-186) for one request's drop history.
int ref_decode_seqused(int64_t original_length, int64_t decode_appended, int32_t num_events,
                       const int32_t* event_layers, const int64_t* retained_lengths, int32_t layer, int64_t* out) {
    return guarded([&] {
        DropHistory h;
        h.original_length = original_length;
        h.decode_appended = decode_appended;
        for (int32_t e = 0; e < num_events; ++e) {
            DropEvent ev;
            ev.layer = event_layers[e];
            ev.retained_length = retained_lengths[e];
            h.events.push_back(ev);
        }
        *out = decode_seqused(h, layer);
    });
}

// patch_metadata (scheduler.hpp:52-53) over a packed batch.  selected[s] != 0 attaches a
// Selection built from keep; is_decode[s] marks decode-phase segments.
int ref_patch_metadata(const float* tokens, int64_t total_rows, int64_t cols,
                       const int64_t* cu_seqlens, int32_t num_requests, const uint8_t* keep,
                       const uint8_t* selected, const uint8_t* is_decode, float* out_tokens,
                       int64_t* out_cu) {
    return guarded([&] {
        PackedBatch batch;
        batch.tokens = Matrix(total_rows, cols);
        std::memcpy(batch.tokens.data.data(), tokens,
                    sizeof(float) * static_cast<size_t>(total_rows * cols));
        batch.cu_seqlens.assign(cu_seqlens, cu_seqlens + num_requests + 1);
        std::vector<std::optional<Selection>> sels(static_cast<size_t>(num_requests));
        for (int32_t s = 0; s < num_requests; ++s) {
            batch.request_ids.push_back(s);
            batch.phases.push_back(is_decode && is_decode[s] ? Phase::Decode : Phase::Prefill);
            if (selected && selected[s]) {
                Selection sel;
                const int64_t b = cu_seqlens[s], e = cu_seqlens[s + 1];
                sel.keep_mask.assign(keep + b, keep + e);
                for (int64_t i = 0; i < e - b; ++i) {
                    if (keep[b + i]) sel.retained_indices.push_back(i);
                }
                sels[static_cast<size_t>(s)] = sel;
            }
        }
        patch_metadata(batch, sels, 0);
        std::memcpy(out_tokens, batch.tokens.data.data(), sizeof(float) * batch.tokens.data.size());
        std::memcpy(out_cu, batch.cu_seqlens.data(), sizeof(int64_t) * batch.cu_seqlens.size());
    });
}

// The reference hot path over a varlen batch, exactly as Engine::run_batch drives it per
// drop layer (scheduler.cpp:293-332): per segment score_tokens -> top_p_select, then the
// segment's rows are compacted (patch_metadata).  Segments are independent units
// (SPEC.md:202,265), so `threads` workers process segments concurrently; each segment's
// arithmetic is unchanged.  block_scores_out is Σ ceil(N_r/G) floats (segment-major),
// keep_out T bytes.  hidden (T x hidden_cols) is compacted into hidden_out.
int ref_drop_layer_varlen(const float* q, int64_t q_ld, const float* k, int64_t k_ld,
                          const float* hidden, int64_t hidden_cols, const int64_t* cu_seqlens,
                          int32_t num_requests, int num_heads, int num_kv_heads, int head_dim,
                          const RefScoreConfig* cfg, int threads, float* block_scores_out,
                          uint8_t* keep_out, float* hidden_out, int64_t* cu_out) {
    return guarded([&] {
        const ScoreConfig sc = to_cfg(cfg);
        const int G = sc.block_size_g;
        std::vector<int64_t> cu_blocks(static_cast<size_t>(num_requests) + 1, 0);
        for (int32_t s = 0; s < num_requests; ++s) {
            const int64_t n = cu_seqlens[s + 1] - cu_seqlens[s];
            cu_blocks[s + 1] = cu_blocks[s] + (n + G - 1) / G;
        }
        std::vector<int> status(static_cast<size_t>(num_requests), 0);
        auto work = [&](int32_t s) {
            status[static_cast<size_t>(s)] = guarded([&] {
                const int64_t b = cu_seqlens[s], n = cu_seqlens[s + 1] - cu_seqlens[s];
                const Matrix qm = expand_heads(q + b * q_ld, q_ld, n, num_heads, num_heads, head_dim);
                const Matrix km = expand_heads(k + b * k_ld, k_ld, n, num_kv_heads, num_heads, head_dim);
                const ImportanceScores scores = score_tokens(qm, km, num_heads, sc);
                const Selection sel = top_p_select(scores.block_scores, sc, n);
                std::memcpy(block_scores_out + cu_blocks[s], scores.block_scores.data(),
                            scores.block_scores.size() * 4);
                std::memcpy(keep_out + b, sel.keep_mask.data(), sel.keep_mask.size());
            });
        };
        const int nt = threads < 1 ? 1 : threads;
        if (nt == 1 || num_requests <= 1) {
            for (int32_t s = 0; s < num_requests; ++s) work(s);
        } else {
            std::vector<std::thread> pool;
            std::atomic<int32_t> next{0};
            for (int t = 0; t < nt; ++t) {
                pool.emplace_back([&] {
                    for (int32_t s = next++; s < num_requests; s = next++) work(s);
                });
            }
            for (auto& th : pool) th.join();
        }
        for (int st : status) {
            if (st == 1) throw ConfigError("segment failed");
            if (st != 0) throw ContractViolation("segment failed");
        }
        // Compaction through the reference's own patch_metadata.
        PackedBatch batch;
        const int64_t T = cu_seqlens[num_requests];
        batch.tokens = Matrix(T, hidden_cols);
        std::memcpy(batch.tokens.data.data(), hidden, sizeof(float) * static_cast<size_t>(T * hidden_cols));
        batch.cu_seqlens.assign(cu_seqlens, cu_seqlens + num_requests + 1);
        std::vector<std::optional<Selection>> sels(static_cast<size_t>(num_requests));
        for (int32_t s = 0; s < num_requests; ++s) {
            batch.request_ids.push_back(s);
            batch.phases.push_back(Phase::Prefill);
            Selection sel;
            const int64_t b = cu_seqlens[s], e = cu_seqlens[s + 1];
            sel.keep_mask.assign(keep_out + b, keep_out + e);
            for (int64_t i = 0; i < e - b; ++i) {
                if (keep_out[b + i]) sel.retained_indices.push_back(i);
            }
            sels[static_cast<size_t>(s)] = sel;
        }
        patch_metadata(batch, sels, 0);
        std::memcpy(hidden_out, batch.tokens.data.data(), sizeof(float) * batch.tokens.data.size());
        std::memcpy(cu_out, batch.cu_seqlens.data(), sizeof(int64_t) * batch.cu_seqlens.size());
    });
}

} // extern "C"
