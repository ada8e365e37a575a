/*
 * uniprefill_oracle.c -- CPU restatement of the UniPrefill token-selection hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see uniprefill_oracle.h).  Parity is pinned against the
 * reference itself (oracle/_ref/libuniprefill_ref.so, built from
 * /root/reference/proj/core/src by oracle/Makefile) and against the golden vectors in
 * tests/golden/.  Build with -O2 -ffp-contract=off: the arithmetic order and rounding
 * below are the reference's, and FMA contraction would change the last bits.
 */
#include "uniprefill_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ config */

/* ScoreConfig::validate (config.cpp:98-103). */
int orc_config_validate(const orc_score_config* cfg) {
    if (cfg->query_window_n <= 0) return ORC_ERR_CONFIG;
    if (cfg->block_size_g <= 0) return ORC_ERR_CONFIG;
    if (cfg->sink_count_a < 0) return ORC_ERR_CONFIG;
    if (!(cfg->top_p > 0.0f && cfg->top_p <= 1.0f)) return ORC_ERR_CONFIG;
    return ORC_OK;
}

/* ------------------------------------------------------------------ phi / packing */

static uint32_t f2u(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return u;
}
static float u2f(uint32_t u) {
    float x;
    memcpy(&x, &u, 4);
    return x;
}

/* phi_encode (selection.cpp:14-19): -0 collapses to +0, then a sign-dependent xor. */
int orc_phi_encode(float x, uint32_t* out) {
    if (!isfinite(x)) return ORC_ERR_CONTRACT;
    if (x == 0.0f) x = 0.0f;
    const uint32_t bits = f2u(x);
    *out = x >= 0.0f ? (bits ^ 0x80000000u) : (bits ^ 0xFFFFFFFFu);
    return ORC_OK;
}

/* phi_decode (selection.cpp:21-25). */
float orc_phi_decode(uint32_t bits) {
    const uint32_t raw = (bits & 0x80000000u) ? (bits ^ 0x80000000u) : (bits ^ 0xFFFFFFFFu);
    return u2f(raw);
}

/* PackedScore::pack (selection.cpp:27-30): phi(s) << 32 | ~g (ones' complement, so the
 * lower block index wins ties in descending order). */
int orc_pack_score(float score, uint32_t block_index, uint64_t* out) {
    uint32_t e;
    const int st = orc_phi_encode(score, &e);
    if (st != ORC_OK) return st;
    *out = ((uint64_t)e << 32) | (uint64_t)(~block_index);
    return ORC_OK;
}

/* ------------------------------------------------------------------ rng */

/* hash_mix / hash_combine / CounterRng (rng.cpp:10-40). */
uint64_t orc_hash_mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

static uint64_t hash_combine(uint64_t a, uint64_t b) {
    return orc_hash_mix(a ^ (0x9e3779b97f4a7c15ULL + (b << 6) + (b >> 2) + orc_hash_mix(b)));
}

uint64_t orc_rng_key(uint64_t seed, uint64_t stream) { return hash_combine(seed, stream); }

uint64_t orc_rng_bits(uint64_t key, uint64_t i) {
    return orc_hash_mix(key ^ (i * 0xd1342543de82ef95ULL + 0x2545f4914f6cdd1dULL));
}

double orc_rng_uniform(uint64_t key, uint64_t i) {
    const double u = (double)(orc_rng_bits(key, i) >> 11) * 0x1.0p-53;
    return u > 0.0 ? u : 0x1.0p-53;
}

float orc_rng_normal(uint64_t key, uint64_t i, double stddev) {
    const double u1 = orc_rng_uniform(key, 2 * i);
    const double u2 = orc_rng_uniform(key, 2 * i + 1);
    const double r = sqrt(-2.0 * log(u1));
    const double z = r * cos(2.0 * 3.14159265358979323846 * u2);
    return (float)(z * stddev);
}

void orc_rng_normal_fill(uint64_t key, uint64_t first, int64_t count, double stddev, float* out) {
    for (int64_t j = 0; j < count; ++j) out[j] = orc_rng_normal(key, first + (uint64_t)j, stddev);
}

/* ------------------------------------------------------------------ acceptance c3 inputs */

/* The vector stream of criterion_3 (acceptance_main.cpp:175-199), counter for counter. */
int64_t orc_c3_vector(uint64_t* ctr, int trial, float* scores, float* top_p) {
    const uint64_t key = orc_rng_key(31, 0x6333ULL);
    const double u = orc_rng_uniform(key, (*ctr)++);
    int64_t len = (int64_t)pow(2.0, u * 12.0);
    if (len < 1) len = 1;
    for (int64_t i = 0; i < len; ++i) {
        float v;
        switch (orc_rng_bits(key, (*ctr)++) % 5) {
        case 0: v = 0.0f; break;
        case 1: v = (float)(int)(orc_rng_uniform(key, (*ctr)++) * 8.0) * 0.125f; break;
        case 2: v = 1.40129846e-45f * (float)(1 + orc_rng_bits(key, (*ctr)++) % 7); break;
        default: v = (float)orc_rng_uniform(key, (*ctr)++); break;
        }
        scores[i] = v;
    }
    *top_p = trial % 7 == 0 ? 1.0f : (float)(0.3 + 0.7 * orc_rng_uniform(key, (*ctr)++));
    return len;
}

static const float* g_c3_scores;
static int cmp_c3_order(const void* a, const void* b) {  /* score desc, index asc (stable) */
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    const float sx = g_c3_scores[x], sy = g_c3_scores[y];
    if (sx != sy) return sx > sy ? -1 : 1;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* reference_blocks (acceptance_main.cpp:148-173) + the forced last token (:205-206). */
void orc_c3_reference_blocks(const float* scores, int64_t len, double top_p, uint8_t* keep) {
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(len > 0 ? len : 1));
    double total = 0.0;
    for (int64_t i = 0; i < len; ++i) {
        order[i] = i;
        total += scores[i];
        keep[i] = 0;
    }
    g_c3_scores = scores;
    qsort(order, (size_t)len, sizeof(int64_t), cmp_c3_order);
    if (total <= 0.0) {
        for (int64_t i = 0; i < len; ++i) keep[i] = 1;
    } else {
        double cum = 0.0;
        for (int64_t r = 0; r < len; ++r) {
            keep[order[r]] = 1;
            cum += scores[order[r]];
            if (cum / total >= top_p) break;
        }
    }
    if (len > 0) keep[len - 1] = 1;
    free(order);
}

/* ------------------------------------------------------------------ scorer */

/* block_reduce (importance.cpp:76-90): float token scores summed in double in index order,
 * divided by the member count (ragged tail uses its real size), rounded to float. */
int orc_block_reduce(const float* token_scores, int64_t N, int block_size, float* out) {
    if (N <= 0) return ORC_ERR_CONTRACT;
    if (block_size <= 0) return ORC_ERR_CONTRACT;
    const int64_t nb = (N + block_size - 1) / block_size;
    for (int64_t g = 0; g < nb; ++g) {
        const int64_t b = g * block_size;
        const int64_t e = (b + block_size < N) ? b + block_size : N;
        double sum = 0.0;
        for (int64_t i = b; i < e; ++i) sum += token_scores[i];
        out[g] = (float)(sum / (double)(e - b));
    }
    return ORC_OK;
}

/* score_tokens_heads (importance.cpp:92-127) with partial_scores (:17-33) and
 * online_softmax_reduce (:35-74) fused per query row.  The reference materialises every
 * head's n x N raw matrix first; the arithmetic per element and the order in which the
 * shared double accumulator acc[] is updated (head, then row, then key) are identical, so
 * the results are bit-identical while memory stays O(N). */
int orc_score_tokens_heads(const float* q, int64_t q_ld, const float* k, int64_t k_ld, int64_t N,
                           int num_heads, int num_kv_heads, int head_dim, int head_begin,
                           int head_end, const orc_score_config* cfg, float* token_scores,
                           float* block_scores, int32_t* effective_n) {
    if (num_heads <= 0 || num_kv_heads <= 0 || head_dim <= 0) return ORC_ERR_CONTRACT;
    if (num_heads % num_kv_heads != 0) return ORC_ERR_CONTRACT;
    if (head_begin < 0 || head_end > num_heads || head_begin >= head_end) return ORC_ERR_CONTRACT;
    if (N <= 0) return ORC_ERR_CONTRACT; /* block_reduce rejects empty scores */
    if (cfg->query_window_n <= 0) return ORC_ERR_CONFIG;
    if (cfg->block_size_g <= 0) return ORC_ERR_CONTRACT;
    const int group = num_heads / num_kv_heads;
    const int64_t n_eff = cfg->query_window_n < N ? cfg->query_window_n : N;
    if (effective_n) *effective_n = (int32_t)n_eff;

    const double scale = 1.0 / sqrt((double)head_dim);
    const double inv_n = 1.0 / (double)n_eff;
    double* acc = (double*)calloc((size_t)N, sizeof(double));
    float* raw = (float*)malloc((size_t)N * sizeof(float));
    if (!acc || !raw) {
        free(acc);
        free(raw);
        return ORC_ERR_CONTRACT;
    }
    int status = ORC_OK;
    for (int h = head_begin; h < head_end && status == ORC_OK; ++h) {
        const int kvh = h / group;
        for (int64_t j = 0; j < n_eff; ++j) {
            const float* qrow = q + (N - n_eff + j) * q_ld + (int64_t)h * head_dim;
            const int64_t query_pos = N - n_eff + j;
            /* partial_scores row j: float(double dot * scale), -inf past the query. */
            for (int64_t i = 0; i < N; ++i) {
                if (i > query_pos) {
                    raw[i] = -INFINITY;
                    continue;
                }
                const float* krow = k + i * k_ld + (int64_t)kvh * head_dim;
                double dot = 0.0;
                for (int c = 0; c < head_dim; ++c) dot += (double)qrow[c] * (double)krow[c];
                raw[i] = (float)(dot * scale);
            }
            /* Pass 1: running max and denominator in index order (importance.cpp:45-56). */
            double max_logit = -INFINITY;
            double denom = 0.0;
            for (int64_t i = 0; i < N; ++i) {
                const double x = raw[i];
                if (x == -INFINITY) continue;
                if (x > max_logit) {
                    denom = denom * exp(max_logit - x) + 1.0;
                    max_logit = x;
                } else {
                    denom += exp(x - max_logit);
                }
            }
            if (denom <= 0.0 || !isfinite(max_logit)) {
                status = ORC_ERR_CONTRACT; /* fully masked query row (:57-59) */
                break;
            }
            /* Pass 2: normalized weights into the shared accumulator (:61-66). */
            for (int64_t i = 0; i < N; ++i) {
                const double x = raw[i];
                if (x == -INFINITY) continue;
                acc[i] += exp(x - max_logit) / denom * inv_n;
            }
        }
    }
    if (status == ORC_OK) {
        float* ts = token_scores ? token_scores : (float*)malloc((size_t)N * sizeof(float));
        for (int64_t i = 0; i < N; ++i) ts[i] = (float)acc[i];
        status = orc_block_reduce(ts, N, cfg->block_size_g, block_scores);
        if (!token_scores) free(ts);
    }
    free(acc);
    free(raw);
    return status;
}

/* ------------------------------------------------------------------ TP reduction */

/* allreduce_scores (tp_sim.cpp:29-49): ids must be exactly 0..T-1; fp32 sum in ascending
 * shard id starting from 0.0f. */
int orc_allreduce_scores(const float* const* shards, const int32_t* shard_ids, int32_t tp,
                         int64_t length, float* out) {
    if (tp <= 0) return ORC_ERR_CONTRACT;
    const float** by_id = (const float**)calloc((size_t)tp, sizeof(float*));
    for (int32_t t = 0; t < tp; ++t) {
        const int32_t id = shard_ids[t];
        if (id < 0 || id >= tp || by_id[id] != NULL) {
            free(by_id);
            return ORC_ERR_CONTRACT;
        }
        by_id[id] = shards[t];
    }
    for (int64_t g = 0; g < length; ++g) out[g] = 0.0f;
    for (int32_t t = 0; t < tp; ++t) {
        const float* b = by_id[t];
        for (int64_t g = 0; g < length; ++g) out[g] += b[g];
    }
    free(by_id);
    return ORC_OK;
}

/* ------------------------------------------------------------------ selection */

/* expand_mask (selection.cpp:36-49). */
int orc_expand_mask(const uint8_t* block_mask, int64_t num_blocks, int block_size,
                    int64_t num_tokens, int64_t sink_count, int64_t window_n, uint8_t* keep) {
    if (block_size <= 0) return ORC_ERR_CONTRACT;
    if (num_blocks != (num_tokens + block_size - 1) / block_size) return ORC_ERR_CONTRACT;
    for (int64_t i = 0; i < num_tokens; ++i) {
        const int block_kept = block_mask[i / block_size] != 0;
        keep[i] = (block_kept || i < sink_count || i >= num_tokens - window_n) ? 1 : 0;
    }
    return ORC_OK;
}

static int cmp_u64_desc(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? 1 : (x > y ? -1 : 0);
}

/* Token-level covered mass (selection.cpp:108-120, propagation.cpp:126-135). */
static double covered_sum(const uint8_t* keep, int64_t num_tokens, const float* block_scores,
                          int64_t num_blocks, int G) {
    double covered = 0.0;
    for (int64_t g = 0; g < num_blocks; ++g) {
        const int64_t b = g * G;
        const int64_t e = (b + G < num_tokens) ? b + G : num_tokens;
        int64_t kept = 0;
        for (int64_t i = b; i < e; ++i) kept += keep[i];
        covered += (double)block_scores[g] * ((double)kept / (double)(e - b));
    }
    return covered;
}

/* top_p_select (selection.cpp:51-122). */
int orc_top_p_select(const float* block_scores, int64_t num_blocks, const orc_score_config* cfg,
                     int64_t num_tokens, uint8_t* keep, orc_selection_info* info) {
    int st = orc_config_validate(cfg);
    if (st != ORC_OK) return st;
    if (num_tokens < 1) return ORC_ERR_CONTRACT;
    const int G = cfg->block_size_g;
    const int64_t nb = (num_tokens + G - 1) / G;
    if (num_blocks != nb) return ORC_ERR_CONTRACT;

    /* total: sequential double sum in block-index order (:61-67). */
    double total = 0.0;
    for (int64_t g = 0; g < nb; ++g) {
        const float s = block_scores[g];
        if (!(s >= 0.0f) || !isfinite(s)) return ORC_ERR_CONTRACT;
        total += s;
    }
    const int64_t n_eff = cfg->query_window_n < num_tokens ? cfg->query_window_n : num_tokens;
    if (nb < 0) return ORC_ERR_CONTRACT;
    uint8_t* block_mask = (uint8_t*)calloc((size_t)nb + 1, 1);
    int degenerate = 0;
    int64_t k_star = 0;
    if (total <= 0.0) {
        degenerate = 1;
        k_star = nb;
        memset(block_mask, 1, (size_t)nb);
    } else {
        uint64_t* packed = (uint64_t*)malloc((size_t)nb * sizeof(uint64_t));
        for (int64_t g = 0; g < nb; ++g) orc_pack_score(block_scores[g], (uint32_t)g, &packed[g]);
        qsort(packed, (size_t)nb, sizeof(uint64_t), cmp_u64_desc);
        /* cum: sequential double sum of decoded floats in sorted order; the threshold is
         * compared as cum/total >= double(top_p) (:80-93). */
        double cumulative = 0.0;
        const double threshold = (double)cfg->top_p;
        for (int64_t r = 0; r < nb; ++r) {
            const uint64_t w = packed[r];
            cumulative += (double)orc_phi_decode((uint32_t)(w >> 32));
            block_mask[~(uint32_t)(w & 0xFFFFFFFFu)] = 1;
            k_star = r + 1;
            if (cumulative / total >= threshold) break;
        }
        free(packed);
    }
    orc_expand_mask(block_mask, nb, G, num_tokens, cfg->sink_count_a, n_eff, keep);
    free(block_mask);

    int64_t retained = 0;
    for (int64_t i = 0; i < num_tokens; ++i) retained += keep[i];
    info->cutoff_rank = k_star;
    info->retained_count = retained;
    info->retention_ratio = (double)retained / (double)num_tokens;
    info->degenerate_keep_all = degenerate;
    if (degenerate || total <= 0.0) {
        info->covered_mass = 1.0;
    } else {
        info->covered_mass = covered_sum(keep, num_tokens, block_scores, nb, G) / total;
    }
    return ORC_OK;
}

/* Veto + restrict_selection (propagation.cpp:116-136, :173-183): only when the veto
 * actually removes a kept row are retained/ratio/covered recomputed. */
int orc_restrict_selection(uint8_t* keep, const uint8_t* veto, int64_t num_tokens,
                           const float* block_scores, int64_t num_blocks, int block_size,
                           orc_selection_info* info) {
    int changed = 0;
    for (int64_t i = 0; i < num_tokens; ++i) {
        if (keep[i] && veto[i]) {
            keep[i] = 0;
            changed = 1;
        }
    }
    if (!changed) return ORC_OK;
    int64_t retained = 0;
    for (int64_t i = 0; i < num_tokens; ++i) retained += keep[i];
    info->retained_count = retained;
    info->retention_ratio = (double)retained / (double)num_tokens;
    double total = 0.0;
    for (int64_t g = 0; g < num_blocks; ++g) total += block_scores[g];
    const double covered = covered_sum(keep, num_tokens, block_scores, num_blocks, block_size);
    info->covered_mass = total > 0.0 ? covered / total : 1.0;
    return ORC_OK;
}

/* ------------------------------------------------------------------ compaction */

/* patch_metadata (scheduler.cpp:50-90) + apply_drop's stable row compaction
 * (propagation.cpp:47-77): kept rows of selected segments, all rows of the others, in
 * order; new_cu[s+1] = new_cu[s] + kept_s. */
int orc_compact(const uint8_t* keep, const int64_t* cu_seqlens, int32_t num_requests,
                const uint8_t* selected, int32_t n_planes, const void* const* src,
                void* const* dst, const int64_t* row_bytes, int64_t* cu_out,
                int64_t* retained_index, int64_t* num_out) {
    if (num_requests < 0 || cu_seqlens[0] != 0) return ORC_ERR_CONTRACT;
    for (int32_t s = 0; s < num_requests; ++s) {
        if (cu_seqlens[s + 1] <= cu_seqlens[s]) return ORC_ERR_CONTRACT;
    }
    int64_t out = 0;
    cu_out[0] = 0;
    for (int32_t s = 0; s < num_requests; ++s) {
        const int sel = selected == NULL || selected[s] != 0;
        for (int64_t i = cu_seqlens[s]; i < cu_seqlens[s + 1]; ++i) {
            if (sel && !keep[i]) continue;
            for (int32_t p = 0; p < n_planes; ++p) {
                memcpy((char*)dst[p] + out * row_bytes[p], (const char*)src[p] + i * row_bytes[p],
                       (size_t)row_bytes[p]);
            }
            if (retained_index) retained_index[out] = i;
            ++out;
        }
        cu_out[s + 1] = out;
    }
    *num_out = out;
    return ORC_OK;
}

/* ------------------------------------------------------------------ reconstitution & KV metadata */

/* reconstitute (propagation.cpp:79-100): walk positions 0..n-1; a parked position takes
 * its parked row, any other position the next active row (active rows are in position
 * order). */
int orc_reconstitute(const void* active, const int64_t* active_pos, int64_t n_active, const void* parked,
                     const int64_t* parked_pos, int64_t n_parked, int64_t row_bytes, int64_t n_orig,
                     void* out) {
    if (n_active + n_parked != n_orig) return ORC_ERR_CONTRACT;
    int64_t a = 0;
    for (int64_t pos = 0; pos < n_orig; ++pos) {
        int64_t k = -1;
        for (int64_t q = 0; q < n_parked; ++q)
            if (parked_pos[q] == pos) { k = q; break; }
        if (k >= 0) {
            memcpy((char*)out + pos * row_bytes, (const char*)parked + k * row_bytes, (size_t)row_bytes);
        } else {
            if (a >= n_active || active_pos[a] != pos) return ORC_ERR_CONTRACT;
            memcpy((char*)out + pos * row_bytes, (const char*)active + a * row_bytes, (size_t)row_bytes);
            ++a;
        }
    }
    return ORC_OK;
}

/* PagedKVCache::slot_for (kvcache.cpp:67-80). */
int orc_slot_for(const int64_t* table, int64_t table_len, int block_size, int64_t pos, int64_t* slot) {
    if (pos < 0 || block_size <= 0) return ORC_ERR_CONTRACT;
    const int64_t page = pos / block_size;
    if (page >= table_len || table[page] < 0) return ORC_ERR_ALLOCATION_MISS;
    *slot = table[page] * block_size + pos % block_size;
    return ORC_OK;
}

/* decode_seqused (kvcache.cpp:182-186) with DropHistory::last_event_before (:32-39). */
int64_t orc_decode_seqused(int64_t original_length, int64_t decode_appended, int32_t num_events,
                           const int32_t* event_layers, const int64_t* retained_lengths, int32_t layer) {
    int32_t found = -1;
    for (int32_t e = 0; e < num_events; ++e) {
        if (event_layers[e] < layer) found = e;
        else break;
    }
    const int64_t base = found >= 0 ? retained_lengths[found] : original_length;
    return base + decode_appended;
}

/* scoring_flops (flops.cpp:35-39). */
uint64_t orc_scoring_flops(int64_t effective_n, int64_t num_keys, int head_dim, int num_heads) {
    return 2ULL * (uint64_t)effective_n * (uint64_t)num_keys * (uint64_t)head_dim *
           (uint64_t)num_heads;
}
