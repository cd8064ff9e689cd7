/*
 * fusesim_oracle.c -- plain-C restatement of the reference decode path.
 * TEST INFRASTRUCTURE ONLY (see fusesim_oracle.h).  Compiled with
 * -ffp-contract=off so every f32/f64 operation rounds exactly like the
 * reference's -O2 x86-64 build (proj/CMakeLists.txt:8).
 */
#include "fusesim_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static void set_err(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

const char *fo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ */
/* std::mt19937_64 / std::mt19937 (libstdc++ <bits/random.h>)          */
/* ------------------------------------------------------------------ */
void fo_mt64_seed(fo_mt64 *g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static void mt64_gen(fo_mt64 *g) {
    const uint64_t upper = ~0ull << 31, lower = ~upper;
    for (int k = 0; k < 312; ++k) {
        uint64_t y = (g->mt[k] & upper) | (g->mt[(k + 1) % 312] & lower);
        g->mt[k] = g->mt[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ull) ? 0xb5026f5aa96619e9ull : 0ull);
    }
    g->idx = 0;
}

uint64_t fo_mt64_next(fo_mt64 *g) {
    if (g->idx >= 312) mt64_gen(g);
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71d67fffeda60000ull;
    z ^= (z << 37) & 0xfff7eee000000000ull;
    z ^= (z >> 43);
    return z;
}

void fo_mt32_seed(fo_mt32 *g, uint32_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 624; ++i)
        g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
    g->idx = 624;
}

static void mt32_gen(fo_mt32 *g) {
    for (int k = 0; k < 624; ++k) {
        uint32_t y = (g->mt[k] & 0x80000000u) | (g->mt[(k + 1) % 624] & 0x7fffffffu);
        g->mt[k] = g->mt[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    }
    g->idx = 0;
}

uint32_t fo_mt32_next(fo_mt32 *g) {
    if (g->idx >= 624) mt32_gen(g);
    uint32_t z = g->mt[g->idx++];
    z ^= (z >> 11);
    z ^= (z << 7) & 0x9d2c5680u;
    z ^= (z << 15) & 0xefc60000u;
    z ^= (z >> 18);
    return z;
}

/* types.hpp:142-152 */
uint64_t fo_fnv1a(const void *data, uint64_t n, uint64_t seed) {
    const unsigned char *p = (const unsigned char *)data;
    uint64_t h = seed;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

uint64_t fo_fnv1a_str(const char *s) { return fo_fnv1a(s, strlen(s), 0xcbf29ce484222325ull); }

/* generate_canonical<double,53>(mt19937_64): one draw, u / 2^64 (random.tcc:3349-3380) */
static double canon_f64(fo_mt64 *g) {
    double r = (double)fo_mt64_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

/* generate_canonical<float,24>(mt19937_64) */
static float canon_f32(fo_mt64 *g) {
    float r = (float)fo_mt64_next(g) / 18446744073709551616.0f;
    if (r >= 1.0f) r = nextafterf(1.0f, 0.0f);
    return r;
}

/* normal_distribution<double>::operator() (random.tcc:1811-1844), Marsaglia polar */
typedef struct { int saved_ok; double saved; } norm64;
static double normal_f64(norm64 *st, fo_mt64 *g, double mean, double stddev) {
    double ret;
    if (st->saved_ok) {
        st->saved_ok = 0;
        ret = st->saved;
    } else {
        double x, y, r2;
        do {
            x = 2.0 * canon_f64(g) - 1.0;
            y = 2.0 * canon_f64(g) - 1.0;
            r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        double mult = sqrt(-2 * log(r2) / r2);
        st->saved = x * mult;
        st->saved_ok = 1;
        ret = y * mult;
    }
    return ret * stddev + mean;
}

/* normal_distribution<float>: float arithmetic, `- 1.0` promoted to double */
typedef struct { int saved_ok; float saved; } norm32;
static float normal_f32(norm32 *st, fo_mt64 *g, float mean, float stddev) {
    float ret;
    if (st->saved_ok) {
        st->saved_ok = 0;
        ret = st->saved;
    } else {
        float x, y, r2;
        do {
            x = (float)((double)(2.0f * canon_f32(g)) - 1.0);
            y = (float)((double)(2.0f * canon_f32(g)) - 1.0);
            r2 = x * x + y * y;
        } while ((double)r2 > 1.0 || (double)r2 == 0.0);
        float mult = sqrtf(-2.0f * logf(r2) / r2);
        st->saved = x * mult;
        st->saved_ok = 1;
        ret = y * mult;
    }
    return ret * stddev + mean;
}

void fo_normal_f64(uint64_t seed, double mean, double stddev, double *out, int64_t n) {
    fo_mt64 g;
    norm64 st = {0, 0.0};
    fo_mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = normal_f64(&st, &g, mean, stddev);
}

/* ------------------------------------------------------------------ */
/* element helpers                                                      */
/* ------------------------------------------------------------------ */
float fo_bf16_round(float x) { /* types.hpp:50-59 */
    uint32_t bits;
    memcpy(&bits, &x, 4);
    uint32_t lsb = (bits >> 16) & 1u;
    bits += 0x7fffu + lsb;
    bits &= 0xffff0000u;
    float out;
    memcpy(&out, &bits, 4);
    return out;
}

float fo_dequantize_code(uint8_t code, float scale, float zero_point) { /* quant.hpp:23-25 */
    return ((float)code - zero_point) * scale;
}

uint8_t fo_quantize_value(float v, float scale, float zero_point, int32_t levels) {
    float c = roundf(v / scale + zero_point); /* quant.hpp:36-39 */
    if (c < 0.0f) c = 0.0f;
    if (c > (float)levels) c = (float)levels;
    return (uint8_t)c;
}

void fo_quantize_group(const float *values, int64_t n, int32_t levels, uint8_t *codes,
                       float *scale, float *zero_point, float *deq) {
    /* quant.hpp:42-54 (levels=15); the int8 extension uses levels=255 */
    float lo = 0.0f, hi = 0.0f;
    if (n > 0) {
        lo = values[0];
        hi = values[0];
        for (int64_t i = 1; i < n; ++i) {
            if (values[i] < lo) lo = values[i];
            if (hi < values[i]) hi = values[i];
        }
    }
    float range = hi - lo;
    float s = range > 0 ? range / (float)levels : 1.0f;
    float z = roundf(-lo / s);
    if (z < 0.0f) z = 0.0f;
    if (z > (float)levels) z = (float)levels;
    for (int64_t i = 0; i < n; ++i) {
        uint8_t c = fo_quantize_value(values[i], s, z, levels);
        if (codes) codes[i] = c;
        if (deq) deq[i] = fo_dequantize_code(c, s, z);
    }
    *scale = s;
    *zero_point = z;
}

/* ------------------------------------------------------------------ */
/* config / layout                                                      */
/* ------------------------------------------------------------------ */
int64_t fo_qkv_rows(const fo_config *c) {
    return c->n_q_heads * c->d_head + 2 * c->n_kv_heads * c->d_head;
}

int fo_validate(const fo_config *c) { /* config.hpp:61-83 (decoder kind) */
    if (c->layers < 0) { set_err("model: layers must be >= 0"); return 2; }
    if (c->d_model <= 0) { set_err("model: d_model must be positive"); return 2; }
    if (c->batch < 1 || c->batch > 16) { set_err("model: batch must be in [1,16]"); return 2; }
    if (c->d_inter <= 0) { set_err("model: d_inter must be positive"); return 2; }
    if (c->d_head <= 0 || c->d_head % 2 != 0) {
        set_err("model: d_head must be positive and even");
        return 2;
    }
    if (c->n_q_heads <= 0 || c->n_kv_heads <= 0) {
        set_err("model: head counts must be positive");
        return 2;
    }
    if (c->n_q_heads % c->n_kv_heads != 0) {
        set_err("model: GQA grouping requires n_q_heads mod n_kv_heads == 0");
        return 2;
    }
    if (c->d_model != c->n_q_heads * c->d_head) {
        set_err("model: d_model must equal n_q_heads * d_head");
        return 2;
    }
    if (c->vocab_size <= 0) { set_err("model: vocab_size must be positive"); return 2; }
    if (c->quant_bits != 0) {
        if (c->quant_bits != 4 && c->quant_bits != 8) {
            set_err("quant: only 4-bit (reference) and 8-bit (extension) codes are supported");
            return 2;
        }
        if (c->quant_group <= 0) { set_err("quant: group_size must be positive"); return 2; }
        if (c->d_model % c->quant_group != 0) {
            set_err("quant: group_size must divide every quantized row length");
            return 2;
        }
    }
    return 0;
}

static uint64_t row_bytes(const fo_config *c, int64_t cols) { /* tensor_store.hpp:29-32 */
    if (c->quant_bits == 4) return (uint64_t)cols / 2 + (uint64_t)(cols / c->quant_group) * 4;
    if (c->quant_bits == 8) return (uint64_t)cols + (uint64_t)(cols / c->quant_group) * 4;
    return (uint64_t)cols * (c->dtype == 0 ? 2 : 4);
}

uint64_t fo_streamed_weight_bytes(const fo_config *c) { /* tensor_store.hpp:170-174 */
    uint64_t per_layer = (uint64_t)fo_qkv_rows(c) * row_bytes(c, c->d_model) +
                         (uint64_t)c->d_model * row_bytes(c, c->d_model) +
                         (uint64_t)(2 * c->d_inter) * row_bytes(c, c->d_model) +
                         (uint64_t)c->d_inter * row_bytes(c, c->d_model);
    return per_layer * (uint64_t)c->layers + (uint64_t)c->vocab_size * row_bytes(c, c->d_model);
}

uint64_t fo_total_weight_bytes(const fo_config *c) { /* tensor_store.hpp:178-186 */
    uint64_t eb = c->dtype == 0 ? 2 : 4;
    return fo_streamed_weight_bytes(c) + (uint64_t)c->vocab_size * c->d_model * eb +
           (uint64_t)(2 * c->layers + 1) * c->d_model * eb;
}

/* ------------------------------------------------------------------ */
/* init_weights (tensor_store.hpp:270-366)                              */
/* ------------------------------------------------------------------ */
typedef struct fill_job {
    char name[64];
    float *dst;
    int64_t rows, cols;
    double fan_in_scale;
    int kind; /* 0 = matrix (quantizable), 1 = norm vector, 2 = embedding (never quantized) */
} fill_job;

typedef struct fill_ctx {
    const fo_config *cfg;
    uint64_t seed;
    fill_job *jobs;
    int njobs;
    int next;
    pthread_mutex_t mu;
} fill_ctx;

static void run_fill(const fo_config *cfg, uint64_t seed, const fill_job *j) {
    fo_mt64 g;
    fo_mt64_seed(&g, seed ^ fo_fnv1a_str(j->name));
    int64_t n = j->rows * j->cols;
    if (j->kind == 1) { /* fill_vector: N(1, 0.02), not rounded */
        norm64 st = {0, 0.0};
        for (int64_t i = 0; i < n; ++i) j->dst[i] = (float)normal_f64(&st, &g, 1.0, 0.02);
        return;
    }
    norm64 st = {0, 0.0};
    for (int64_t i = 0; i < n; ++i) j->dst[i] = (float)normal_f64(&st, &g, 0.0, j->fan_in_scale);
    int quantize = (j->kind == 0) && cfg->quant_bits != 0;
    if (quantize) {
        int32_t levels = cfg->quant_bits == 4 ? 15 : 255;
        int64_t gs = cfg->quant_group;
        float s, z;
        for (int64_t r = 0; r < j->rows; ++r)
            for (int64_t c0 = 0; c0 < j->cols; c0 += gs) {
                float *grp = j->dst + r * j->cols + c0;
                fo_quantize_group(grp, gs, levels, NULL, &s, &z, grp);
            }
    } else if (cfg->dtype == 0) {
        for (int64_t i = 0; i < n; ++i) j->dst[i] = fo_bf16_round(j->dst[i]);
    }
}

static void *fill_worker(void *arg) {
    fill_ctx *ctx = (fill_ctx *)arg;
    for (;;) {
        pthread_mutex_lock(&ctx->mu);
        int i = ctx->next++;
        pthread_mutex_unlock(&ctx->mu);
        if (i >= ctx->njobs) break;
        run_fill(ctx->cfg, ctx->seed, &ctx->jobs[i]);
    }
    return NULL;
}

static float *alloc_f32(int64_t n) {
    float *p = (float *)calloc((size_t)(n > 0 ? n : 1), sizeof(float));
    return p;
}

void fo_free(fo_store *s) {
    if (!s) return;
    if (s->layers) {
        for (int64_t l = 0; l < s->cfg.layers; ++l) {
            free(s->layers[l].wqkv);
            free(s->layers[l].waout);
            free(s->layers[l].wffn1);
            free(s->layers[l].wffn2t);
            free(s->layers[l].norm_attn);
            free(s->layers[l].norm_ffn);
        }
        free(s->layers);
    }
    free(s->final_norm);
    free(s->embedding);
    free(s->lm_head);
    free(s->k);
    free(s->v);
    free(s->kv_len);
    free(s);
}

/* TensorStore shapes (tensor_store.hpp:304-366) with zeroed values and an
 * empty KV cache [B][L][Hkv][S][dh]. */
static fo_store *store_alloc(const fo_config *c, int64_t max_seq_len) {
    fo_store *s = (fo_store *)calloc(1, sizeof(fo_store));
    s->cfg = *c;
    s->max_seq_len = max_seq_len;
    const int64_t d = c->d_model;
    s->layers = (fo_layer *)calloc((size_t)(c->layers > 0 ? c->layers : 1), sizeof(fo_layer));
    for (int64_t l = 0; l < c->layers; ++l) {
        fo_layer *L = &s->layers[l];
        L->wqkv = alloc_f32(fo_qkv_rows(c) * d);
        L->waout = alloc_f32(d * d);
        L->wffn1 = alloc_f32(2 * c->d_inter * d);
        L->wffn2t = alloc_f32(c->d_inter * d);
        L->norm_attn = alloc_f32(d);
        L->norm_ffn = alloc_f32(d);
    }
    s->final_norm = alloc_f32(d);
    s->embedding = alloc_f32(c->vocab_size * d);
    s->lm_head = alloc_f32(c->vocab_size * d);
    size_t kv = (size_t)c->batch * c->layers * c->n_kv_heads * max_seq_len * c->d_head;
    s->k = alloc_f32((int64_t)kv);
    s->v = alloc_f32((int64_t)kv);
    s->kv_len = (int64_t *)calloc((size_t)(c->layers > 0 ? c->layers : 1), sizeof(int64_t));
    return s;
}

fo_store *fo_init_weights(const fo_config *c, uint64_t seed, int64_t max_seq_len, int nthreads) {
    if (fo_validate(c)) return NULL;
    fo_store *s = store_alloc(c, max_seq_len);
    const int64_t d = c->d_model;
    int njobs = (int)(6 * c->layers + 3);
    fill_job *jobs = (fill_job *)calloc((size_t)njobs, sizeof(fill_job));
    int j = 0;
    /* fan-in: d_inter for the GLU output projection, stored cols otherwise (:330-333) */
    double sd_d = 1.0 / sqrt((double)d), sd_i = 1.0 / sqrt((double)c->d_inter);
    for (int64_t l = 0; l < c->layers; ++l) {
        fo_layer *L = &s->layers[l];
#define JOB(NAME, DST, R, C, SD, K)                                                        \
    do {                                                                                   \
        snprintf(jobs[j].name, sizeof(jobs[j].name), "layer.%lld." NAME, (long long)l);   \
        jobs[j].dst = (DST); jobs[j].rows = (R); jobs[j].cols = (C);                       \
        jobs[j].fan_in_scale = (SD); jobs[j].kind = (K); ++j;                              \
    } while (0)
        JOB("wqkv", L->wqkv, fo_qkv_rows(c), d, sd_d, 0);
        JOB("waout", L->waout, d, d, sd_d, 0);
        JOB("wffn1", L->wffn1, 2 * c->d_inter, d, sd_d, 0);
        JOB("wffn2t", L->wffn2t, c->d_inter, d, sd_i, 0);
        JOB("norm_attn", L->norm_attn, 1, d, 0.0, 1);
        JOB("norm_ffn", L->norm_ffn, 1, d, 0.0, 1);
#undef JOB
    }
    snprintf(jobs[j].name, 64, "final_norm");
    jobs[j].dst = s->final_norm; jobs[j].rows = 1; jobs[j].cols = d; jobs[j].kind = 1; ++j;
    snprintf(jobs[j].name, 64, "embedding");
    jobs[j].dst = s->embedding; jobs[j].rows = c->vocab_size; jobs[j].cols = d;
    jobs[j].fan_in_scale = sd_d; jobs[j].kind = 2; ++j;
    snprintf(jobs[j].name, 64, "lm_head");
    jobs[j].dst = s->lm_head; jobs[j].rows = c->vocab_size; jobs[j].cols = d;
    jobs[j].fan_in_scale = sd_d; jobs[j].kind = 0; ++j;

    /* biggest jobs first so the per-tensor parallelism balances */
    for (int a = 0; a < njobs; ++a)
        for (int b = a + 1; b < njobs; ++b)
            if (jobs[b].rows * jobs[b].cols > jobs[a].rows * jobs[a].cols) {
                fill_job t = jobs[a]; jobs[a] = jobs[b]; jobs[b] = t;
            }
    fill_ctx ctx;
    ctx.cfg = &s->cfg; ctx.seed = seed; ctx.jobs = jobs; ctx.njobs = njobs; ctx.next = 0;
    pthread_mutex_init(&ctx.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 64) nthreads = 64;
    pthread_t th[64];
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, fill_worker, &ctx);
    fill_worker(&ctx);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&ctx.mu);
    free(jobs);
    return s;
}

/* ------------------------------------------------------------------ */
/* KV cache (tensor_store.hpp:63-150)                                   */
/* ------------------------------------------------------------------ */
static size_t kv_index(const fo_store *s, int64_t b, int64_t l, int64_t h, int64_t pos) {
    const fo_config *c = &s->cfg;
    return ((((size_t)b * c->layers + l) * c->n_kv_heads + h) * s->max_seq_len + pos) *
           c->d_head;
}

static float round_store(const fo_store *s, float x) {
    return s->cfg.dtype == 0 ? fo_bf16_round(x) : x;
}

float *fo_k_at(fo_store *s, int64_t b, int64_t l, int64_t h, int64_t pos) {
    return s->k + kv_index(s, b, l, h, pos);
}
float *fo_v_at(fo_store *s, int64_t b, int64_t l, int64_t h, int64_t pos) {
    return s->v + kv_index(s, b, l, h, pos);
}

void fo_kv_set_position(fo_store *s, int64_t b, int64_t l, int64_t h, int64_t pos,
                        const float *k, const float *v) {
    float *kd = fo_k_at(s, b, l, h, pos), *vd = fo_v_at(s, b, l, h, pos);
    for (int64_t d = 0; d < s->cfg.d_head; ++d) {
        kd[d] = round_store(s, k[d]);
        vd[d] = round_store(s, v[d]);
    }
}

void fo_kv_set_length(fo_store *s, int64_t layer, int64_t n) { s->kv_len[layer] = n; }
int64_t fo_kv_length(const fo_store *s, int64_t layer) { return s->kv_len[layer]; }

void fo_synthetic_prefill(fo_store *s, int64_t prefill, uint64_t seed) {
    const fo_config *c = &s->cfg;
    fo_mt64 g;
    norm32 st = {0, 0.0f};
    fo_mt64_seed(&g, seed);
    float *k = alloc_f32(c->d_head), *v = alloc_f32(c->d_head);
    for (int64_t b = 0; b < c->batch; ++b)
        for (int64_t l = 0; l < c->layers; ++l)
            for (int64_t h = 0; h < c->n_kv_heads; ++h)
                for (int64_t p = 0; p < prefill; ++p) {
                    for (int64_t i = 0; i < c->d_head; ++i) k[i] = normal_f32(&st, &g, 0.0f, 0.3f);
                    for (int64_t i = 0; i < c->d_head; ++i) v[i] = normal_f32(&st, &g, 0.0f, 0.3f);
                    fo_kv_set_position(s, b, l, h, p, k, v);
                }
    for (int64_t l = 0; l < c->layers; ++l) s->kv_len[l] = prefill;
    free(k);
    free(v);
}

/* ------------------------------------------------------------------ */
/* numerics (numerics.hpp)                                              */
/* ------------------------------------------------------------------ */
void fo_rmsnorm_f64(const double *x, const double *w, int64_t n, double eps, double *y) {
    double ms = 0; /* numerics.hpp:14-24 */
    for (int64_t i = 0; i < n; ++i) ms += x[i] * x[i];
    ms /= (double)n;
    double inv = 1.0 / sqrt(ms + eps);
    for (int64_t i = 0; i < n; ++i) y[i] = w[i] * x[i] * inv;
}

void fo_rope_f64(double *v, int64_t d_head, int64_t pos, double theta) {
    for (int64_t k = 0; k < d_head / 2; ++k) { /* numerics.hpp:27-37 */
        double freq = pow(theta, -(double)(2 * k) / (double)d_head);
        double angle = (double)pos * freq;
        double c = cos(angle), s = sin(angle);
        double a = v[2 * k], b = v[2 * k + 1];
        v[2 * k] = a * c - b * s;
        v[2 * k + 1] = a * s + b * c;
    }
}

double fo_silu(double z) { return z / (1.0 + exp(-z)); } /* numerics.hpp:46 */

int64_t fo_argmax_f64(const double *logits, int64_t n) { /* numerics.hpp:169-175 */
    int64_t best = 0;
    for (int64_t i = 1; i < n; ++i)
        if (logits[i] > logits[best]) best = i;
    return best;
}

void fo_attn_partial_update(double *m, double *l, double *o, int64_t d, const double *q,
                            const double *k_rows, const double *v_rows, int64_t rows,
                            double alpha) {
    if (rows == 0) return; /* numerics.hpp:76-98 */
    double *s = (double *)malloc(sizeof(double) * (size_t)rows);
    double chunk_max = -INFINITY;
    for (int64_t j = 0; j < rows; ++j) {
        double dot = 0;
        for (int64_t k = 0; k < d; ++k) dot += q[k] * k_rows[j * d + k];
        s[j] = alpha * dot;
        chunk_max = chunk_max > s[j] ? chunk_max : s[j];
    }
    double m_new = *m > chunk_max ? *m : chunk_max;
    double scale = (*l == 0.0) ? 0.0 : exp(*m - m_new);
    *l *= scale;
    for (int64_t k = 0; k < d; ++k) o[k] *= scale;
    for (int64_t j = 0; j < rows; ++j) {
        double w = exp(s[j] - m_new);
        *l += w;
        for (int64_t k = 0; k < d; ++k) o[k] += w * v_rows[j * d + k];
    }
    *m = m_new;
    free(s);
}

int fo_attn_reduce(const double *m, const double *l, const double *o, int64_t n_partials,
                   int64_t d, double *out) {
    double M = -INFINITY; /* numerics.hpp:123-145 */
    int any = 0;
    for (int64_t i = 0; i < n_partials; ++i)
        if (l[i] != 0.0) {
            M = M > m[i] ? M : m[i];
            any = 1;
        }
    if (!any) {
        set_err("attn_reduce: all partials empty");
        return 2;
    }
    double L = 0;
    for (int64_t i = 0; i < n_partials; ++i)
        if (l[i] != 0.0) L += l[i] * exp(m[i] - M);
    for (int64_t k = 0; k < d; ++k) out[k] = 0.0;
    for (int64_t i = 0; i < n_partials; ++i) {
        if (l[i] == 0.0) continue;
        double r = exp(m[i] - M) / L;
        for (int64_t k = 0; k < d; ++k) out[k] += r * o[i * d + k];
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* reference_forward (reference.hpp:37-139)                             */
/* ------------------------------------------------------------------ */
/* y[b * ystride + r] = sum_c w[r][c] * u_b[c] for every batch row b at once
 * (reference.hpp:21-30).  ut holds the inputs transposed, [cols][B], so one
 * pass over a weight row feeds every batch row.  Each (r, b) is still one
 * sequential f64 sum in column order with a separately rounded product
 * (-ffp-contract=off), so the result is bit-identical to the reference's
 * per-row loop for any thread count. */
#define FO_BBLK 16
static void matvec_batch(const float *w, int64_t rows, int64_t cols, const double *ut, int64_t B,
                         double *y, int64_t ystride) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        const float *row = w + r * cols;
        for (int64_t b0 = 0; b0 < B; b0 += FO_BBLK) {
            const int64_t nb = B - b0 < FO_BBLK ? B - b0 : FO_BBLK;
            double acc[FO_BBLK] = {0};
            if (nb == FO_BBLK) { /* fixed trip count: accumulators stay in registers */
                for (int64_t c = 0; c < cols; ++c) {
                    const double wc = (double)row[c];
                    const double *uc = ut + c * B + b0;
                    for (int b = 0; b < FO_BBLK; ++b) acc[b] += wc * uc[b];
                }
            } else {
                for (int64_t c = 0; c < cols; ++c) {
                    const double wc = (double)row[c];
                    const double *uc = ut + c * B + b0;
                    for (int64_t b = 0; b < nb; ++b) acc[b] += wc * uc[b];
                }
            }
            for (int64_t b = 0; b < nb; ++b) y[(b0 + b) * ystride + r] = acc[b];
        }
    }
}

static void transpose_in(const double *u, int64_t B, int64_t n, double *ut) { /* [B][n] -> [n][B] */
    for (int64_t b = 0; b < B; ++b)
        for (int64_t i = 0; i < n; ++i) ut[i * B + b] = u[b * n + i];
}

static void widen(const float *src, int64_t n, double *dst) {
    for (int64_t i = 0; i < n; ++i) dst[i] = (double)src[i];
}

int fo_reference_forward(fo_store *s, const int64_t *tokens, int64_t pos, double *logits) {
    return fo_reference_forward_ex(s, tokens, pos, logits, NULL, NULL);
}

/* reference_forward (reference.hpp:37-139).  The reference walks the batch
 * rows one after another inside each layer; rows never interact (only the
 * KV append, which lands for every row before any attention reads it), so
 * this restatement runs them side by side -- same per-element arithmetic,
 * one pass over each weight matrix per layer. */
int fo_reference_forward_ex(fo_store *s, const int64_t *tokens, int64_t pos, double *logits,
                            const float *k_app, const float *v_app) {
    const fo_config *m = &s->cfg;
    const int64_t B = m->batch, D = m->d_model, dh = m->d_head, nq = m->n_q_heads,
                  nkv = m->n_kv_heads, qpg = nq / nkv, V = m->vocab_size, DI = m->d_inter;
    const double alpha = 1.0 / sqrt((double)dh);
    for (int64_t b = 0; b < B; ++b)
        if (tokens[b] < 0 || tokens[b] >= V) {
            set_err("reference_forward: token id out of range");
            return 2;
        }
    const int64_t qkvr = fo_qkv_rows(m);
    const int64_t DIc = DI > 0 ? DI : 1;
    double *x = (double *)malloc(sizeof(double) * (size_t)(B * D));
    double *u = (double *)malloc(sizeof(double) * (size_t)(B * D));
    double *ut = (double *)malloc(sizeof(double) * (size_t)(B * (D > nq * dh ? D : nq * dh)));
    double *w = (double *)malloc(sizeof(double) * (size_t)D);
    double *qkv = (double *)malloc(sizeof(double) * (size_t)(B * qkvr));
    float *krow = (float *)malloc(sizeof(float) * (size_t)(B * nkv * dh));
    float *vrow = (float *)malloc(sizeof(float) * (size_t)(B * nkv * dh));
    double *attn = (double *)malloc(sizeof(double) * (size_t)(B * nq * dh));
    double *aout = (double *)malloc(sizeof(double) * (size_t)(B * D));
    double *scores = (double *)malloc(sizeof(double) * (size_t)(nq * (pos + 1)));
    double *hbuf = (double *)malloc(sizeof(double) * (size_t)(DIc * B));
    int rc = 0;

    for (int64_t b = 0; b < B; ++b) widen(s->embedding + tokens[b] * D, D, x + b * D);

    for (int64_t l = 0; l < m->layers; ++l) {
        const fo_layer *lw = &s->layers[l];
        if (s->kv_len[l] != pos) {
            set_err("reference_forward: cache length does not match position");
            rc = 2;
            goto done;
        }
        widen(lw->norm_attn, D, w);
        for (int64_t b = 0; b < B; ++b) fo_rmsnorm_f64(x + b * D, w, D, m->rmsnorm_eps, u + b * D);
        transpose_in(u, B, D, ut);
        matvec_batch(lw->wqkv, qkvr, D, ut, B, qkv, qkvr);
        for (int64_t b = 0; b < B; ++b) {
            double *qb = qkv + b * qkvr;
            for (int64_t h = 0; h < nq; ++h) fo_rope_f64(qb + h * dh, dh, pos, m->rope_theta);
            for (int64_t h = 0; h < nkv; ++h) {
                double *k = qb + (nq + h) * dh;
                fo_rope_f64(k, dh, pos, m->rope_theta);
                for (int64_t d = 0; d < dh; ++d) {
                    krow[b * nkv * dh + h * dh + d] = (float)k[d];
                    vrow[b * nkv * dh + h * dh + d] = (float)qb[(nq + nkv + h) * dh + d];
                }
            }
        }
        /* append_token: every row lands, then the length advances once (:102-106) */
        if (pos >= s->max_seq_len) {
            set_err("kv_append: cache capacity reached (max_seq_len)");
            rc = 2;
            goto done;
        }
        if (k_app && v_app) { /* checker hook: append externally rounded rows */
            for (int64_t b = 0; b < B; ++b)
                for (int64_t i = 0; i < nkv * dh; ++i) {
                    krow[b * nkv * dh + i] = k_app[(b * m->layers + l) * nkv * dh + i];
                    vrow[b * nkv * dh + i] = v_app[(b * m->layers + l) * nkv * dh + i];
                }
        }
        for (int64_t b = 0; b < B; ++b)
            for (int64_t h = 0; h < nkv; ++h)
                fo_kv_set_position(s, b, l, h, pos, krow + b * nkv * dh + h * dh,
                                   vrow + b * nkv * dh + h * dh);
        s->kv_len[l] += 1;

        for (int64_t b = 0; b < B; ++b) {
            double *ab = attn + b * nq * dh;
            for (int64_t i = 0; i < nq * dh; ++i) ab[i] = 0.0;
            /* heads are independent: one per thread, each with its own score row */
#pragma omp parallel for schedule(dynamic, 1)
            for (int64_t h = 0; h < nq; ++h) {
                int64_t kvh = h / qpg;
                const double *qh = qkv + b * qkvr + h * dh;
                int64_t n = pos + 1;
                double *sc = scores + h * (pos + 1);
                double mx = -INFINITY;
                for (int64_t j = 0; j < n; ++j) {
                    const float *kj = fo_k_at(s, b, l, kvh, j);
                    double dot = 0;
                    for (int64_t d = 0; d < dh; ++d) dot += qh[d] * (double)kj[d];
                    sc[j] = alpha * dot;
                    mx = mx > sc[j] ? mx : sc[j];
                }
                double denom = 0;
                for (int64_t j = 0; j < n; ++j) denom += exp(sc[j] - mx);
                for (int64_t j = 0; j < n; ++j) {
                    double wj = exp(sc[j] - mx) / denom;
                    const float *vj = fo_v_at(s, b, l, kvh, j);
                    for (int64_t d = 0; d < dh; ++d) ab[h * dh + d] += wj * (double)vj[d];
                }
            }
        }
        transpose_in(attn, B, nq * dh, ut);
        matvec_batch(lw->waout, D, nq * dh, ut, B, aout, D);
        for (int64_t i = 0; i < B * D; ++i) x[i] += aout[i];

        /* reference.hpp:114-128 in two parallel passes with the same
         * per-element operation order: h[t] for every pair t, then
         * x[k] += h[t] * wffn2t[t][k] in increasing t for each k. */
        widen(lw->norm_ffn, D, w);
        for (int64_t b = 0; b < B; ++b) fo_rmsnorm_f64(x + b * D, w, D, m->rmsnorm_eps, u + b * D);
        transpose_in(u, B, D, ut);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < DI; ++t) {
            const float *in_row = lw->wffn1 + (2 * t) * D;
            const float *gate_row = lw->wffn1 + (2 * t + 1) * D;
            for (int64_t b0 = 0; b0 < B; b0 += FO_BBLK) {
                const int64_t nb = B - b0 < FO_BBLK ? B - b0 : FO_BBLK;
                double a[FO_BBLK] = {0}, g[FO_BBLK] = {0};
                for (int64_t c = 0; c < D; ++c) {
                    const double wi = (double)in_row[c], wg = (double)gate_row[c];
                    const double *uc = ut + c * B + b0;
                    for (int64_t b = 0; b < nb; ++b) {
                        a[b] += wi * uc[b];
                        g[b] += wg * uc[b];
                    }
                }
                for (int64_t b = 0; b < nb; ++b) hbuf[t * B + b0 + b] = fo_silu(g[b]) * a[b];
            }
        }
#pragma omp parallel for schedule(static)
        for (int64_t k0 = 0; k0 < D; k0 += 64) {
            int64_t k1 = k0 + 64 < D ? k0 + 64 : D;
            for (int64_t t = 0; t < DI; ++t) {
                const float *col = lw->wffn2t + t * D;
                for (int64_t b = 0; b < B; ++b) {
                    const double hh = hbuf[t * B + b];
                    double *xb = x + b * D;
                    for (int64_t k = k0; k < k1; ++k) xb[k] += hh * (double)col[k];
                }
            }
        }
    }
    widen(s->final_norm, D, w);
    for (int64_t b = 0; b < B; ++b) fo_rmsnorm_f64(x + b * D, w, D, m->rmsnorm_eps, u + b * D);
    transpose_in(u, B, D, ut);
    matvec_batch(s->lm_head, V, D, ut, B, logits, V);
done:
    free(x); free(u); free(ut); free(w); free(qkv); free(krow); free(vrow);
    free(attn); free(aout); free(scores); free(hbuf);
    return rc;
}

/* ------------------------------------------------------------------ */
/* Stacked-linear kind                                                  */
/* ------------------------------------------------------------------ */
/* fill_matrix of one named tensor (tensor_store.hpp:270-290) with the
 * stacked-linear rules: fan-in = cols, never quantized (weight_meta,
 * tensor_store.hpp:199-210), bf16-rounded when dtype == 0. */
void fo_fill_linear(const char *name, int64_t rows, int64_t cols, uint64_t seed, int32_t dtype,
                    float *dst) {
    fo_config c;
    memset(&c, 0, sizeof(c));
    c.dtype = dtype;
    fill_job j;
    memset(&j, 0, sizeof(j));
    snprintf(j.name, sizeof(j.name), "%s", name);
    j.dst = dst;
    j.rows = rows;
    j.cols = cols;
    j.fan_in_scale = 1.0 / sqrt((double)cols);
    j.kind = 2;
    run_fill(&c, seed, &j);
}

/* reference_linear_forward (reference.hpp:141-152): x <- W_l x for every
 * layer, f64 accumulation of f32 weights; w = [layers][d][d] row-major. */
void fo_linear_forward(const float *w, int64_t layers, int64_t d, int64_t batch, const float *x0,
                       double *out) {
    double *x = (double *)malloc(sizeof(double) * d), *y = (double *)malloc(sizeof(double) * d);
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t i = 0; i < d; ++i) x[i] = (double)x0[b * d + i];
        for (int64_t l = 0; l < layers; ++l) {
            const float *wl = w + (size_t)l * d * d;
            for (int64_t r = 0; r < d; ++r) {
                double acc = 0.0;
                const float *row = wl + (size_t)r * d;
                for (int64_t c2 = 0; c2 < d; ++c2) acc += (double)row[c2] * x[c2];
                y[r] = acc;
            }
            double *t = x;
            x = y;
            y = t;
        }
        for (int64_t i = 0; i < d; ++i) out[b * d + i] = x[i];
    }
    free(x);
    free(y);
}

/* ------------------------------------------------------------------ */
/* Weight fixture container "FSTW" v1 (tensor_store.hpp:367-482)        */
/* ------------------------------------------------------------------ */
/* Layout (little-endian u64 fields, detail::put_u64/put_str/put_floats,
 * tensor_store.hpp:374-397):
 *   magic 0x46535457, version 1, str(serialize(RunConfig{model}))
 *   u64 n_layers, per layer: matrix(wqkv) matrix(waout) matrix(wffn1)
 *   matrix(wffn2t) floats(norm_attn) floats(norm_ffn); floats(final_norm)
 *   matrix(embedding) matrix(lm_head)
 *   matrix = str(name) u64(dtype) u64(rows) u64(cols) floats(values)
 *   str = u64 n + bytes; floats = u64 n + n f32.
 * The config text is serialize() (config.hpp:245-287) of a RunConfig whose
 * hardware / pipeline / run sections hold the defaults (config.hpp:88-140),
 * so a store saved here is byte-identical to the reference's save_store. */
#define FO_STORE_MAGIC 0x46535457ull
#define FO_STORE_VERSION 1ull

static int put_u64(FILE *f, uint64_t v) { return fwrite(&v, 8, 1, f) == 1 ? 0 : -1; }
static int put_bytes(FILE *f, const void *p, uint64_t n) {
    if (put_u64(f, n)) return -1;
    return (n == 0 || fwrite(p, 1, (size_t)n, f) == (size_t)n) ? 0 : -1;
}
static int put_floats(FILE *f, const float *v, uint64_t n) {
    if (put_u64(f, n)) return -1;
    return (n == 0 || fwrite(v, 4, (size_t)n, f) == (size_t)n) ? 0 : -1;
}
static int put_matrix(FILE *f, const char *name, int32_t dtype, int64_t rows, int64_t cols,
                      const float *v) {
    if (put_bytes(f, name, strlen(name)) || put_u64(f, (uint64_t)dtype) ||
        put_u64(f, (uint64_t)rows) || put_u64(f, (uint64_t)cols))
        return -1;
    return put_floats(f, v, (uint64_t)(rows * cols));
}

/* serialize(RunConfig) for the decoder kind with default hardware/pipeline/run */
int64_t fo_serialize_config(const fo_config *c, char *out, int64_t cap) {
    char q[256] = "";
    if (c->quant_bits)
        snprintf(q, sizeof q,
                 "quant_bits = %d\nquant_group_size = %d\nquant_scheme = weight_only_affine\n",
                 c->quant_bits, c->quant_group);
    int n = snprintf(out, (size_t)(cap > 0 ? cap : 0),
        "[model]\nkind = llama_decoder\nlayers = %lld\nd_model = %lld\nd_inter = %lld\n"
        "d_head = %lld\nn_q_heads = %lld\nn_kv_heads = %lld\nvocab_size = %lld\n"
        "rope_theta = %.17g\nrmsnorm_eps = %.17g\ndtype = %s\nbatch = %lld\n%s"
        "\n[hardware]\nnum_sms = 132\nshared_mem_per_sm = %llu\nregisters_per_sm = %llu\n"
        "hbm_capacity = %llu\npeak_bandwidth = %.17g\nkernel_launch_overhead = %.17g\n"
        "barrier_latency = %.17g\ncompute_throughput_per_sm = %.17g\n"
        "\n[pipeline]\nstage_size = %llu\ndepth = 3\nconsumer_warps = 8\n"
        "\n[run]\nmode = fused_overlap\nseq_len = 0\nseed = 0\n",
        (long long)c->layers, (long long)c->d_model, (long long)c->d_inter,
        (long long)c->d_head, (long long)c->n_q_heads, (long long)c->n_kv_heads,
        (long long)c->vocab_size, c->rope_theta, c->rmsnorm_eps,
        c->dtype == 0 ? "bf16" : "fp32", (long long)c->batch, q,
        228ull * 1024, 256ull * 1024, 80ull * 1000 * 1000 * 1000, 3.35e12, 8e-6, 3e-7, 8e10,
        64ull * 1024);
    return n;
}

int fo_save_store(const fo_store *s, const char *path) { /* tensor_store.hpp:410-444 */
    FILE *f = fopen(path, "wb");
    if (!f) {
        set_err("save_store: cannot open %s", path);
        return 1;
    }
    const fo_config *c = &s->cfg;
    const int64_t d = c->d_model;
    char text[2048];
    int64_t tn = fo_serialize_config(c, text, sizeof text);
    int bad = put_u64(f, FO_STORE_MAGIC) || put_u64(f, FO_STORE_VERSION) ||
              put_bytes(f, text, (uint64_t)tn) || put_u64(f, (uint64_t)c->layers);
    char name[64];
    for (int64_t l = 0; l < c->layers && !bad; ++l) {
        const fo_layer *L = &s->layers[l];
#define PM(T, PTR, R)                                                            \
    snprintf(name, sizeof name, "layer.%lld." T, (long long)l);                  \
    bad = bad || put_matrix(f, name, c->dtype, (R), d, (PTR));
        PM("wqkv", L->wqkv, fo_qkv_rows(c))
        PM("waout", L->waout, d)
        PM("wffn1", L->wffn1, 2 * c->d_inter)
        PM("wffn2t", L->wffn2t, c->d_inter)
#undef PM
        bad = bad || put_floats(f, L->norm_attn, (uint64_t)d) ||
              put_floats(f, L->norm_ffn, (uint64_t)d);
    }
    bad = bad || put_floats(f, s->final_norm, (uint64_t)d) ||
          put_matrix(f, "embedding", c->dtype, c->vocab_size, d, s->embedding) ||
          put_matrix(f, "lm_head", c->dtype, c->vocab_size, d, s->lm_head);
    bad = fclose(f) || bad;
    if (bad) {
        set_err("save_store: write failed on %s", path);
        return 1;
    }
    return 0;
}

static int get_u64(FILE *f, uint64_t *v) { return fread(v, 8, 1, f) == 1 ? 0 : -1; }

/* floats(n) into dst when n == want */
static int get_floats_into(FILE *f, float *dst, uint64_t want, const char *what) {
    uint64_t n;
    if (get_u64(f, &n)) { set_err("load_store: truncated file (%s)", what); return -1; }
    if (n != want) {
        set_err("load_store: %s has %llu values, expected %llu", what, (unsigned long long)n,
                (unsigned long long)want);
        return -1;
    }
    if (n && fread(dst, 4, (size_t)n, f) != (size_t)n) {
        set_err("load_store: truncated file (%s)", what);
        return -1;
    }
    return 0;
}

static int get_matrix_into(FILE *f, float *dst, const char *want_name, int64_t rows,
                           int64_t cols) {
    uint64_t n, dt, r, cc;
    char name[128];
    if (get_u64(f, &n) || n >= sizeof name || fread(name, 1, (size_t)n, f) != (size_t)n) {
        set_err("load_store: bad tensor record (expected %s)", want_name);
        return -1;
    }
    name[n] = 0;
    if (get_u64(f, &dt) || get_u64(f, &r) || get_u64(f, &cc)) {
        set_err("load_store: truncated file (%s)", want_name);
        return -1;
    }
    if (strcmp(name, want_name) != 0 || (int64_t)r != rows || (int64_t)cc != cols) {
        set_err("load_store: record '%s' [%llu x %llu] where '%s' [%lld x %lld] was expected",
                name, (unsigned long long)r, (unsigned long long)cc, want_name,
                (long long)rows, (long long)cols);
        return -1;
    }
    return get_floats_into(f, dst, (uint64_t)(rows * cols), want_name);
}

/* [model] section of the INI text (config.hpp:153-205, 289-329) */
static int parse_model_section(const char *text, fo_config *c) {
    memset(c, 0, sizeof *c);
    c->rope_theta = 500000.0;
    c->rmsnorm_eps = 1e-5;
    c->batch = 1;
    c->quant_group = 128;
    int in_model = 0, seen = 0;
    const char *p = text;
    char line[512];
    while (*p) {
        const char *e = strchr(p, '\n');
        size_t n = e ? (size_t)(e - p) : strlen(p);
        if (n >= sizeof line) n = sizeof line - 1;
        memcpy(line, p, n);
        line[n] = 0;
        p = e ? e + 1 : p + n;
        char *h = strchr(line, '#');
        if (h) *h = 0;
        char *a = line;
        while (*a == ' ' || *a == '\t' || *a == '\r') ++a;
        char *z = a + strlen(a);
        while (z > a && (z[-1] == ' ' || z[-1] == '\t' || z[-1] == '\r')) *--z = 0;
        if (!*a) continue;
        if (*a == '[') {
            in_model = strcmp(a, "[model]") == 0;
            seen |= in_model;
            continue;
        }
        if (!in_model) continue;
        char *eq = strchr(a, '=');
        if (!eq) { set_err("config: expected key = value"); return -1; }
        *eq = 0;
        char *k = a, *v = eq + 1;
        for (char *t = eq; t > k && (t[-1] == ' ' || t[-1] == '\t'); ) *--t = 0;
        while (*v == ' ' || *v == '\t') ++v;
        if (!strcmp(k, "kind")) {
            if (strcmp(v, "llama_decoder")) {
                set_err("load_store: only the llama_decoder kind is restated (got %s)", v);
                return -1;
            }
        } else if (!strcmp(k, "layers")) c->layers = atoll(v);
        else if (!strcmp(k, "d_model")) c->d_model = atoll(v);
        else if (!strcmp(k, "d_inter")) c->d_inter = atoll(v);
        else if (!strcmp(k, "d_head")) c->d_head = atoll(v);
        else if (!strcmp(k, "n_q_heads")) c->n_q_heads = atoll(v);
        else if (!strcmp(k, "n_kv_heads")) c->n_kv_heads = atoll(v);
        else if (!strcmp(k, "vocab_size")) c->vocab_size = atoll(v);
        else if (!strcmp(k, "rope_theta")) c->rope_theta = strtod(v, NULL);
        else if (!strcmp(k, "rmsnorm_eps")) c->rmsnorm_eps = strtod(v, NULL);
        else if (!strcmp(k, "dtype")) {
            if (!strcmp(v, "bf16")) c->dtype = 0;
            else if (!strcmp(v, "fp32") || !strcmp(v, "f32")) c->dtype = 1;
            else { set_err("unknown dtype: %s", v); return -1; }
        } else if (!strcmp(k, "batch")) c->batch = atoll(v);
        else if (!strcmp(k, "quant_bits")) c->quant_bits = atoi(v);
        else if (!strcmp(k, "quant_group_size")) c->quant_group = atoi(v);
        else if (!strcmp(k, "quant_scheme")) continue;
        else { set_err("config: unknown [model] field '%s'", k); return -1; }
    }
    if (!seen) { set_err("config: missing [model] section"); return -1; }
    return 0;
}

fo_store *fo_load_store(const char *path, int64_t max_seq_len) { /* tensor_store.hpp:446-482 */
    FILE *f = fopen(path, "rb");
    if (!f) { set_err("load_store: cannot open %s", path); return NULL; }
    fo_store *s = NULL;
    uint64_t magic = 0, ver = 0, tn = 0;
    char *text = NULL;
    if (get_u64(f, &magic) || magic != FO_STORE_MAGIC) { set_err("load_store: bad magic"); goto fail; }
    if (get_u64(f, &ver) || ver != FO_STORE_VERSION) { set_err("load_store: bad version"); goto fail; }
    if (get_u64(f, &tn) || tn > (1u << 20)) { set_err("load_store: bad config record"); goto fail; }
    text = (char *)calloc((size_t)tn + 1, 1);
    if (fread(text, 1, (size_t)tn, f) != (size_t)tn) { set_err("load_store: truncated file"); goto fail; }
    fo_config c;
    if (parse_model_section(text, &c) || fo_validate(&c)) goto fail;
    s = store_alloc(&c, max_seq_len);
    uint64_t nl;
    if (get_u64(f, &nl) || (int64_t)nl != c.layers) { set_err("load_store: layer count mismatch"); goto fail; }
    const int64_t d = c.d_model;
    char name[64];
    for (int64_t l = 0; l < c.layers; ++l) {
        fo_layer *L = &s->layers[l];
#define GM(T, PTR, R)                                              \
    snprintf(name, sizeof name, "layer.%lld." T, (long long)l);    \
    if (get_matrix_into(f, (PTR), name, (R), d)) goto fail;
        GM("wqkv", L->wqkv, fo_qkv_rows(&c))
        GM("waout", L->waout, d)
        GM("wffn1", L->wffn1, 2 * c.d_inter)
        GM("wffn2t", L->wffn2t, c.d_inter)
#undef GM
        if (get_floats_into(f, L->norm_attn, (uint64_t)d, "norm_attn") ||
            get_floats_into(f, L->norm_ffn, (uint64_t)d, "norm_ffn"))
            goto fail;
    }
    if (get_floats_into(f, s->final_norm, (uint64_t)d, "final_norm") ||
        get_matrix_into(f, s->embedding, "embedding", c.vocab_size, d) ||
        get_matrix_into(f, s->lm_head, "lm_head", c.vocab_size, d))
        goto fail;
    free(text);
    fclose(f);
    return s;
fail:
    free(text);
    fo_free(s);
    fclose(f);
    return NULL;
}

/* Same weights, a new batch size: the KV cache is reallocated empty (the
 * weights of a TensorStore do not depend on the batch, tensor_store.hpp:
 * 304-366; only KVCache(model, max_seq_len) does). */
int fo_store_set_batch(fo_store *s, int64_t batch, int64_t max_seq_len) {
    if (batch < 1) { set_err("model: batch must be positive"); return 2; }
    const fo_config *c = &s->cfg;
    size_t kv = (size_t)batch * c->layers * c->n_kv_heads * max_seq_len * c->d_head;
    float *k = alloc_f32((int64_t)kv), *v = alloc_f32((int64_t)kv);
    if (!k || !v) { free(k); free(v); set_err("set_batch: out of memory"); return 1; }
    free(s->k);
    free(s->v);
    s->k = k;
    s->v = v;
    s->cfg.batch = batch;
    s->max_seq_len = max_seq_len;
    for (int64_t l = 0; l < c->layers; ++l) s->kv_len[l] = 0;
    return 0;
}
