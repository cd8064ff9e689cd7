/*
 * fusesim_oracle.h -- CPU restatement of the FlashFormer/fusesim decode path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2505_22758_b200/,
 * include/) links, loads or calls this code; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg do, and only as the checker.
 *
 * Plain C99 restatement of the reference algorithm (paths relative to
 * /root/reference/proj/include/fusesim/):
 *   - weight generation     tensor_store.hpp:270-366 (init_weights, fill_matrix,
 *                           fill_vector) incl. libstdc++'s mt19937_64,
 *                           generate_canonical and normal_distribution (polar)
 *   - int4 affine snapping  quant.hpp:23-54
 *   - bf16 rounding         types.hpp:50-59
 *   - dense f64 decode step reference.hpp:37-139 (reference_forward)
 *   - numerics primitives   numerics.hpp:14-175
 *   - synthetic prefill     tests/test_interpreter.cpp:16-30
 * Parity of this restatement with the reference itself is pinned by
 * tests/test_oracle_vs_ref.py (bit-exact weights and logits against
 * oracle/_ref, the reference headers compiled unchanged) and by the golden
 * fixtures in tests/golden/.
 */
#ifndef FUSESIM_ORACLE_H
#define FUSESIM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors fusesim::ModelConfig (config.hpp:45-86).  dtype: 0 = bf16, 1 = f32.
 * quant_bits: 0 = none, 4 = reference int4 g128 scheme, 8 = int8 extension
 * (same affine formula with 255 levels; not in the reference -> parity unpinned). */
typedef struct fo_config {
    int64_t layers, d_model, d_inter, d_head, n_q_heads, n_kv_heads, vocab_size;
    double rope_theta, rmsnorm_eps;
    int32_t dtype;
    int32_t quant_bits;
    int32_t quant_group;
    int64_t batch;
} fo_config;

typedef struct fo_layer {
    float *wqkv;      /* qkv_rows x d_model                    */
    float *waout;     /* d_model x d_model                     */
    float *wffn1;     /* 2*d_inter x d_model, even=in odd=gate */
    float *wffn2t;    /* d_inter x d_model (transposed W2)     */
    float *norm_attn; /* d_model */
    float *norm_ffn;  /* d_model */
} fo_layer;

typedef struct fo_store {
    fo_config cfg;
    int64_t max_seq_len;
    fo_layer *layers;
    float *final_norm;
    float *embedding; /* vocab x d_model */
    float *lm_head;   /* vocab x d_model */
    /* KV cache [B][L][Hkv][S][dh] as in tensor_store.hpp:139-148 */
    float *k, *v;
    int64_t *kv_len;  /* per layer */
} fo_store;

const char *fo_last_error(void);

/* -------- RNG restatement (libstdc++ <random>) -------- */
typedef struct fo_mt64 { uint64_t mt[312]; int idx; } fo_mt64;
typedef struct fo_mt32 { uint32_t mt[624]; int idx; } fo_mt32;
void fo_mt64_seed(fo_mt64 *g, uint64_t seed);
uint64_t fo_mt64_next(fo_mt64 *g);
void fo_mt32_seed(fo_mt32 *g, uint32_t seed);
uint32_t fo_mt32_next(fo_mt32 *g);
uint64_t fo_fnv1a(const void *data, uint64_t n, uint64_t seed);
uint64_t fo_fnv1a_str(const char *s);

/* fills n doubles from normal_distribution<double>(mean, stddev) on mt19937_64(seed) */
void fo_normal_f64(uint64_t seed, double mean, double stddev, double *out, int64_t n);

/* -------- element helpers -------- */
float fo_bf16_round(float x);
float fo_dequantize_code(uint8_t code, float scale, float zero_point);
uint8_t fo_quantize_value(float v, float scale, float zero_point, int32_t levels);
/* quantize_group (quant.hpp:42-54); levels = 15 (int4) or 255 (int8 extension).
 * codes may be NULL.  Writes dequantized values to deq (may alias values). */
void fo_quantize_group(const float *values, int64_t n, int32_t levels, uint8_t *codes,
                       float *scale, float *zero_point, float *deq);

/* -------- store -------- */
int fo_validate(const fo_config *c);
uint64_t fo_streamed_weight_bytes(const fo_config *c);
uint64_t fo_total_weight_bytes(const fo_config *c);
fo_store *fo_init_weights(const fo_config *c, uint64_t seed, int64_t max_seq_len, int nthreads);
void fo_free(fo_store *s);

/* -------- weight fixture container "FSTW" v1 (tensor_store.hpp:367-482) -------- */
/* serialize(RunConfig) text (config.hpp:245-287) with default hardware /
 * pipeline / run sections; returns its length (snprintf semantics). */
int64_t fo_serialize_config(const fo_config *c, char *out, int64_t cap);
/* save_store: byte-identical to the reference's file for the decoder kind. */
int fo_save_store(const fo_store *s, const char *path);
/* same weights, new batch size: empty KV cache [batch][L][Hkv][max_seq_len][dh] */
int fo_store_set_batch(fo_store *s, int64_t batch, int64_t max_seq_len);
/* load_store: NULL + fo_last_error() on a bad magic / version / record. */
fo_store *fo_load_store(const char *path, int64_t max_seq_len);
int64_t fo_qkv_rows(const fo_config *c);
/* set_position / set_length / k_at / v_at (tensor_store.hpp:109-125) */
void fo_kv_set_position(fo_store *s, int64_t b, int64_t l, int64_t h, int64_t pos,
                        const float *k, const float *v);
float *fo_k_at(fo_store *s, int64_t b, int64_t l, int64_t h, int64_t pos);
float *fo_v_at(fo_store *s, int64_t b, int64_t l, int64_t h, int64_t pos);
void fo_kv_set_length(fo_store *s, int64_t layer, int64_t n);
int64_t fo_kv_length(const fo_store *s, int64_t layer);
/* tests/test_interpreter.cpp:16-30: mt19937_64(seed), normal_distribution<float>(0, 0.3) */
void fo_synthetic_prefill(fo_store *s, int64_t prefill, uint64_t seed);

/* -------- decode step (reference.hpp:37-139) --------
 * logits: batch x vocab doubles.  Appends one KV position per layer.
 * Returns 0 on success, 2 on validation error (see fo_last_error). */
int fo_reference_forward(fo_store *s, const int64_t *tokens, int64_t pos, double *logits);
/* Checker hook: identical to fo_reference_forward, except that the K/V rows
 * appended at `pos` are taken from k_app/v_app ([B][L][Hkv][dh], already on
 * the cache grid) instead of the oracle's own f64->f32->bf16 rounding.  Lets a
 * test separate 1-ulp bf16 rounding flips of the appended K/V (a property of
 * any non-f64 producer) from the rest of the arithmetic. */
int fo_reference_forward_ex(fo_store *s, const int64_t *tokens, int64_t pos, double *logits,
                            const float *k_app, const float *v_app);

/* -------- numerics primitives (numerics.hpp) -------- */
void fo_rmsnorm_f64(const double *x, const double *w, int64_t n, double eps, double *y);
void fo_rope_f64(double *v, int64_t d_head, int64_t pos, double theta);
double fo_silu(double z);
int64_t fo_argmax_f64(const double *logits, int64_t n);
/* online-softmax partial state (numerics.hpp:64-98): state = {m, l, o[d]} */
void fo_attn_partial_update(double *m, double *l, double *o, int64_t d, const double *q,
                            const double *k_rows, const double *v_rows, int64_t rows,
                            double alpha);
/* 3-stage reduction (numerics.hpp:123-145); partials are (m_i, l_i, o_i[d]) */
int fo_attn_reduce(const double *m, const double *l, const double *o, int64_t n_partials,
                   int64_t d, double *out);

/* Stacked-linear kind: fill_matrix of "linear.<l>" (tensor_store.hpp:270-290,
 * fan-in = cols, never quantized) and reference_linear_forward
 * (reference.hpp:141-152) in f64. */
void fo_fill_linear(const char *name, int64_t rows, int64_t cols, uint64_t seed, int32_t dtype,
                    float *dst);
void fo_linear_forward(const float *w, int64_t layers, int64_t d, int64_t batch, const float *x0,
                       double *out);

#ifdef __cplusplus
}
#endif
#endif
