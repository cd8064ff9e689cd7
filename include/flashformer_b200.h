/*
 * flashformer_b200.h -- C-ABI of the B200 whole-model decode kernel.
 *
 * Drop-in boundary for the reference's decode path.  The reference
 * (/root/reference/proj/include/fusesim/) has no FFI: its "operator API" is two
 * header-only C++ calls that this ABI replaces:
 *
 *   fusesim::execute_program(programs, plan, store, tokens, pos)
 *       interpreter.hpp:502-506  -> ffb_decode_step(...)
 *   fusesim::reference_forward(store, tokens, pos)
 *       reference.hpp:37-139     -> ffb_decode_step(...) (same contract)
 *
 * and the pieces of fusesim::TensorStore those calls mutate or read:
 *   init_weights / TensorStore weights   tensor_store.hpp:240-366 -> ffb_upload_tensor
 *   KVCache::set_position / k_at / v_at  tensor_store.hpp:109-125 -> ffb_kv_set / ffb_kv_get
 *   KVCache::set_length / length         tensor_store.hpp:77,118  -> ffb_kv_set_length / ffb_kv_length
 *   ModelConfig (+ validate)             config.hpp:45-86         -> ffb_model_config / ffb_create
 *   RunMode {Baseline,Fused,FusedOverlap} types.hpp:64            -> ffb_set_mode
 *
 * Conventions:
 *   - plain pointers and sizes only; host pointers unless a name says _device.
 *   - every call returns an ffb_status; ffb_last_error() holds a thread-local
 *     message.  FFB_VALIDATION mirrors fusesim::ValidationError (bad token,
 *     position != cache length, cache capacity), FFB_UNSUPPORTED means no
 *     compiled kernel specialisation matches the config.
 *   - one CUDA stream per handle (or the caller's stream); a handle is not
 *     re-entrant.  The KV length advances only when a step succeeds.
 *   - no CPU fallback: on a machine without an sm_100 device ffb_create fails.
 */
#ifndef FLASHFORMER_B200_H
#define FLASHFORMER_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ffb_status {
    FFB_OK = 0,
    FFB_USAGE = 1,         /* bad argument / handle / name (CLI usage=1, types.hpp:14) */
    FFB_VALIDATION = 2,    /* fusesim::ValidationError equivalent (CLI validation=2) */
    FFB_DEVICE = 3,        /* CUDA error */
    FFB_UNSUPPORTED = 4    /* no template instantiation for this model shape */
} ffb_status;

/* fusesim::RunMode (types.hpp:64): one launch per sublayer stage, one
 * persistent launch with the producer waiting at every barrier, or one
 * persistent launch whose producer streams across barriers. */
typedef enum ffb_mode {
    FFB_MODE_BASELINE = 0,
    FFB_MODE_FUSED = 1,
    FFB_MODE_FUSED_OVERLAP = 2,
    /* tensor parallelism only: the Baseline's per-stage launches with the two
     * per-layer residual sums done by the host as ncclAllReduce between the
     * kernels and the argmax by ncclAllGather (SURVEY.md §8(e) "Baseline:
     * host ncclAllReduce between per-layer kernels"); needs ffb_tp_nccl_init */
    FFB_MODE_BASELINE_NCCL = 3
} ffb_mode;

/* fusesim::ModelConfig (config.hpp:45-86).
 * kind: 0 = llama_decoder, 1 = stacked_linear (config.hpp:18; only layers,
 *       d_model and batch are used; square d_model x d_model layers).
 * dtype: 0 = bf16 (the only compiled storage type).
 * quant_bits: 0 (bf16 weights), 4 (reference int4 g128), 8 (int8 extension).
 * batch: 1..16; batch 8 / 16 (bf16, TP 1) run every projection on tensor
 * cores and keep the streamed matrices in a chunk-major fp16 layout (the
 * upload converts; ffb_tensor values are the reference's bf16 values). */
typedef struct ffb_model_config {
    int64_t layers, d_model, d_inter, d_head, n_q_heads, n_kv_heads, vocab_size;
    double rope_theta, rmsnorm_eps;
    int32_t dtype;
    int32_t quant_bits;
    int32_t quant_group;
    int64_t batch;
    int32_t kind;
    int32_t reserved_;
} ffb_model_config;

typedef struct ffb_model ffb_model;

const char *ffb_last_error(void);
const char *ffb_version(void);

/* Host-only weight packer (no device needed).  Row format of a streamed
 * matrix with `cols` columns: bf16 (quant_bits 0) = cols*2 bytes; int4 / int8
 * = [codes: int4 two per byte, little nibble first | f32 scale per group of
 * 128 | u8 zero point per group | zero pad to 16 B].  Returns the bytes per
 * row, or -1 for an unsupported (cols, quant_bits). */
int64_t ffb_quant_row_bytes(int64_t cols, int32_t quant_bits);
/* Packs rows x cols f32 values (quant_bits 4 or 8) into `out`
 * (rows * ffb_quant_row_bytes bytes), re-deriving the reference's
 * quantize_group grid (quant.hpp:42-54) per group of 128 columns.  Returns the
 * number of groups whose values lie on no such grid (packed lossily), or -1. */
int64_t ffb_pack_quant_rows(const float *values, int64_t rows, int64_t cols,
                            int32_t quant_bits, uint8_t *out);
/* Same with an explicit code order: layout 0 = plain (column order, used by
 * Wffn2^T and the CUDA-core GEMV), 1 = tensor-core order (mma.sync m16n8k32
 * u8 A fragments: per 128-column group, lane quad q reads columns 32s + 4q +
 * {0..3} and 32s + 16 + 4q + {0..3} of k32-step s as one word (int4: low /
 * high nibbles) or 8 bytes (int8), q-major 16 / 32-byte blocks; used by
 * Wqkv / Wffn1 / lm_head / Waout rows whose width is a multiple of 1024). */
int64_t ffb_pack_quant_rows_ex(const float *values, int64_t rows, int64_t cols,
                               int32_t quant_bits, int32_t layout, uint8_t *out);

/* 1 if a kernel specialisation exists for this shape (no device needed). */
int ffb_config_supported(const ffb_model_config *cfg);

/* Allocates weights, KV cache [L][B][Hkv][max_seq_len][d_head] bf16 and
 * scratch on `device`.  tp_rank/tp_size: tensor-parallel shard (tp_size 1 =
 * whole model): rank r holds kv heads [r Hkv/tp, (r+1)
 * Hkv/tp) with their q heads (Wqkv rows, KV cache), the matching input
 * columns of Waout, d_inter slice r of Wffn1 / Wffn2^T and vocab slice r of
 * lm_head; embedding and norms are replicated.  Per layer the residual
 * deltas of the O-projection and the FFN are summed across ranks inside the
 * persistent kernel over peer memory (NVLink P2P), plus one argmax exchange
 * per step.  A TP rank must be connected (ffb_tp_connect) before stepping. */
ffb_status ffb_create(const ffb_model_config *cfg, int64_t max_seq_len, int device,
                      int tp_rank, int tp_size, ffb_model **out);
/* Same, with the persistent grid limited to `grid` CTAs (0 = one per SM),
 * e.g. to co-locate the ranks of a TP group on one GPU for testing. */
ffb_status ffb_create_ex(const ffb_model_config *cfg, int64_t max_seq_len, int device,
                         int tp_rank, int tp_size, int grid, ffb_model **out);

/* Tensor-parallel wiring: every rank exports a blob (ffb_tp_blob_bytes
 * bytes: its exchange buffers as raw pointers + CUDA IPC handles), the blobs
 * are all-gathered by the caller (e.g. torch.distributed), and every rank
 * connects to the array of tp_size blobs ordered by rank.  Same-process
 * ranks use the raw pointers, other processes open the IPC handles. */
int64_t ffb_tp_blob_bytes(void);
ffb_status ffb_tp_export(ffb_model *m, void *blob);
ffb_status ffb_tp_connect(ffb_model *m, const void *blobs, int32_t n);

/* Host-NCCL communicator for FFB_MODE_BASELINE_NCCL.  NCCL is loaded at run
 * time (dlopen "libnccl.so.2"; FFB_USAGE if absent), not linked.  Rank 0
 * makes the 128-byte unique id with ffb_nccl_unique_id, the caller
 * broadcasts it, every rank calls ffb_tp_nccl_init (collective over the
 * tp_size ranks, one process per GPU). */
ffb_status ffb_nccl_unique_id(uint8_t id[128]);
ffb_status ffb_tp_nccl_init(ffb_model *m, const uint8_t id[128]);
void ffb_destroy(ffb_model *m);

/* Weight packer.  `name` uses the reference's tensor names
 * (tensor_store.hpp:344-363): "layer.<l>.wqkv", "layer.<l>.waout",
 * "layer.<l>.wffn1", "layer.<l>.wffn2t", "layer.<l>.norm_attn",
 * "layer.<l>.norm_ffn", "final_norm", "embedding", "lm_head".  `values` is the
 * TensorStore's row-major f32 array (n = rows*cols).  bf16 matrices are
 * rounded RNE (exact for reference stores, whose values are already on the
 * bf16 grid); norm gains stay f32.  Quantized models (quant_bits 4 or 8,
 * quant_group 128) pack every streamed matrix (wqkv, waout, wffn1, wffn2t,
 * lm_head; the embedding stays bf16) into per-row codes + f32 group scales +
 * zero points, re-deriving the reference's quantize_group grid
 * (quant.hpp:42-54) so that (code - zero) * scale reproduces reference store
 * values bit for bit; values off any grid are quantized (lossy, counted in
 * ffb_info.quant_inexact_groups). */
ffb_status ffb_upload_tensor(ffb_model *m, const char *name, const float *values, int64_t n);

/* Weight fixture container: reads a "FSTW" v1 file
 * written by fusesim::save_store (tensor_store.hpp:410-444) and packs every
 * record through ffb_upload_tensor -- the drop-in for load_store
 * (tensor_store.hpp:446-482) without a host TensorStore.  The file's model
 * shape must equal the handle's (batch, dtype and quant fields may differ:
 * values are packed into the handle's format).  FFB_USAGE on a bad magic /
 * version / truncated record, FFB_VALIDATION on a shape mismatch. */
ffb_status ffb_load_store(ffb_model *m, const char *path);

/* Packed device image cache: every streamed matrix, norm and the embedding
 * exactly as the kernel reads them (after the packer, TP slicing, chunk-major
 * swizzle, quant grid re-derivation), plus a header naming the model, the TP
 * shard and the kernel specialisation.  ffb_load_image refuses an image of
 * another shape / shard / specialisation (FFB_VALIDATION). */
ffb_status ffb_save_image(ffb_model *m, const char *path);
ffb_status ffb_load_image(ffb_model *m, const char *path);

/* Fills every weight on the device with seeded synthetic values of the right
 * scale (bench / smoke use; no host arrays involved). */
ffb_status ffb_init_synthetic(ffb_model *m, uint64_t seed);

/* KV cache access mirroring KVCache (tensor_store.hpp:63-150).  k/v: d_head
 * f32 values, rounded to bf16 on store. */
ffb_status ffb_kv_set(ffb_model *m, int64_t b, int64_t layer, int64_t head, int64_t pos,
                      const float *k, const float *v);
ffb_status ffb_kv_get(ffb_model *m, int64_t b, int64_t layer, int64_t head, int64_t pos,
                      float *k, float *v);
/* Bulk import of the reference layout [B][L][Hkv][S_src][dh] f32, positions [0, n_pos). */
ffb_status ffb_kv_import(ffb_model *m, const float *k, const float *v, int64_t src_max_seq,
                         int64_t n_pos);
/* Bulk export of positions [pos0, pos0 + n_pos) in the reference layout
 * [B][L][Hkv][n_pos][dh] f32 (KVCache::k_at / v_at, tensor_store.hpp:109-125;
 * a TP rank exports its own kv heads).  One gather kernel and one
 * device-to-host copy per call (chunked when the block exceeds 32 MiB);
 * synchronous. */
ffb_status ffb_kv_export(ffb_model *m, int64_t pos0, int64_t n_pos, float *k_out, float *v_out);
ffb_status ffb_kv_set_length(ffb_model *m, int64_t layer, int64_t n);
int64_t ffb_kv_length(const ffb_model *m, int64_t layer);

ffb_status ffb_set_mode(ffb_model *m, ffb_mode mode);

/* Tuning knobs.  "l2_prefetch_bytes": how far (bytes per SM) the producer's
 * L2 prefetch cursor runs ahead of the shared-memory ring in FusedOverlap
 * mode (0 disables; default 512 KiB).  "l2_prefetch_stages": 6-bit mask of
 * the stage types (bit s = stage s of a layer: 0 QKV, 1 ATTN, 2 AOUT, 3 GLU,
 * 4 RED; bit 5 = LM head) in which the prefetch may run, only while the ring
 * is full (default ATTN|AOUT = 0x6).  "l2_prefetch_delay_ns": how long the
 * prefetch window's burst is held after a layer's first K/V chunk is issued,
 * so the attention's own K/V reaches HBM first (0..100000; default 4750 for
 * the Llama-3.1-8B and Llama-3-70B shapes at batch 1-2 on one GPU, else 0).
 * "attn_group_max": cap on the CTAs per
 * (batch row, kv head) split-K attention group (0 = min(grid / units, 32)).
 * Plan options (rebuild the per-CTA plan): "calib_mask", "plan_reverse",
 * "attn_group_max".  "stage_mask": 0x1f, or 0x07 / 0x18 for the component
 * ablation (attention / GLU blocks only).  "prefill_terms": bf16 terms per
 * f32 activation in ffb_prefill's GEMMs -- 3 (default, f32-exact products)
 * or 2 (hi + lo, ~2^-17 relative, a third fewer tensor-core FLOPs). */
ffb_status ffb_set_option(ffb_model *m, const char *key, int64_t value);

/* Diagnostics only (never needed for correct use): bit 0 = streaming-only
 * run, the consumer warps just wait for and release every ring slot of the
 * schedule -- measures the TMA streaming rate with no math and no
 * inter-SM flags.  Results are garbage while set. */
ffb_status ffb_set_debug(ffb_model *m, int32_t flags);

/* Tracing: when enabled, consumer thread 0 of every CTA
 * records %globaltimer at each stage's entry, dependency-met, done and a
 * stage-specific mark, plus the ns it spent starved waiting for ring data,
 * into a device buffer [grid][5*L+1][8] (u64).  ffb_get_trace copies it out
 * (out may be NULL to query the element count); returns -1 on error. */
ffb_status ffb_set_trace(ffb_model *m, int enable);
int64_t ffb_get_trace(ffb_model *m, uint64_t *out, int64_t n);

/* One decode step for every batch row (reference.hpp:37-139 contract).
 * With tensor parallelism every rank calls it with the same tokens; logits
 * are this rank's vocab slice [batch][vocab/tp], greedy is the global argmax.
 * tokens[batch] (host), pos == kv length of every layer, appends one KV
 * position per layer.  logits_out: batch x vocab f32 (host, may be NULL);
 * greedy_out: batch int64 argmax with lowest-index tie break (host, may be
 * NULL).  stream: cudaStream_t or NULL for the handle's stream.  Synchronous
 * w.r.t. the host outputs. */
ffb_status ffb_decode_step(ffb_model *m, const int64_t *tokens, int64_t pos, float *logits_out,
                           int64_t *greedy_out, void *stream);

/* Same step with device-resident inputs/outputs, fully asynchronous on
 * `stream`: d_tokens[batch] int64, d_logits (batch x vocab f32) and d_greedy
 * (batch int64) device pointers (either may be NULL -> internal buffers).
 * The caller guarantees pos == kv length; the length advances on enqueue. */
ffb_status ffb_decode_step_device(ffb_model *m, const int64_t *d_tokens, int64_t pos,
                                  float *d_logits, int64_t *d_greedy, void *stream);

/* Waits for every step enqueued on the handle (any stream: device-wide
 * synchronize) and reports device-side validation latched by them: a
 * device-resident token id outside [0, vocab) reads embedding row 0 and
 * latches FFB_VALIDATION ("token id out of range"), returned (and cleared)
 * by the next ffb_sync or ffb_decode_step. */
ffb_status ffb_sync(ffb_model *m);

/* Device-resident multi-token decode: n_steps
 * decode steps enqueued back to back on `stream` with no host round trip.
 * teacher_forced = 0 (generation): step 0 reads d_tokens[batch], step i > 0
 * the greedy tokens of step i-1; teacher_forced = 1 (prompt ingestion,
 * decode-as-prefill like the reference): step i reads d_tokens[i][batch].
 * d_out[n_steps][batch] receives every step's greedy tokens; the device
 * logits (ffb_logits_device) hold the last step's.  pos == cache length;
 * the length advances by n_steps on enqueue. */
ffb_status ffb_decode_loop(ffb_model *m, const int64_t *d_tokens, int64_t pos, int32_t n_steps,
                           int32_t teacher_forced, int64_t *d_out, void *stream);

/* Prompt ingestion as GEMMs (replaces the
 * reference's decode-as-prefill loop, reference.hpp:60-61 / engine prefill):
 * tokens[n][batch] (host) at positions pos0 .. pos0+n-1 of every batch row go
 * through each layer together -- projections as cuBLAS bf16 GEMMs over
 * n*batch rows with the f32 activations split into three bf16 terms
 * (f32-accurate products; int4 / int8 weights are dequantised per
 * projection into three exact bf16 planes of w = (code - zero) * scale),
 * RoPE / K-V append / causal attention / SiLU in f32 kernels.  Leaves the KV
 * cache and its lengths where n decode steps would (pos0 + n), so
 * ffb_decode_step continues at pos0 + n.  logits_out (batch x vocab f32,
 * host, may be NULL) / greedy_out (batch int64, host, may be NULL) are those
 * of the LAST position.  Decoders on one GPU (batch >= 8: the fp16
 * tensor-core weight layout is unpacked per projection; tensor-parallel
 * shards return FFB_UNSUPPORTED); n * batch <= 1024 per call (longer prompts:
 * call again with pos0 advanced).  Synchronous; the scratch (activations,
 * split planes, expanded weight chunks: ~1-2 GB at the 8B shape and 1024
 * rows) is allocated on first use, grown as needed and freed with the
 * handle; cuBLAS is loaded at run time (libcublas.so.12). */
ffb_status ffb_prefill(ffb_model *m, const int64_t *tokens, int64_t n, int64_t pos0,
                       float *logits_out, int64_t *greedy_out);

/* Stacked-linear kind (reference_linear_forward, reference.hpp:141-152; the
 * paper's cross-layer fusion ablation): tensors
 * "linear.<l>" (d_model x d_model, bf16-rounded) and "residual" (batch x
 * d_model input) via ffb_upload_tensor; x_in (host [batch][d_model], NULL =
 * the uploaded residual) -> x_out = W_{L-1} ... W_0 x_in (host, may be
 * NULL).  Run modes apply (baseline = one launch per layer).  Synchronous. */
ffb_status ffb_linear_forward(ffb_model *m, const float *x_in, float *x_out, void *stream);
/* Same, device pointers (either may be NULL), asynchronous on `stream`. */
ffb_status ffb_linear_forward_device(ffb_model *m, const float *d_x_in, float *d_x_out,
                                     void *stream);

/* Introspection for roofline accounting and tests. */
typedef struct ffb_info {
    int32_t grid;            /* CTAs per launch (one per SM)               */
    int32_t threads;         /* threads per CTA                            */
    int32_t smem_bytes;      /* dynamic shared memory per CTA              */
    int32_t ring_slots;      /* TMA ring depth                             */
    int32_t slot_bytes;      /* bytes per ring slot                        */
    int32_t attn_group;      /* CTAs per (batch row, kv head)              */
    int32_t launches_per_step; /* 1 (fused) or 5*L+1 (baseline)            */
    int32_t mode;
    uint64_t weight_bytes;   /* streamed weight bytes per step (device format) */
    uint64_t device_bytes;   /* total device allocation                    */
    uint64_t quant_inexact_groups; /* packer: groups not on a 4/8-bit grid  */
    int32_t row_bytes;       /* bytes per streamed-matrix row              */
    int32_t kc_layout;       /* batch >= 8 GEMV: 2 = mma.sync, 3 = tcgen05 (libffb200_tc05.so); 0 otherwise */
    uint64_t fp16_inexact;   /* batch >= 8: bf16 weights below the fp16 normal
                                range (stored rounded to 2^-24; the tcgen05
                                operands are fp16); weights beyond the fp16
                                range are rejected by ffb_upload_tensor      */
} ffb_info;
ffb_status ffb_get_info(const ffb_model *m, ffb_info *out);

/* Per-SM load balance (the reference's calibrate step, on
 * real hardware).  Runs `iterations` rounds of 3 traced decode steps at the
 * current cache length (positions beyond the length are scratch), measures
 * each SM's GLU streaming time and re-splits the rows of every streamed
 * matrix in proportion to each SM's measured rate (weights clamped to
 * [0.7, 1.3] of the mean).  Persistent launches map CTAs to plans by SM id,
 * so the weights follow the SM.  iterations == 0 restores the uniform plan.
 * Results stay deterministic for a given plan; a different plan changes the
 * cross-CTA summation grouping (~1e-7 relative). */
ffb_status ffb_calibrate(ffb_model *m, int32_t iterations);
/* Current per-SM plan weights (mean 1); returns the count (grid) or -1. */
int64_t ffb_get_plan_weights(const ffb_model *m, double *out, int64_t n);

/* Device pointer to the most recent logits (batch x vocab f32) of
 * ffb_decode_step_device / ffb_decode_loop (ffb_decode_step with host logits
 * writes them straight into pinned host memory instead). */
const float *ffb_logits_device(const ffb_model *m);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif
