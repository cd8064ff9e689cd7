// model.cuh -- the ffb_model handle (device store + runtime state) shared by
// the runtime translation units (runtime.cu: create / upload / step;
// store_io.cu: FSTW store files, device images, bulk KV export).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/flashformer_b200.h"
#include "kernel_ops.cuh"

namespace ffb200 {
extern thread_local std::string g_err;
ffb_status fail(ffb_status s, const char* fmt, ...);
}  // namespace ffb200

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return ::ffb200::fail(FFB_DEVICE, "%s: %s (%s:%d)", #expr,                   \
                                  cudaGetErrorString(e_), __FILE__, __LINE__);           \
    } while (0)

using namespace ffb200;  // CtaPlan, KernelOps, stage ids (internal header)

constexpr int kMaxTP = 8;

struct ffb_model {
    ffb_model_config cfg{};   // this shard's config (== gcfg when tp_size == 1)
    ffb_model_config gcfg{};  // the whole model
    int64_t vocab_base = 0;   // first global vocab row of this shard's lm_head
    // tensor-parallel exchange (decode_kernel.cuh: tp_exchange_add)
    float* xch = nullptr;           // [2][2][B][D] + [kMaxTP][B][2]
    uint32_t* xflag = nullptr;      // [L][2][grid] + 1
    size_t xch_bytes = 0, xflag_bytes = 0;
    float* peer_xch[kMaxTP] = {};
    uint32_t* peer_xflag[kMaxTP] = {};
    bool tp_connected = false;
    std::vector<void*> ipc_opened;
    const KernelOps* ops = nullptr;
    int device = 0, grid = 0, tp_rank = 0, tp_size = 1;
    int64_t max_seq = 0;
    int attn_group = 0, n_units = 0;
    ffb_mode mode = FFB_MODE_FUSED_OVERLAP;
    int32_t debug = 0;
    uint64_t* trace = nullptr;  // per-CTA stage timestamps (ffb_set_trace)
    // per-CTA L2 prefetch window (ffb_set_option), issued only while the
    // producer is blocked on a full ring in S_ATTN / S_AOUT (the attention
    // latency chain, when HBM would otherwise idle); measured -2% on the 8B
    // shape at 512 KiB, while prefetching during the streaming-bound GLU
    // stage costs up to +8% (profiles/summary_r01.md)
    int64_t l2_prefetch = 512 << 10;
    int32_t l2_pf_stages = (1 << S_ATTN) | (1 << S_AOUT);
    int32_t l2_pf_delay = 0;          // option "l2_prefetch_delay_ns"
    int32_t stage_mask = 0x1f;        // option "stage_mask" (component ablation)
    int plan_reverse = 0;             // weight slices assigned in reverse CTA order
    int attn_group_max = 0;           // option "attn_group_max": cap on CTAs per attention unit (0: auto)
    // per-SM plan weights (ffb_calibrate): streamed-row shares of QKV / AOUT /
    // GLU / LM head proportional to each SM's measured streaming rate
    std::vector<double> sm_weight;
    // LM-head row shares (ffb_calibrate, from the LM-head stage's own per-CTA
    // times; used instead of sm_weight for calib_mask bit 3): its per-SM
    // rates differ from the GLU's that sm_weight follows
    std::vector<double> lm_weight;
    std::vector<CtaPlan> plan_host;
    int16_t* sm_rank = nullptr;       // device [max smid + 1] -> dense rank, or null
    int calib_mask = 0xf;             // option "calib_mask": matrices using the weights
    int use_sm_rank = 1;              // option "sm_rank": plans follow SM ids
    uint32_t epoch = 0;
    cudaStream_t stream = nullptr;
    std::vector<int64_t> kv_len;
    std::vector<void*> allocs;
    uint64_t device_bytes = 0;

    // streamed matrices: rows of ops->row_bytes (bf16 or packed int4/int8)
    uint8_t *wqkv = nullptr, *waout = nullptr, *wffn1 = nullptr, *wffn2t = nullptr,
            *lm_head = nullptr;
    __nv_bfloat16 *embedding = nullptr, *kcache = nullptr, *vcache = nullptr;
    uint64_t fp16_inexact = 0;  // batch >= 8 packer: bf16 weights below the fp16 normal range, rounded
    uint64_t quant_inexact_groups = 0;  // packer: groups not on a 4/8-bit grid (lossy)
    uint8_t* wlin = nullptr;            // stacked linear: [L][D] bf16 rows
    float* xbuf = nullptr;              // stacked linear: [2][B][D]
    float *norm_attn = nullptr, *norm_ffn = nullptr, *final_norm = nullptr;
    uint8_t *xfrag_a = nullptr, *xfrag_f = nullptr, *afrag = nullptr, *hfrag = nullptr;  // batch >= 8
    float* ssq = nullptr;                                                               // [2][grid][B]
    float *x = nullptr, *q = nullptr, *attn_out = nullptr, *glu_part = nullptr,
          *attn_part = nullptr, *logits = nullptr, *amax_val = nullptr;
    int32_t* amax_idx = nullptr;
    void* nccl_comm = nullptr;        // ncclComm_t of FFB_MODE_BASELINE_NCCL (ffb_tp_nccl_init)
    void (*nccl_destroy)(void*) = nullptr;
    float* amax_gather = nullptr;
    // prefill (prefill.cu): cuBLAS handle + scratch, created on first use
    void* cublas = nullptr;
    void (*cublas_destroy)(void*) = nullptr;
    int prefill_terms = 3;  // option "prefill_terms": bf16 terms per f32 activation in the GEMMs
    void* pf_buf = nullptr;
    size_t pf_bytes = 0;     // [kMaxTP][B][2] the ranks' (value, index) candidates
    int64_t *greedy = nullptr, *tokens_dev = nullptr;
    uint32_t *counters = nullptr, *head_counters = nullptr, *amax_counter = nullptr,
             *qkv_head_counters = nullptr;
    CtaPlan* plan = nullptr;
    int64_t* tokens_pinned = nullptr;
    int64_t* greedy_pinned = nullptr;
    float* logits_pinned = nullptr;
    float* staging = nullptr;  // f32 upload staging
    static constexpr int64_t kStagingElems = 8 << 20;

    int64_t qkv_rows() const { return (cfg.n_q_heads + 2 * cfg.n_kv_heads) * cfg.d_head; }

    template <class Tp>
    ffb_status alloc(Tp** p, size_t count) {
        void* ptr = nullptr;
        size_t bytes = std::max<size_t>(count * sizeof(Tp), 256);
        cudaError_t e = cudaMalloc(&ptr, bytes);
        if (e != cudaSuccess)
            return fail(FFB_DEVICE, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
        allocs.push_back(ptr);
        device_bytes += bytes;
        *p = static_cast<Tp*>(ptr);
        return FFB_OK;
    }

    ~ffb_model() {
        if (device >= 0) cudaSetDevice(device);
        if (nccl_comm && nccl_destroy) nccl_destroy(nccl_comm);
        if (cublas && cublas_destroy) cublas_destroy(cublas);
        if (pf_buf) cudaFree(pf_buf);
        for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
        for (void* p : allocs) cudaFree(p);
        if (tokens_pinned) cudaFreeHost(tokens_pinned);
        if (greedy_pinned) cudaFreeHost(greedy_pinned);
        if (logits_pinned) cudaFreeHost(logits_pinned);
        if (stream) cudaStreamDestroy(stream);
    }
};
