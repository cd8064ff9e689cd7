// runtime.cu -- host runtime + C-ABI (include/flashformer_b200.h).
//
// Replaces, on the device side, the subsystems of the reference that change
// (SURVEY.md §2.2):
//   * weight packer   TensorStore f32 arrays (tensor_store.hpp:240-366) ->
//                     device bf16 matrices, f32 norm gains
//   * KV allocator    KVCache (tensor_store.hpp:63-150) -> one device block
//                     [L][B][Hkv][S][dh] bf16, position-major per head so a
//                     run of positions is one TMA bulk copy
//   * static planner  build_plan / assign_chunks (partition.hpp:80-343) ->
//                     balanced contiguous per-CTA row ranges (CtaPlan)
//   * launch shim     execute_program (interpreter.hpp:502-506) -> one
//                     cooperative persistent launch per step (or 5L+1
//                     launches in baseline mode)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is dlopen'ed by the NCCL baseline mode
#include <unistd.h>

#include "../../include/flashformer_b200.h"
#include "model.cuh"

using namespace ffb200;

namespace ffb200 {

thread_local std::string g_err;

ffb_status fail(ffb_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

}  // namespace ffb200

namespace {

const std::vector<KernelOps>& registry() {
    static std::vector<KernelOps> v;
    static std::once_flag once;
    std::call_once(once, [] {
        register_kernels_small(v);
        register_kernels_1b(v);
        register_kernels_8b(v);
        register_kernels_quant(v);
        register_kernels_70b(v);
        register_kernels_kc(v);
        register_kernels_tp(v);
    });
    return v;
}

const KernelOps* find_ops(const ffb_model_config& c) {
    if (c.dtype != 0) return nullptr;
    if (c.kind == 1) {  // stacked linear: only the d_model-column GEMV is used
        for (const auto& k : registry())
            if (k.D == c.d_model && k.B == c.batch && k.QB == 0 && k.D == k.NQ * k.DH && k.B < 8)
                return &k;
        return nullptr;
    }
    if (c.quant_bits != 0 && c.quant_group != kQuantGroup) return nullptr;
    for (const auto& k : registry())
        if (k.D == c.d_model && k.DI == c.d_inter && k.DH == c.d_head && k.NQ == c.n_q_heads &&
            k.NKV == c.n_kv_heads && k.B == c.batch && k.QB == c.quant_bits)
            return &k;
    return nullptr;
}

ffb_status validate_cfg(const ffb_model_config* c) {  // config.hpp:61-83
    if (!c) return fail(FFB_USAGE, "config is NULL");
    if (c->layers < 0) return fail(FFB_VALIDATION, "model: layers must be >= 0");
    if (c->d_model <= 0) return fail(FFB_VALIDATION, "model: d_model must be positive");
    if (c->batch < 1 || c->batch > 16) return fail(FFB_VALIDATION, "model: batch must be in [1,16]");
    if (c->kind != 0 && c->kind != 1) return fail(FFB_VALIDATION, "model: unknown kind");
    if (c->kind == 1) return FFB_OK;  // stacked_linear: other fields ignored-but-valid
    if (c->d_inter <= 0) return fail(FFB_VALIDATION, "model: d_inter must be positive");
    if (c->d_head <= 0 || c->d_head % 2)
        return fail(FFB_VALIDATION, "model: d_head must be positive and even");
    if (c->n_q_heads <= 0 || c->n_kv_heads <= 0)
        return fail(FFB_VALIDATION, "model: head counts must be positive");
    if (c->n_q_heads % c->n_kv_heads)
        return fail(FFB_VALIDATION, "model: GQA grouping requires n_q_heads mod n_kv_heads == 0");
    if (c->d_model != c->n_q_heads * c->d_head)
        return fail(FFB_VALIDATION, "model: d_model must equal n_q_heads * d_head");
    if (c->vocab_size <= 0) return fail(FFB_VALIDATION, "model: vocab_size must be positive");
    if (c->quant_bits && c->quant_bits != 4 && c->quant_bits != 8)
        return fail(FFB_VALIDATION, "quant: only 4-bit (reference) and 8-bit codes are supported");
    if (c->quant_bits && (c->quant_group <= 0 || c->d_model % c->quant_group))
        return fail(FFB_VALIDATION, "quant: group_size must divide every quantized row length");
    return FFB_OK;
}

uint16_t bf16_bits_rne(float x) {  // types.hpp:50-59
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    if ((bits & 0x7f800000u) == 0x7f800000u && (bits & 0x7fffffu)) return (bits >> 16) | 0x40;
    uint32_t lsb = (bits >> 16) & 1u;
    bits += 0x7fffu + lsb;
    return static_cast<uint16_t>(bits >> 16);
}

float bf16_bits_to_f32(uint16_t h) {
    uint32_t bits = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &bits, 4);
    return f;
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                   int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// synthetic weights: uniform with the reference's N(0, 1/sqrt(fan_in)) variance
__global__ void synth_bf16_kernel(__nv_bfloat16* dst, int64_t n, uint64_t seed, float stddev) {
    const float a = stddev * 1.7320508f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = splitmix(seed ^ (static_cast<uint64_t>(i) * 0xd1b54a32d192ed03ull));
        const float u = static_cast<float>(r >> 40) * (1.0f / 16777216.0f);  // [0,1)
        dst[i] = __float2bfloat16_rn((2.0f * u - 1.0f) * a);
    }
}

// the same bf16 values held as fp16 (batch >= 8 matrix layout, see upload)
__global__ void synth_bf16_as_f16_kernel(__half* dst, int64_t n, uint64_t seed, float stddev) {
    const float a = stddev * 1.7320508f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = splitmix(seed ^ (static_cast<uint64_t>(i) * 0xd1b54a32d192ed03ull));
        const float u = static_cast<float>(r >> 40) * (1.0f / 16777216.0f);  // [0,1)
        dst[i] = __float2half_rn(__bfloat162float(__float2bfloat16_rn((2.0f * u - 1.0f) * a)));
    }
}

// bf16-rounded f32 -> fp16 (exact for |v| >= 2^-14; 2^-24 absolute below)
__global__ void f32_to_bf16_as_f16_kernel(const float* __restrict__ src, __half* __restrict__ dst,
                                          int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2half_rn(__bfloat162float(__float2bfloat16_rn(src[i])));
}

// synthetic packed quant rows (decode_kernel.cuh weight formats): random
// codes, scale = 2 sqrt(3) stddev / levels (jittered), zero = levels / 2
__global__ void synth_quant_kernel(uint8_t* dst, int64_t rows, int cols, int qb, int row_bytes,
                                   uint64_t seed, float stddev) {
    const int levels = qb == 4 ? 15 : 255;
    const int code_words = (qb == 4 ? cols / 2 : cols) / 4;
    const int ng = cols / kQuantGroup;
    const int code_bytes = code_words * 4;
    const int64_t n = rows * (code_words + ng);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = splitmix(seed ^ (static_cast<uint64_t>(i) * 0xd1b54a32d192ed03ull));
        if (i < rows * code_words) {
            const int64_t row = i / code_words, w = i % code_words;
            *reinterpret_cast<uint32_t*>(dst + row * row_bytes + 4 * w) = static_cast<uint32_t>(r);
        } else {
            const int64_t j = i - rows * code_words, row = j / ng, g = j % ng;
            const float u = static_cast<float>(r >> 40) * (1.0f / 16777216.0f);
            const float sc = 2.0f * 1.7320508f * stddev / levels * (0.75f + 0.5f * u);
            uint8_t* rp = dst + row * row_bytes;
            *reinterpret_cast<float*>(rp + code_bytes + 4 * g) = sc;
            rp[code_bytes + 4 * ng + g] = static_cast<uint8_t>(levels / 2);
        }
    }
}

__global__ void synth_f32_kernel(float* dst, int64_t n, uint64_t seed, float mean, float stddev) {
    const float a = stddev * 1.7320508f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = splitmix(seed ^ (static_cast<uint64_t>(i) * 0xd1b54a32d192ed03ull));
        const float u = static_cast<float>(r >> 40) * (1.0f / 16777216.0f);
        dst[i] = mean + (2.0f * u - 1.0f) * a;
    }
}

int64_t split_at(int64_t units, int64_t c, int64_t grid) { return (units * c) / grid; }

// fn(r0, r1) over [0, n) split into contiguous blocks on the host's cores
// (the packer: quant grid re-derivation, transposes, chunk-major swizzles).
template <class F>
void parallel_rows(int64_t n, F fn) {
    const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nt = std::min<int64_t>(std::min<int64_t>(hw, 32), std::max<int64_t>(1, n / 64));
    if (nt <= 1) {
        fn(int64_t{0}, n);
        return;
    }
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nt; ++t)
        th.emplace_back([&, t] { fn(n * t / nt, n * (t + 1) / nt); });
    for (auto& x : th) x.join();
}

// One CTA per SM (the decode kernel's shared memory): which SM ids exist.
__global__ void smid_probe_kernel(int32_t* out) {
    extern __shared__ uint8_t probe_smem[];
    if (threadIdx.x == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        out[blockIdx.x] = static_cast<int32_t>(smid);
        probe_smem[0] = 0;
    }
}

// KV row layout: 16-byte chunks XOR-swizzled by (pos & 7) so that the
// attention kernel's 32 lanes on 32 positions read 32 distinct smem banks
// (decode_kernel.cuh: kv_swz_dim).  Element d of position pos:
int64_t kv_swz(int64_t d, int64_t pos) { return (((d >> 3) ^ (pos & 7)) << 3) | (d & 7); }

}  // namespace


namespace {

// The plan is read by every launch on any stream: wait for in-flight steps,
// copy it on the handle's stream and wait for the copy to land (a pageable
// cudaMemcpy on the legacy stream returns before its DMA completes and does
// not order against the non-blocking handle stream).
ffb_status upload_plan(ffb_model* m) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyAsync(m->plan, m->plan_host.data(), sizeof(CtaPlan) * m->plan_host.size(),
                             cudaMemcpyHostToDevice, m->stream));
    CUDA_TRY(cudaStreamSynchronize(m->stream));
    return FFB_OK;
}

ffb_status build_plan(ffb_model* m) {
    const auto& c = m->cfg;
    const int64_t G = m->grid;
    if (c.kind == 1) {  // stacked linear: rows of every layer split over the CTAs
        if ((int64_t)m->sm_weight.size() != G) m->sm_weight.assign(G, 1.0);
        std::vector<double> cum(G + 1, 0.0);
        for (int64_t k = 0; k < G; ++k) cum[k + 1] = cum[k] + m->sm_weight[k];
        std::vector<CtaPlan> plan(G);
        for (int64_t i = 0; i < G; ++i) {
            CtaPlan& p = plan[i];
            std::memset(&p, 0, sizeof(p));
            p.aout_r0 = static_cast<int32_t>(i == 0 ? 0 : std::llround(c.d_model * cum[i] / cum[G]));
            p.aout_r1 = static_cast<int32_t>(i + 1 == G ? c.d_model
                                                          : std::llround(c.d_model * cum[i + 1] / cum[G]));
            p.attn_unit = -1;
        }
        m->n_units = 0;
        m->attn_group = 0;
        m->plan_host = plan;
        return upload_plan(m);
    }
    m->n_units = static_cast<int>(c.batch * c.n_kv_heads);
    if (m->n_units > G) return fail(FFB_UNSUPPORTED, "batch * n_kv_heads exceeds the SM count");
    // split-K group per (batch row, kv head): as many SMs as fit, at most
    // kMaxGroup so the last-arriver combine keeps every load in flight, and,
    // for d_head 64 (1B-class shapes), no more than give each member ~64 KiB
    // of the cache's K/V (256 positions): below that the combine outweighs
    // the split (same box, 1B at 1k context: 18 CTAs 0.652, 5 CTAs 0.630 ms;
    // at 4k the SM bound, 18, stays).  d_head 128 shapes keep the SM bound:
    // their 4k-context optimum, and the group size fixes the summation order
    // the full-depth greedy-identity tests were pinned with.
    const int64_t kv_group = c.d_head <= 64 ? std::max<int64_t>(1, (m->max_seq * c.d_head + 16383) / 16384)
                                            : kMaxGroup;
    m->attn_group = static_cast<int>(std::min<int64_t>({G / m->n_units, kMaxGroup, kv_group}));
    if (m->attn_group_max > 0) m->attn_group = std::min(m->attn_group, m->attn_group_max);
    std::vector<CtaPlan> plan(G);
    const int64_t qkv_pairs = m->qkv_rows() / 2;
    const int64_t glu_static = c.d_inter;
    // slice k of every streamed matrix goes to CTA ord[k]; boundaries follow
    // the cumulative per-SM weights (all 1 unless ffb_calibrate ran)
    if ((int64_t)m->sm_weight.size() != G) m->sm_weight.assign(G, 1.0);
    std::vector<double> cum(G + 1, 0.0);
    for (int64_t k = 0; k < G; ++k)
        cum[k + 1] = cum[k] + m->sm_weight[m->plan_reverse ? G - 1 - k : k];
    // calib_mask bit 0/1/2/3: QKV / AOUT / GLU / LM head rows follow the
    // weights (the others split uniformly)
    if ((int64_t)m->lm_weight.size() != G) m->lm_weight.assign(G, 1.0);
    std::vector<double> cum_lm(G + 1, 0.0);
    for (int64_t k = 0; k < G; ++k)
        cum_lm[k + 1] = cum_lm[k] + m->lm_weight[m->plan_reverse ? G - 1 - k : k];
    auto wsplit_m = [&](int64_t units, int64_t k, int bit) {
        if (k >= G) return units;
        if (!((m->calib_mask >> bit) & 1)) return (units * k) / G;
        const std::vector<double>& cw = bit == 3 ? cum_lm : cum;
        return std::min<int64_t>(units, std::llround(units * cw[k] / cw[G]));
    };
    // batch >= 8: row ranges in whole 8-row groups (the tcgen05 weight
    // layout, decode_kernel.cuh frag_off): QKV / GLU in units of 4 pairs
    const int64_t g8 = m->ops->kc > 0 ? 8 : 1;
    if (qkv_pairs % (g8 / 2 > 0 ? g8 / 2 : 1) != 0 || c.d_model % g8 != 0 ||
        glu_static % (g8 / 2 > 0 ? g8 / 2 : 1) != 0 || c.vocab_size % g8 != 0)
        return fail(FFB_UNSUPPORTED, "batch >= 8: matrix rows must split in 8-row groups");
    auto wsplit_g = [&](int64_t units, int64_t k, int bit, int64_t gran) {
        return gran * wsplit_m(units / gran, k, bit);
    };
    const int64_t gp = g8 > 1 ? g8 / 2 : 1;  // pairs per group
    for (int64_t i = 0; i < G; ++i) {
        CtaPlan& p = plan[i];
        std::memset(&p, 0, sizeof(p));
        const int64_t k = m->plan_reverse ? G - 1 - i : i;  // weight-slice order
        p.qkv_r0 = static_cast<int32_t>(2 * wsplit_g(qkv_pairs, k, 0, gp));
        p.qkv_r1 = static_cast<int32_t>(2 * wsplit_g(qkv_pairs, k + 1, 0, gp));
        p.aout_r0 = static_cast<int32_t>(wsplit_g(c.d_model, k, 1, g8));
        p.aout_r1 = static_cast<int32_t>(wsplit_g(c.d_model, k + 1, 1, g8));
        p.glu_t0 = static_cast<int32_t>(wsplit_g(glu_static, k, 2, gp));
        p.glu_t1 = static_cast<int32_t>(wsplit_g(glu_static, k + 1, 2, gp));
        p.lm_r0 = static_cast<int32_t>(wsplit_g(c.vocab_size, k, 3, g8));
        p.lm_r1 = static_cast<int32_t>(wsplit_g(c.vocab_size, k + 1, 3, g8));
        p.red_c0 = static_cast<int32_t>(split_at(c.d_model, i, G));
        p.red_c1 = static_cast<int32_t>(split_at(c.d_model, i + 1, G));
        if (i < static_cast<int64_t>(m->n_units) * m->attn_group) {
            p.attn_unit = static_cast<int32_t>(i / m->attn_group);
            p.attn_g = static_cast<int32_t>(i % m->attn_group);
        } else {
            p.attn_unit = -1;
            p.attn_g = 0;
        }
        // kv heads whose q / k / v rows intersect [qkv_r0, qkv_r1)
        {
            const int64_t QR = c.n_q_heads * c.d_head, KR = c.n_kv_heads * c.d_head;
            const int64_t qpg = c.n_q_heads / c.n_kv_heads;
            p.qkv_heads = 0;
            for (int64_t r = p.qkv_r0; r < p.qkv_r1; ++r) {
                const int64_t h = r < QR ? r / (qpg * c.d_head)
                                         : (r < QR + KR ? (r - QR) / c.d_head
                                                        : (r - QR - KR) / c.d_head);
                p.qkv_heads |= 1 << h;
            }
        }
        if (p.glu_t1 - p.glu_t0 > m->ops->tmax || p.aout_r1 - p.aout_r0 > m->ops->tmax)
            return fail(FFB_UNSUPPORTED, "d_inter too large for the per-CTA GLU buffer");
    }
    if (c.n_kv_heads > 31) return fail(FFB_UNSUPPORTED, "more than 31 kv heads");
    for (int64_t i = 0; i < G; ++i) {  // S_ATTN dependency counts per kv head
        CtaPlan& p = plan[i];
        p.attn_dep = 0;
        if (p.attn_unit < 0) continue;
        const int h = p.attn_unit % static_cast<int>(c.n_kv_heads);
        for (int64_t j = 0; j < G; ++j) p.attn_dep += (plan[j].qkv_heads >> h) & 1;
    }
    m->plan_host = plan;
    return upload_plan(m);
}

// SM id -> dense rank table for persistent launches (decode_kernel.cuh:
// DecodeCta ctor).  Left null (block index = plan index) if the probe does
// not see `grid` distinct SMs.
ffb_status probe_sm_ranks(ffb_model* m) {
    const int G = m->grid;
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device));
    if (G < std::min(sms, 160)) return FFB_OK;  // partial grid: SM set varies per launch
    int32_t* d_ids = nullptr;
    CUDA_TRY(cudaMalloc(&d_ids, sizeof(int32_t) * G));
    cudaError_t e = cudaFuncSetAttribute(smid_probe_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, m->ops->smem);
    if (e == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = m->ops->smem;
        cfg.stream = m->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, smid_probe_kernel, d_ids);
    }
    std::vector<int32_t> ids(G, -1);
    if (e == cudaSuccess) e = cudaStreamSynchronize(m->stream);
    if (e == cudaSuccess)
        e = cudaMemcpy(ids.data(), d_ids, sizeof(int32_t) * G, cudaMemcpyDeviceToHost);
    cudaFree(d_ids);
    if (e != cudaSuccess) return fail(FFB_DEVICE, "SM probe: %s", cudaGetErrorString(e));
    std::vector<int32_t> sorted = ids;
    std::sort(sorted.begin(), sorted.end());
    if (sorted.front() < 0 || std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
        return FFB_OK;  // not one CTA per distinct SM: keep block-index plans
    std::vector<int16_t> table(sorted.back() + 1, 0);
    for (int r = 0; r < G; ++r) table[sorted[r]] = static_cast<int16_t>(r);
    ffb_status st = m->alloc(&m->sm_rank, table.size());
    if (st) return st;
    CUDA_TRY(cudaMemcpy(m->sm_rank, table.data(), sizeof(int16_t) * table.size(),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaDeviceSynchronize());
    return FFB_OK;
}

DecodeParams make_params(const ffb_model* m, int64_t pos, const int64_t* d_tokens,
                         float* d_logits, int64_t* d_greedy) {
    DecodeParams p{};
    p.wqkv = m->wqkv;
    p.waout = m->waout;
    p.wffn1 = m->wffn1;
    p.wffn2t = m->wffn2t;
    p.norm_attn = m->norm_attn;
    p.norm_ffn = m->norm_ffn;
    p.final_norm = m->final_norm;
    p.embedding = m->embedding;
    p.lm_head = m->lm_head;
    p.kcache = m->kcache;
    p.vcache = m->vcache;
    p.x = m->x;
    p.xfrag_a = m->xfrag_a;
    p.xfrag_f = m->xfrag_f;
    p.afrag = m->afrag;
    p.hfrag = m->hfrag;
    p.ssq = m->ssq;
    p.q = m->q;
    p.attn_out = m->attn_out;
    p.glu_part = m->glu_part;
    p.attn_part = m->attn_part;
    p.logits = d_logits ? d_logits : m->logits;
    p.amax_val = m->amax_val;
    p.amax_idx = m->amax_idx;
    p.greedy = d_greedy ? d_greedy : m->greedy;
    p.counters = m->counters;
    p.head_counters = m->head_counters;
    p.qkv_head_counters = m->qkv_head_counters;
    p.amax_counter = m->amax_counter;
    p.plan = m->plan;
    p.tokens = d_tokens;
    p.err_flag = m->greedy ? reinterpret_cast<uint32_t*>(m->greedy + m->cfg.batch) : nullptr;
    p.vocab_embed = static_cast<int32_t>(m->gcfg.vocab_size);
    p.max_seq = m->max_seq;
    p.layers = static_cast<int32_t>(m->cfg.layers);
    p.vocab = static_cast<int32_t>(m->cfg.vocab_size);
    p.pos = static_cast<int32_t>(pos);
    p.epoch = m->epoch;
    p.stage_begin = 0;
    p.stage_end = static_cast<int32_t>(m->cfg.layers * kStagesPerLayer + 1);
    p.overlap = m->mode == FFB_MODE_FUSED_OVERLAP ? 1 : 0;
    p.stage_mask = m->stage_mask;
    p.attn_group = m->attn_group;
    p.n_units = m->n_units;
    p.eps = static_cast<float>(m->cfg.rmsnorm_eps);
    p.rope_theta = m->cfg.rope_theta;
    p.debug = m->debug;
    p.trace = m->trace;
    p.l2_prefetch = m->l2_prefetch;
    p.l2_pf_stages = m->l2_pf_stages;
    p.l2_pf_delay_ns = m->l2_pf_delay;
    p.sm_rank = (m->mode == FFB_MODE_BASELINE || !m->use_sm_rank) ? nullptr : m->sm_rank;
    p.kind = m->cfg.kind;
    p.wlin = m->wlin;
    p.xbuf = m->xbuf;
    if (m->cfg.kind == 1) p.stage_end = static_cast<int32_t>(m->cfg.layers);
    p.tp_size = m->tp_size;
    p.tp_rank = m->tp_rank;
    p.tp_host = m->mode == FFB_MODE_BASELINE_NCCL ? 1 : 0;
    p.vocab_base = static_cast<int32_t>(m->vocab_base);
    for (int r = 0; r < kMaxTP; ++r) {
        p.xch[r] = m->peer_xch[r];
        p.xflag[r] = m->peer_xflag[r];
    }
    return p;
}

// Zero every inter-CTA counter (stage, head-combine, argmax); the caller
// restarts epochs from 0.  Needed before the epoch wraps and whenever the
// plan changes (per-head arrival counts depend on it).
ffb_status reset_sync_state(ffb_model* m, cudaStream_t stream) {
    const int64_t Lc = std::max<int64_t>(1, m->cfg.layers);
    if (m->cfg.kind == 1) {
        CUDA_TRY(cudaMemsetAsync(m->counters, 0, sizeof(uint32_t) * (Lc + 1), stream));
        return FFB_OK;
    }
    CUDA_TRY(cudaMemsetAsync(m->counters, 0, sizeof(uint32_t) * (Lc * 5 + 2), stream));
    if (m->xflag) CUDA_TRY(cudaMemsetAsync(m->xflag, 0, m->xflag_bytes, stream));
    CUDA_TRY(cudaMemsetAsync(m->qkv_head_counters, 0,
                             sizeof(uint32_t) * Lc * m->cfg.n_kv_heads, stream));
    CUDA_TRY(cudaMemsetAsync(m->head_counters, 0,
                             sizeof(uint32_t) * std::max<int64_t>(1, Lc * m->n_units), stream));
    CUDA_TRY(cudaMemsetAsync(m->amax_counter, 0, sizeof(uint32_t), stream));
    return FFB_OK;
}

// ---- host-NCCL multi-kernel TP baseline (FFB_MODE_BASELINE_NCCL) ----------
// NCCL is loaded at run time: the library works (and the other modes run)
// where it is absent.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*);
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t);
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    const char* (*error_string)(ncclResult_t);
};

const NcclApi* nccl_api() {
    static NcclApi api{};
    static bool ok = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
        api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
        api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
        return api.get_unique_id && api.comm_init_rank && api.all_reduce && api.all_gather &&
               api.comm_destroy && api.error_string;
    }();
    return ok ? &api : nullptr;
}

#define NCCL_TRY(expr)                                                                         \
    do {                                                                                       \
        ncclResult_t r_ = (expr);                                                              \
        if (r_ != ncclSuccess) return fail(FFB_DEVICE, "%s: %s", #expr, nccl_api()->error_string(r_)); \
    } while (0)

__global__ void apply_delta_kernel(float* __restrict__ x, const float* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] += d[i];
}

// greedy[b] from the ranks' (value, global index) candidates [tp][B][2]:
// ranks own ascending vocab slices, so scanning them in order and keeping the
// first maximum is the lowest index on ties (numerics.hpp:169-175)
__global__ void amax_pick_kernel(const float* __restrict__ cand, int tp, int B, int64_t* __restrict__ greedy) {
    const int b = threadIdx.x;
    if (b >= B) return;
    float bv = -INFINITY;
    int bi = 0;
    for (int r = 0; r < tp; ++r) {
        const float v = cand[((size_t)r * B + b) * 2];
        const int i = __float_as_int(cand[((size_t)r * B + b) * 2 + 1]);
        if (r == 0 || v > bv) {
            bv = v;
            bi = i;
        }
    }
    greedy[b] = bi;
}

// Each stage its own launch (as FFB_MODE_BASELINE); after S_AOUT and S_RED
// of every layer the ranks' residual deltas (own exchange slot, written by
// tp_exchange_add) are summed by ncclAllReduce on the launch stream and added
// to x; after the LM head the argmax candidates are ncclAllGather'ed.
ffb_status launch_step_nccl(ffb_model* m, DecodeParams p, cudaStream_t stream) {
    const auto* nc = nccl_api();
    if (!nc || !m->nccl_comm || m->tp_size < 2 || m->cfg.kind != 0)
        return fail(FFB_USAGE, "BASELINE_NCCL: tensor-parallel ranks with ffb_tp_nccl_init only");
    auto comm = static_cast<ncclComm_t>(m->nccl_comm);
    const int64_t L = m->cfg.layers, B = m->cfg.batch, D = m->cfg.d_model;
    const int n = static_cast<int>(L * kStagesPerLayer + 1);
    for (int s = 0; s < n; ++s) {
        p.stage_begin = s;
        p.stage_end = s + 1;
        CUDA_TRY(m->ops->launch(p, m->grid, stream, false));
        const int sk = s % kStagesPerLayer;
        if (s < L * kStagesPerLayer && (sk == S_AOUT || sk == S_RED)) {
            const int64_t l = s / kStagesPerLayer, slot = sk == S_AOUT ? 0 : 1;
            float* d = m->xch + (size_t)(slot * 2 + (l & 1)) * B * D;
            NCCL_TRY(nc->all_reduce(d, d, (size_t)(B * D), ncclFloat32, ncclSum, comm, stream));
            apply_delta_kernel<<<std::max<int64_t>(1, (B * D + 255) / 256), 256, 0, stream>>>(m->x, d, B * D);
            CUDA_TRY(cudaGetLastError());
        }
    }
    const float* mine = m->xch + (size_t)4 * B * D + (size_t)m->tp_rank * B * 2;
    NCCL_TRY(nc->all_gather(mine, m->amax_gather, (size_t)(B * 2), ncclFloat32, comm, stream));
    amax_pick_kernel<<<1, 32 * ((B + 31) / 32), 0, stream>>>(m->amax_gather, m->tp_size, static_cast<int>(B),
                                                            p.greedy);
    CUDA_TRY(cudaGetLastError());
    return FFB_OK;
}

ffb_status launch_step(ffb_model* m, int64_t pos, const int64_t* d_tokens, float* d_logits,
                       int64_t* d_greedy, cudaStream_t stream) {
    m->epoch += 1;
    if (m->epoch >= 0x00ffffffu) {  // keep epoch * grid far from u32 wrap
        ffb_status s = reset_sync_state(m, stream);
        if (s) return s;
        m->epoch = 1;
    }
    DecodeParams p = make_params(m, pos, d_tokens, d_logits, d_greedy);
    if (m->mode == FFB_MODE_BASELINE_NCCL) return launch_step_nccl(m, p, stream);
    if (m->mode == FFB_MODE_BASELINE) {
        const int n = m->cfg.kind == 1 ? static_cast<int>(m->cfg.layers)
                                       : static_cast<int>(m->cfg.layers * kStagesPerLayer + 1);
        for (int s = 0; s < n; ++s) {
            // (component ablation: a masked stage is not launched -- except
            // stage 0, whose launch also initialises the residual)
            if (m->cfg.kind == 0 && s > 0 && s < n - 1 && !((m->stage_mask >> (s % kStagesPerLayer)) & 1))
                continue;
            p.stage_begin = s;
            p.stage_end = s + 1;
            CUDA_TRY(m->ops->launch(p, m->grid, stream, false));
        }
    } else {
        CUDA_TRY(m->ops->launch(p, m->grid, stream, true));
    }
    return FFB_OK;
}

// Destination of one reference tensor: kind 0 = streamed matrix (rows of
// `row_bytes`, bf16 or packed quant), 1 = f32 vector, 2 = bf16 embedding.
// The caller passes the WHOLE reference tensor (gcols columns); a TP shard
// keeps the rows listed in `rows` (global row ranges, concatenated) and the
// columns [col0, col0 + cols).
struct TensorDst {
    void* ptr = nullptr;
    int kind = 0;
    int64_t gn = 0;          // expected element count of the reference tensor
    int64_t gcols = 0;
    int64_t col0 = 0, cols = 0;
    std::vector<std::pair<int64_t, int64_t>> rows;  // [r0, r1) ranges
    size_t row_bytes = 0;
    int layout = 0;  // quant code order: 1 = tensor-core (decode_kernel.cuh: tc_slot)
    bool transpose = false;  // store the shard block transposed (W2 as [D][DI], KTraits::F2R)
    int64_t local_rows() const {
        int64_t n = 0;
        for (auto& r : rows) n += r.second - r.first;
        return n;
    }
};

bool resolve(ffb_model* m, const std::string& name, TensorDst* d) {
    const auto& c = m->cfg;   // shard
    const auto& g = m->gcfg;  // whole model
    const int64_t D = c.d_model, r = m->tp_rank;
    const size_t RB = m->ops->row_bytes;
    auto mat = [&](void* ptr, int64_t grows, std::vector<std::pair<int64_t, int64_t>> rows,
                   int64_t col0, int64_t cols, size_t rb) {
        d->ptr = ptr;
        d->kind = 0;
        d->gn = grows * D;
        d->gcols = D;
        d->col0 = col0;
        d->cols = cols;
        d->rows = std::move(rows);
        d->row_bytes = rb;
    };
    auto vec = [&](void* ptr, int64_t n, int kind) {
        d->ptr = ptr;
        d->kind = kind;
        d->gn = n;
        d->gcols = kind == 2 ? D : n;
        d->col0 = 0;
        d->cols = d->gcols;
        d->rows = {{0, n / d->gcols}};
        d->row_bytes = kind == 2 ? D * 2 : n * 4;
    };
    if (c.kind == 1) {  // stacked linear: "linear.<l>" (d x d), "residual" (batch x d)
        if (name == "residual") {
            vec(m->xbuf, c.batch * D, 1);
            return true;
        }
        if (name.rfind("linear.", 0) != 0) return false;
        int64_t l = -1;
        try {
            l = std::stoll(name.substr(7));
        } catch (...) {
            return false;
        }
        if (l < 0 || l >= c.layers) return false;
        mat(m->wlin + l * D * RB, D, {{0, D}}, 0, D, RB);
        return true;
    }
    if (name == "embedding") { vec(m->embedding, g.vocab_size * D, 2); return true; }
    if (name == "lm_head") {
        mat(m->lm_head, g.vocab_size, {{m->vocab_base, m->vocab_base + c.vocab_size}}, 0, D, RB);
        d->layout = m->ops->tc_d;
        return true;
    }
    if (name == "final_norm") { vec(m->final_norm, D, 1); return true; }
    if (name.rfind("layer.", 0) != 0) return false;
    size_t dot = name.find('.', 6);
    if (dot == std::string::npos) return false;
    int64_t l = -1;
    try {
        l = std::stoll(name.substr(6, dot - 6));
    } catch (...) {
        return false;
    }
    if (l < 0 || l >= c.layers) return false;
    std::string t = name.substr(dot + 1);
    const int64_t QR = m->qkv_rows(), dh = c.d_head;
    const int64_t AD = c.n_q_heads * dh;  // shard attention width
    const int64_t gQ = g.n_q_heads * dh, gK = g.n_kv_heads * dh, KVl = c.n_kv_heads * dh;
    d->layout = 0;
    if (t == "wqkv")  // this shard's q heads, then its k heads, then its v heads
        mat(m->wqkv + l * QR * RB, (g.n_q_heads + 2 * g.n_kv_heads) * dh,
            {{r * AD, (r + 1) * AD}, {gQ + r * KVl, gQ + (r + 1) * KVl},
             {gQ + gK + r * KVl, gQ + gK + (r + 1) * KVl}},
            0, D, RB);
    else if (t == "waout")  // every output row, the input columns of this shard's q heads
        mat(m->waout + l * D * m->ops->row_bytes_a, D, {{0, D}}, r * AD, AD, m->ops->row_bytes_a);
    else if (t == "wffn1")  // interleaved (in, gate) row pairs of this d_inter slice
        mat(m->wffn1 + l * 2 * c.d_inter * RB, 2 * g.d_inter,
            {{2 * r * c.d_inter, 2 * (r + 1) * c.d_inter}}, 0, D, RB);
    else if (t == "wffn2t") {
        mat(m->wffn2t + l * c.d_inter * RB, g.d_inter, {{r * c.d_inter, (r + 1) * c.d_inter}}, 0,
            D, RB);
        d->transpose = m->ops->ffn2_rows != 0;
    }
    else if (t == "norm_attn") vec(m->norm_attn + l * D, D, 1);
    else if (t == "norm_ffn") vec(m->norm_ffn + l * D, D, 1);
    else return false;
    if (t == "wqkv" || t == "wffn1") d->layout = m->ops->tc_d;
    if (t == "waout") d->layout = m->ops->tc_a;
    return true;
}

// ---- weight packer for the quant formats (quant.hpp:17-60) ----------------
// quantize_group (quant.hpp:42-54) with `levels` = 15 (int4) or 255 (int8):
// scale = range / levels, zero = clamp(round(-lo / scale)), code =
// clamp(round(v / scale + zero)).  Reference stores hold weights already
// snapped to such a grid with the codes discarded (tensor_store.hpp:275-287),
// so the packer re-derives (codes, scale, zero) and accepts them only if
// (code - zero) * scale reproduces every value bit for bit; the scale
// recomputed from the snapped extremes can be off by a few ulps, so nearby
// scales are tried too.  A group with no exact representation (weights that
// were never on a grid) keeps quantize_group's lossy result and is counted.
bool quant_try(const float* v, int n, int levels, float scale, bool exact, uint8_t* codes,
               float* zero) {
    float lo = v[0];
    for (int i = 1; i < n; ++i) lo = std::min(lo, v[i]);
    float z = std::round(-lo / scale);
    z = std::min(std::max(z, 0.0f), static_cast<float>(levels));
    for (int i = 0; i < n; ++i) {
        float c = std::round(v[i] / scale + z);
        c = std::min(std::max(c, 0.0f), static_cast<float>(levels));
        codes[i] = static_cast<uint8_t>(c);
        if (exact && (c - z) * scale != v[i]) return false;
    }
    *zero = z;
    return true;
}

bool quant_group(const float* v, int n, int levels, uint8_t* codes, float* scale, float* zero) {
    float lo = v[0], hi = v[0];
    for (int i = 1; i < n; ++i) {
        lo = std::min(lo, v[i]);
        hi = std::max(hi, v[i]);
    }
    const float range = hi - lo;
    const float s0 = range > 0 ? range / static_cast<float>(levels) : 1.0f;
    // candidate scale c, tried at +-ulps: the snapped extremes usually sit on
    // codes 0 and `levels` (s = range / levels), but float rounding can land
    // the maximum one code lower, and sparse groups need the step itself
    auto try_near = [&](float c, int ulps) {
        if (!(c > 0) || !std::isfinite(c)) return false;
        for (int d = 0; d <= ulps; ++d)
            for (int sign = -1; sign <= 1; sign += 2) {
                if (d == 0 && sign > 0) continue;
                float sc = c;
                for (int k = 0; k < d; ++k) sc = std::nextafter(sc, sign > 0 ? INFINITY : 0.0f);
                if (quant_try(v, n, levels, sc, true, codes, zero)) {
                    *scale = sc;
                    return true;
                }
            }
        return false;
    };
    if (try_near(s0, 8)) return true;
    if (range > 0) {
        for (int k = levels - 1; k >= levels - 2; --k)
            if (try_near(range / static_cast<float>(k), 4)) return true;
        float step = INFINITY;  // smallest gap between distinct values
        std::vector<float> u(v, v + n);
        std::sort(u.begin(), u.end());
        for (int i = 1; i < n; ++i)
            if (u[i] > u[i - 1]) step = std::min(step, u[i] - u[i - 1]);
        if (try_near(step, 4)) return true;
        if (lo < 0)
            for (int z = 1; z <= levels; ++z)
                if (try_near(-lo / static_cast<float>(z), 2)) return true;
        if (hi > 0)
            for (int k = 1; k <= levels; ++k)
                if (try_near(hi / static_cast<float>(k), 2)) return true;
    }
    quant_try(v, n, levels, s0, false, codes, zero);
    *scale = s0;
    return false;
}

// Byte / nibble position of column i (0..127) of a 128-column group in the
// tensor-core code order (decode_kernel.cuh: tc_slot, mma.sync m16n8k32 u8
// A fragments): lane quad q owns columns 32s + 4q + {0..3} (reg a0 / a1) and
// 32s + 16 + 4q + {0..3} (reg a2 / a3) of k32-step s of a 128-column group.
//   int4: 64 bytes = q-major 16-byte blocks of 4 words, word s = step s:
//         nibble 2j = column 4q + j, nibble 2j + 1 = column 16 + 4q + j, so
//         w & 0x0F0F0F0F and (w >> 4) & 0x0F0F0F0F are the two registers.
//   int8: 128 bytes = q-major 32-byte blocks, 8 bytes per step: columns
//         4q + {0..3}, then 16 + 4q + {0..3}.
static int tc_nibble_index(int i) {  // int4: nibble index (byte * 2 + high) in the group
    const int s = i / 32, r = i % 32, half = r / 16, q = (r % 16) / 4, j = r % 4;
    return q * 32 + s * 8 + 2 * j + half;
}

static int tc_byte_index(int i) {  // int8: byte index in the group
    const int s = i / 32, r = i % 32, half = r / 16, q = (r % 16) / 4, j = r % 4;
    return q * 32 + s * 8 + half * 4 + j;
}

// One row of `cols` f32 values -> the device row format of decode_kernel.cuh
// (codes | f32 scales | u8 zeros | pad); layout 1 = tensor-core code order.
// Returns the inexact group count.
int pack_quant_row(const float* v, int64_t cols, int qb, uint8_t* out, size_t row_bytes,
                   int layout = 0) {
    const int levels = qb == 4 ? 15 : 255;
    const int64_t ng = cols / kQuantGroup;
    const int64_t code_bytes = qb == 4 ? cols / 2 : cols;
    std::memset(out, 0, row_bytes);
    uint8_t codes[kQuantGroup];
    int inexact = 0;
    for (int64_t g = 0; g < ng; ++g) {
        float sc = 1.f, z = 0.f;
        if (!quant_group(v + g * kQuantGroup, kQuantGroup, levels, codes, &sc, &z)) ++inexact;
        for (int i = 0; i < kQuantGroup; ++i) {
            int64_t pos = g * kQuantGroup + i;  // nibble (int4) / byte (int8) position
            if (layout == 1) pos = g * kQuantGroup + (qb == 4 ? tc_nibble_index(i) : tc_byte_index(i));
            if (qb == 4) out[pos / 2] |= static_cast<uint8_t>(codes[i] << (4 * (pos & 1)));
            else out[pos] = codes[i];
        }
        std::memcpy(out + code_bytes + 4 * g, &sc, 4);
        out[code_bytes + 4 * ng + g] = static_cast<uint8_t>(z);
    }
    return inexact;
}

size_t kv_offset(const ffb_model* m, int64_t b, int64_t l, int64_t h, int64_t pos) {
    const auto& c = m->cfg;
    return ((((size_t)l * c.batch + b) * c.n_kv_heads + h) * (size_t)m->max_seq + pos) * c.d_head;
}

bool pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

const char* ffb_last_error(void) { return g_err.c_str(); }
const char* ffb_version(void) { return "ffb200 0.1.0 (sm_100a)"; }

int64_t ffb_quant_row_bytes(int64_t cols, int32_t quant_bits) {
    if (cols <= 0 || cols % kQuantGroup || (quant_bits != 0 && quant_bits != 4 && quant_bits != 8))
        return -1;
    return weight_row_bytes(static_cast<int>(cols), quant_bits);
}

int64_t ffb_pack_quant_rows(const float* values, int64_t rows, int64_t cols, int32_t quant_bits,
                            uint8_t* out) {
    return ffb_pack_quant_rows_ex(values, rows, cols, quant_bits, 0, out);
}

int64_t ffb_pack_quant_rows_ex(const float* values, int64_t rows, int64_t cols,
                               int32_t quant_bits, int32_t layout, uint8_t* out) {
    const int64_t rb = ffb_quant_row_bytes(cols, quant_bits);
    if (!values || !out || rows < 0 || rb < 0 || quant_bits == 0) {
        fail(FFB_USAGE, "pack_quant_rows: bad arguments");
        return -1;
    }
    int64_t inexact = 0;
    for (int64_t r = 0; r < rows; ++r)
        inexact += pack_quant_row(values + r * cols, cols, quant_bits, out + r * rb, rb, layout);
    return inexact;
}

int ffb_config_supported(const ffb_model_config* cfg) {
    if (!cfg) return 0;
    return find_ops(*cfg) != nullptr ? 1 : 0;
}

ffb_status ffb_create(const ffb_model_config* cfg, int64_t max_seq_len, int device, int tp_rank,
                      int tp_size, ffb_model** out) {
    return ffb_create_ex(cfg, max_seq_len, device, tp_rank, tp_size, 0, out);
}

// The shard of rank `r` of `tp`: kv heads
// [r NKV/tp, (r+1) NKV/tp) with their q heads, d_inter slice r, vocab slice r.
static ffb_status shard_config(const ffb_model_config& g, int r, int tp, ffb_model_config* out) {
    if (tp < 1 || tp > kMaxTP) return fail(FFB_USAGE, "tp_size must be in [1, %d]", kMaxTP);
    if (r < 0 || r >= tp) return fail(FFB_USAGE, "tp_rank %d out of range", r);
    if (g.n_kv_heads % tp || g.d_inter % tp || g.vocab_size % tp)
        return fail(FFB_UNSUPPORTED,
                    "tensor parallelism needs n_kv_heads, d_inter and vocab_size divisible by tp");
    *out = g;
    out->n_q_heads = g.n_q_heads / tp;
    out->n_kv_heads = g.n_kv_heads / tp;
    out->d_inter = g.d_inter / tp;
    out->vocab_size = g.vocab_size / tp;
    return FFB_OK;
}

ffb_status ffb_create_ex(const ffb_model_config* gcfg, int64_t max_seq_len, int device,
                         int tp_rank, int tp_size, int grid, ffb_model** out) {
    if (!out) return fail(FFB_USAGE, "out is NULL");
    *out = nullptr;
    ffb_status st = validate_cfg(gcfg);
    if (st) return st;
    ffb_model_config local = *gcfg;
    if (gcfg->kind == 1) {
        if (tp_size != 1) return fail(FFB_UNSUPPORTED, "stacked_linear: tensor parallelism not built");
    } else {
        st = shard_config(*gcfg, tp_rank, tp_size, &local);
        if (st) return st;
    }
    const ffb_model_config* cfg = &local;
    if (max_seq_len < 1) return fail(FFB_VALIDATION, "max_seq_len must be >= 1");
    const KernelOps* ops = find_ops(*cfg);
    if (!ops)
        return fail(FFB_UNSUPPORTED,
                    "no kernel specialisation for d_model=%lld d_inter=%lld d_head=%lld "
                    "heads=%lld/%lld batch=%lld quant=%d",
                    (long long)cfg->d_model, (long long)cfg->d_inter, (long long)cfg->d_head,
                    (long long)cfg->n_q_heads, (long long)cfg->n_kv_heads, (long long)cfg->batch,
                    cfg->quant_bits);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(FFB_DEVICE, "no CUDA device visible (this library has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) return fail(FFB_USAGE, "device %d out of range", device);
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(FFB_DEVICE, "device %d is sm_%d%d; this build targets sm_100a", device,
                    prop.major, prop.minor);
    int coop = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) return fail(FFB_DEVICE, "device lacks cooperative launch");

    auto m = new ffb_model();
    m->cfg = *cfg;
    m->gcfg = *gcfg;
    m->tp_rank = tp_rank;
    m->tp_size = tp_size;
    m->vocab_base = cfg->vocab_size * tp_rank;
    m->ops = ops;
    m->device = device;
    m->grid = std::min(prop.multiProcessorCount, 160);  // KTraits::kMaxGrid
    if (grid > 0) m->grid = std::min(m->grid, grid);    // e.g. TP ranks sharing one GPU
    if (tp_size > 1) m->calib_mask = 0xf & ~0x2;        // S_AOUT rows must match across ranks
    m->max_seq = max_seq_len;
    m->kv_len.assign(cfg->layers, 0);
    auto bail = [&](ffb_status s) {
        delete m;
        return s;
    };
    if (ops->prepare() != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(FFB_DEVICE, "cannot configure kernel shared memory"));
    }
    if (cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(FFB_DEVICE, "stream create failed"));

    const auto& c = *cfg;
    const int64_t L = c.layers, D = c.d_model, B = c.batch, V = c.vocab_size;
    const int64_t Lc = std::max<int64_t>(L, 1);
    if (c.kind == 1) {  // stacked linear: weights, ping-pong activations, counters, plan
        m->kv_len.assign(cfg->layers, 0);
        m->l2_prefetch = 0;
        m->tp_connected = true;
        ffb_status s2 = FFB_OK;
        if (!s2) s2 = m->alloc(&m->wlin, (size_t)Lc * D * ops->row_bytes);
        if (!s2) s2 = m->alloc(&m->xbuf, (size_t)2 * B * D);
        if (!s2) s2 = m->alloc(&m->counters, (size_t)Lc + 1);
        if (!s2) s2 = m->alloc(&m->plan, (size_t)m->grid);
        if (!s2) s2 = m->alloc(&m->staging, (size_t)ffb_model::kStagingElems);
        if (s2) return bail(s2);
        if (cudaMemset(m->counters, 0, sizeof(uint32_t) * (Lc + 1)) != cudaSuccess ||
            cudaMemset(m->xbuf, 0, sizeof(float) * 2 * B * D) != cudaSuccess)
            return bail(fail(FFB_DEVICE, "cudaMemset failed"));
        st = build_plan(m);
        if (st) return bail(st);
        st = probe_sm_ranks(m);
        if (st) return bail(st);
        *out = m;
        return FFB_OK;
    }
#define ALLOC(ptr, n)                 \
    do {                              \
        ffb_status s_ = m->alloc(&(ptr), (n)); \
        if (s_) return bail(s_);      \
    } while (0)
    const size_t RB = ops->row_bytes;
    ALLOC(m->wqkv, (size_t)Lc * m->qkv_rows() * RB);
    ALLOC(m->waout, (size_t)Lc * D * ops->row_bytes_a);  // rows of AD = NQ_local * dh columns
    ALLOC(m->wffn1, (size_t)Lc * 2 * c.d_inter * RB);
    ALLOC(m->wffn2t, (size_t)Lc * c.d_inter * RB);
    ALLOC(m->norm_attn, (size_t)Lc * D);
    ALLOC(m->norm_ffn, (size_t)Lc * D);
    ALLOC(m->final_norm, (size_t)D);
    ALLOC(m->embedding, (size_t)gcfg->vocab_size * D);  // replicated, full vocabulary
    ALLOC(m->lm_head, (size_t)V * RB);                   // this shard's vocab rows
    const size_t kv = (size_t)Lc * B * c.n_kv_heads * max_seq_len * c.d_head;
    ALLOC(m->kcache, kv);
    ALLOC(m->vcache, kv);
    ALLOC(m->x, (size_t)B * D);
    if (B >= 8) {  // A-fragment tables (64 bytes per column: 16 rows x hi/lo bf16)
        ALLOC(m->xfrag_a, (size_t)D * 64);
        ALLOC(m->xfrag_f, (size_t)D * 64);
        ALLOC(m->afrag, (size_t)c.n_q_heads * c.d_head * 64);
        ALLOC(m->hfrag, (size_t)c.d_inter * 64);
        ALLOC(m->ssq, (size_t)2 * m->grid * B);
        // rows >= batch of the MMA tiles stay zero
        if (cudaMemset(m->xfrag_a, 0, (size_t)D * 64) != cudaSuccess ||
            cudaMemset(m->xfrag_f, 0, (size_t)D * 64) != cudaSuccess ||
            cudaMemset(m->afrag, 0, (size_t)c.n_q_heads * c.d_head * 64) != cudaSuccess ||
            cudaMemset(m->hfrag, 0, (size_t)c.d_inter * 64) != cudaSuccess)
            return bail(fail(FFB_DEVICE, "cudaMemset failed"));
    }
    ALLOC(m->q, (size_t)B * D);
    ALLOC(m->attn_out, (size_t)B * D);
    // per-CTA partials, or h = [B][DI] for the two-phase FFN
    ALLOC(m->glu_part, std::max<size_t>((size_t)m->grid * ops->rg * B * D, (size_t)B * c.d_inter));
    const int64_t units = B * c.n_kv_heads;
    const int64_t qpg = c.n_q_heads / c.n_kv_heads;
    ALLOC(m->attn_part, (size_t)units * m->grid * qpg * (c.d_head + 2));
    ALLOC(m->logits, (size_t)B * V);
    ALLOC(m->amax_val, (size_t)m->grid * B);
    ALLOC(m->amax_idx, (size_t)m->grid * B);
    ALLOC(m->greedy, (size_t)B + 1);  // + the device error latch (DecodeParams::err_flag)
    ALLOC(m->tokens_dev, (size_t)B);
    ALLOC(m->counters, (size_t)Lc * 5 + 2);
    ALLOC(m->head_counters, (size_t)Lc * units);
    ALLOC(m->qkv_head_counters, (size_t)Lc * c.n_kv_heads);
    ALLOC(m->amax_counter, 1);
    ALLOC(m->plan, (size_t)m->grid);
    ALLOC(m->staging, (size_t)ffb_model::kStagingElems);
    // TP exchange buffer + flags (also allocated at tp_size 1: harmless, 16 KB)
    m->xch_bytes = sizeof(float) * ((size_t)4 * B * D + (size_t)kMaxTP * B * 2);
    m->xflag_bytes = sizeof(uint32_t) * ((size_t)Lc * 2 * m->grid + 1);
    ALLOC(m->xch, m->xch_bytes / sizeof(float));
    ALLOC(m->xflag, m->xflag_bytes / sizeof(uint32_t));
    ALLOC(m->amax_gather, (size_t)kMaxTP * B * 2);
    if (cudaMemset(m->xflag, 0, m->xflag_bytes) != cudaSuccess ||
        cudaMemset(m->xch, 0, m->xch_bytes) != cudaSuccess)
        return bail(fail(FFB_DEVICE, "cudaMemset failed"));
    m->peer_xch[tp_rank] = m->xch;
    m->peer_xflag[tp_rank] = m->xflag;
    m->tp_connected = tp_size == 1;
#undef ALLOC
    if (cudaMemset(m->counters, 0, sizeof(uint32_t) * (Lc * 5 + 2)) != cudaSuccess ||
        cudaMemset(m->head_counters, 0, sizeof(uint32_t) * Lc * units) != cudaSuccess ||
        cudaMemset(m->qkv_head_counters, 0, sizeof(uint32_t) * Lc * c.n_kv_heads) != cudaSuccess ||
        cudaMemset(m->amax_counter, 0, sizeof(uint32_t)) != cudaSuccess ||
        cudaMemset(m->greedy, 0, sizeof(int64_t) * (B + 1)) != cudaSuccess ||
        cudaMemset(m->kcache, 0, kv * 2) != cudaSuccess ||
        cudaMemset(m->vcache, 0, kv * 2) != cudaSuccess)
        return bail(fail(FFB_DEVICE, "cudaMemset failed"));
    if (cudaMallocHost(&m->tokens_pinned, sizeof(int64_t) * B) != cudaSuccess ||
        cudaMallocHost(&m->greedy_pinned, sizeof(int64_t) * (B + 1)) != cudaSuccess ||
        cudaMallocHost(&m->logits_pinned, sizeof(float) * B * V) != cudaSuccess)
        return bail(fail(FFB_DEVICE, "cudaMallocHost failed"));
    st = build_plan(m);
    if (st) return bail(st);
    // quant stages are dequant-compute bound, and at batch 4 the attention
    // stage streams KV through the ring the whole time: L2 prefetch measured
    // slower in both (int4 +5 %, b4 +7 %); on for bf16 batch 1-2 (-4 %)
    if (ops->QB != 0 || cfg->batch > 2) m->l2_prefetch = 0;
    // Llama-3.1-8B-shaped bf16 decode, batch 1-2, one GPU: hold the window's
    // burst 4.75 us after the layer's first K/V chunk is issued, so that the
    // attention's own K/V (on the chain) is not queued behind ~76 MB of
    // prefetch from every SM.  Same-box sweep (profiles/ab_r02e_pf_delay*.log):
    // b1 2.794 -> 2.729-2.737 ms at 4.5-5 us (a smooth optimum, >= 1.5 %
    // better over 4-5.5 us), b2 3.130 -> 3.063-3.068; other shapes keep 0
    // (1B: +-0.3 % at any hold).  The same hold at 8B contexts 512-8192:
    // -1.1..-2.0 %; Llama-3-70B on one GPU: 22.56 -> 22.32 ms
    // (profiles/ab_r02h_hold_ctx_70b.log).
    if (m->l2_prefetch > 0 && cfg->kind == 0 && (cfg->d_model == 4096 || cfg->d_model == 8192) &&
        cfg->n_kv_heads == 8 && cfg->d_head == 128 && tp_size == 1)
        m->l2_pf_delay = 4750;

    st = probe_sm_ranks(m);
    if (st) return bail(st);
    *out = m;
    return FFB_OK;
}

void ffb_destroy(ffb_model* m) { delete m; }

ffb_status ffb_upload_tensor(ffb_model* m, const char* name, const float* values, int64_t n) {
    if (!m || !name || !values) return fail(FFB_USAGE, "NULL argument");
    TensorDst d;
    if (!resolve(m, name, &d)) return fail(FFB_USAGE, "unknown tensor name '%s'", name);
    if (n != d.gn)
        return fail(FFB_USAGE, "tensor '%s': expected %lld values, got %lld", name,
                    (long long)d.gn, (long long)n);
    CUDA_TRY(cudaSetDevice(m->device));
    if (d.kind == 1) {
        CUDA_TRY(cudaMemcpy(d.ptr, values, sizeof(float) * n, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaDeviceSynchronize());  // landed before any stream reads it
        return FFB_OK;
    }
    // the shard's rows / columns as one contiguous f32 block (no copy at TP 1)
    int64_t lrows = d.local_rows(), cols = d.cols;
    std::vector<float> shard;
    const float* src = values;
    if (d.rows.size() != 1 || d.rows[0].first != 0 || d.cols != d.gcols) {
        shard.resize((size_t)lrows * cols);
        int64_t o = 0;
        for (auto& rr : d.rows)
            for (int64_t r = rr.first; r < rr.second; ++r, ++o)
                std::memcpy(shard.data() + o * cols, values + r * d.gcols + d.col0,
                            sizeof(float) * cols);
        src = shard.data();
    }
    if (d.transpose) {  // [lrows][cols] -> [cols][lrows]
        std::vector<float> tr((size_t)lrows * cols);
        constexpr int64_t TB = 64;  // cache-blocked, blocks of output rows per thread
        parallel_rows((cols + TB - 1) / TB, [&](int64_t b0, int64_t b1) {
            for (int64_t k0 = b0 * TB; k0 < std::min(cols, b1 * TB); k0 += TB)
                for (int64_t r0 = 0; r0 < lrows; r0 += TB)
                    for (int64_t r = r0; r < std::min(lrows, r0 + TB); ++r)
                        for (int64_t k = k0; k < std::min(cols, k0 + TB); ++k)
                            tr[(size_t)k * lrows + r] = src[(size_t)r * cols + k];
        });
        shard.swap(tr);
        src = shard.data();
        std::swap(lrows, cols);
    }
#ifdef FFB_KCP_TCGEN05
    if (d.kind == 0 && m->ops->kc > 0) {
        // batch >= 8 (layout 3, decode_kernel.cuh frag_off / gemv_kc): the
        // tcgen05 B operand, K-major with 128-byte swizzle -- [cols / KC]
        // [rows / 8][KC / 64][8 rows][64 values], the 16-byte units of each
        // 128-byte row piece XOR-swizzled by row & 7; the bf16 values are
        // stored as fp16 (exact in the fp16 normal range, 2^-24 absolute
        // below it; counted in fp16_inexact, out of range rejected)
        const int64_t KC = m->ops->kc, nch = cols / KC, NKA = KC / 64;
        if (lrows % 8 != 0) return fail(FFB_UNSUPPORTED, "batch >= 8: matrix rows must be a multiple of 8");
        std::vector<float> cm((size_t)lrows * cols);
        parallel_rows(lrows, [&](int64_t ra, int64_t rb) {
            for (int64_t r = ra; r < rb; ++r)
                for (int64_t c = 0; c < nch; ++c)
                    for (int64_t ka = 0; ka < NKA; ++ka) {
                        float* dst = cm.data() + ((((size_t)c * (lrows / 8) + r / 8) * NKA + ka) * 8 + (r & 7)) * 64;
                        const float* s0 = src + (size_t)r * cols + c * KC + ka * 64;
                        for (int64_t u = 0; u < 8; ++u)
                            std::memcpy(dst + ((u ^ (r & 7)) * 8), s0 + u * 8, sizeof(float) * 8);
                    }
        });
        shard.swap(cm);
        src = shard.data();
#else
    if (d.kind == 0 && m->ops->kc > 0) {
        // batch >= 8 (layout 2, decode_kernel.cuh gemv_kc, mma.sync path):
        // chunk-major [cols / KC][rows][KC], the 8-column units of each row
        // segment XOR-swizzled by row & 7; the bf16 values are stored as fp16
        // (exact in the fp16 normal range, 2^-24 absolute below it; counted
        // in fp16_inexact, out of range rejected), the tensor-core operand type
        const int64_t KC = m->ops->kc, nch = cols / KC;
        std::vector<float> cm((size_t)lrows * cols);
        parallel_rows(lrows, [&](int64_t ra, int64_t rb) {
            for (int64_t r = ra; r < rb; ++r)
                for (int64_t c = 0; c < nch; ++c) {
                    float* dst = cm.data() + ((size_t)c * lrows + r) * KC;
                    const float* s0 = src + (size_t)r * cols + c * KC;
                    for (int64_t u = 0; u < KC / 8; ++u)
                        std::memcpy(dst + ((u ^ (r & 7)) * 8), s0 + u * 8, sizeof(float) * 8);
                }
        });
        shard.swap(cm);
        src = shard.data();
#endif
        // fp16 range / exactness of the bf16-rounded values
        int64_t over = 0, inexact = 0;
        std::mutex mu;
        parallel_rows(lrows, [&](int64_t ra, int64_t rb) {
            int64_t o = 0, ie = 0;
            for (int64_t i = ra * cols; i < rb * cols; ++i) {
                const float v = bf16_bits_to_f32(bf16_bits_rne(src[i]));
                const float a = std::fabs(v);
                if (!(a <= 65504.f)) ++o;
                else if (a != 0.f && a < 6.103515625e-05f &&
                         std::ldexp(a, 24) != std::floor(std::ldexp(a, 24))) ++ie;
            }
            std::lock_guard<std::mutex> g(mu);
            over += o;
            inexact += ie;
        });
        if (over > 0)
            return fail(FFB_UNSUPPORTED, "batch >= 8: %lld weights of '%s' exceed the fp16 range of the "
                                         "tensor-core operands", (long long)over, name);
        m->fp16_inexact += inexact;
    }
    if (d.kind == 0 && m->ops->QB != 0) {  // quant packer, a block of rows at a time
        const size_t rb = d.row_bytes;
        const int64_t rows_per = std::max<int64_t>(1, (64 << 20) / (int64_t)rb);
        std::vector<uint8_t> buf(rows_per * rb);
        auto* dst = static_cast<uint8_t*>(d.ptr);
        for (int64_t r0 = 0; r0 < lrows; r0 += rows_per) {
            const int64_t nr = std::min(rows_per, lrows - r0);
            std::mutex mu;
            parallel_rows(nr, [&](int64_t ra, int64_t rb2) {
                int64_t n = 0;
                for (int64_t r = ra; r < rb2; ++r)
                    n += pack_quant_row(src + (r0 + r) * cols, cols, m->ops->QB,
                                        buf.data() + r * rb, rb, d.layout);
                std::lock_guard<std::mutex> g(mu);
                m->quant_inexact_groups += n;
            });
            CUDA_TRY(cudaMemcpy(dst + r0 * rb, buf.data(), nr * rb, cudaMemcpyHostToDevice));
        }
        CUDA_TRY(cudaDeviceSynchronize());  // landed before any stream reads it
        return FFB_OK;
    }
    const int64_t ln = lrows * cols;
    auto* dst = static_cast<__nv_bfloat16*>(d.ptr);
    for (int64_t off = 0; off < ln; off += ffb_model::kStagingElems) {
        const int64_t cnt = std::min<int64_t>(ffb_model::kStagingElems, ln - off);
        CUDA_TRY(cudaMemcpyAsync(m->staging, src + off, sizeof(float) * cnt,
                                 cudaMemcpyHostToDevice, m->stream));
        if (d.kind == 0 && m->ops->kc > 0)
            f32_to_bf16_as_f16_kernel<<<1184, 256, 0, m->stream>>>(
                m->staging, reinterpret_cast<__half*>(dst) + off, cnt);
        else
            f32_to_bf16_kernel<<<1184, 256, 0, m->stream>>>(m->staging, dst + off, cnt);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(m->stream));  // staging reused
    }
    return FFB_OK;
}

ffb_status ffb_init_synthetic(ffb_model* m, uint64_t seed) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    CUDA_TRY(cudaSetDevice(m->device));
    if (m->cfg.kind == 1) {
        const int64_t D = m->cfg.d_model;
        synth_bf16_kernel<<<4096, 256, 0, m->stream>>>(reinterpret_cast<__nv_bfloat16*>(m->wlin),
                                                       m->cfg.layers * D * D, seed * 31 + 1,
                                                       1.0f / std::sqrt(static_cast<float>(D)));
        synth_f32_kernel<<<64, 256, 0, m->stream>>>(m->xbuf, m->cfg.batch * D, seed * 31 + 2,
                                                    0.0f, 1.0f);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(m->stream));
        return FFB_OK;
    }
    const auto& c = m->cfg;
    const int64_t L = c.layers, D = c.d_model;
    const float sd = 1.0f / std::sqrt(static_cast<float>(D));
    const float sdi = 1.0f / std::sqrt(static_cast<float>(c.d_inter));
    auto bf = [&](__nv_bfloat16* p, int64_t n, uint64_t s, float stddev) {
        synth_bf16_kernel<<<4096, 256, 0, m->stream>>>(p, n, seed * 1315423911ull + s, stddev);
    };
    auto f32 = [&](float* p, int64_t n, uint64_t s) {
        synth_f32_kernel<<<256, 256, 0, m->stream>>>(p, n, seed * 1315423911ull + s, 1.0f, 0.02f);
    };
    // streamed matrices: bf16 values, or random codes with per-group scales
    // spanning the same +-sqrt(3) stddev range and a mid-range zero point
    // (TP shards draw their own matrices; embedding and norms are replicated)
    const uint64_t rs = 0x9e37ull * static_cast<uint64_t>(m->tp_rank);
    auto mat = [&](uint8_t* p, int64_t rows, int64_t cols, size_t rb, uint64_t s, float stddev) {
        if (m->ops->kc > 0) {
            synth_bf16_as_f16_kernel<<<4096, 256, 0, m->stream>>>(
                reinterpret_cast<__half*>(p), rows * cols, seed * 1315423911ull + s + rs, stddev);
        } else if (m->ops->QB == 0) {
            bf(reinterpret_cast<__nv_bfloat16*>(p), rows * cols, s + rs, stddev);
        } else {
            synth_quant_kernel<<<4096, 256, 0, m->stream>>>(
                p, rows, static_cast<int>(cols), m->ops->QB, static_cast<int>(rb),
                seed * 1315423911ull + s + rs, stddev);
        }
    };
    const size_t RB = m->ops->row_bytes, RBA = m->ops->row_bytes_a;
    const int64_t AD = c.n_q_heads * c.d_head;
    mat(m->wqkv, L * m->qkv_rows(), D, RB, 1, sd);
    mat(m->waout, L * D, AD, RBA, 2, sd);
    mat(m->wffn1, L * 2 * c.d_inter, D, RB, 3, sd);
    mat(m->wffn2t, L * c.d_inter, D, RB, 4, sdi);
    bf(m->embedding, m->gcfg.vocab_size * D, 5, sd);
    mat(m->lm_head, c.vocab_size, D, RB, 6, sd);
    f32(m->norm_attn, L * D, 7);
    f32(m->norm_ffn, L * D, 8);
    f32(m->final_norm, D, 9);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(m->stream));
    return FFB_OK;
}

ffb_status ffb_kv_set(ffb_model* m, int64_t b, int64_t layer, int64_t head, int64_t pos,
                      const float* k, const float* v) {
    if (!m || !k || !v) return fail(FFB_USAGE, "NULL argument");
    const auto& c = m->cfg;
    if (b < 0 || b >= c.batch || layer < 0 || layer >= c.layers || head < 0 ||
        head >= c.n_kv_heads || pos < 0 || pos >= m->max_seq)
        return fail(FFB_VALIDATION, "kv_set: index out of range");
    std::vector<uint16_t> kb(c.d_head), vb(c.d_head);
    for (int64_t d = 0; d < c.d_head; ++d) {
        kb[kv_swz(d, pos)] = bf16_bits_rne(k[d]);
        vb[kv_swz(d, pos)] = bf16_bits_rne(v[d]);
    }
    CUDA_TRY(cudaSetDevice(m->device));
    const size_t off = kv_offset(m, b, layer, head, pos);
    CUDA_TRY(cudaMemcpy(m->kcache + off, kb.data(), 2 * c.d_head, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(m->vcache + off, vb.data(), 2 * c.d_head, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaDeviceSynchronize());  // landed before any stream reads it
    return FFB_OK;
}

ffb_status ffb_kv_get(ffb_model* m, int64_t b, int64_t layer, int64_t head, int64_t pos,
                      float* k, float* v) {
    if (!m || !k || !v) return fail(FFB_USAGE, "NULL argument");
    const auto& c = m->cfg;
    if (b < 0 || b >= c.batch || layer < 0 || layer >= c.layers || head < 0 ||
        head >= c.n_kv_heads || pos < 0 || pos >= m->max_seq)
        return fail(FFB_VALIDATION, "kv_get: index out of range");
    std::vector<uint16_t> kb(c.d_head), vb(c.d_head);
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaStreamSynchronize(m->stream));
    const size_t off = kv_offset(m, b, layer, head, pos);
    CUDA_TRY(cudaMemcpy(kb.data(), m->kcache + off, 2 * c.d_head, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(vb.data(), m->vcache + off, 2 * c.d_head, cudaMemcpyDeviceToHost));
    for (int64_t d = 0; d < c.d_head; ++d) {
        k[d] = bf16_bits_to_f32(kb[kv_swz(d, pos)]);
        v[d] = bf16_bits_to_f32(vb[kv_swz(d, pos)]);
    }
    return FFB_OK;
}

ffb_status ffb_kv_import(ffb_model* m, const float* k, const float* v, int64_t src_max_seq,
                         int64_t n_pos) {
    if (!m || !k || !v) return fail(FFB_USAGE, "NULL argument");
    const auto& c = m->cfg;
    if (n_pos < 0 || n_pos > m->max_seq || n_pos > src_max_seq)
        return fail(FFB_VALIDATION, "kv_import: n_pos out of range");
    CUDA_TRY(cudaSetDevice(m->device));
    std::vector<uint16_t> kb(n_pos * c.d_head), vb(n_pos * c.d_head);
    for (int64_t b = 0; b < c.batch; ++b)
        for (int64_t l = 0; l < c.layers; ++l)
            for (int64_t h = 0; h < c.n_kv_heads; ++h) {
                // the reference layout holds every kv head; take this shard's
                const int64_t gh = m->tp_rank * c.n_kv_heads + h;
                const size_t src =
                    (((size_t)b * c.layers + l) * m->gcfg.n_kv_heads + gh) * src_max_seq * c.d_head;
                for (int64_t ps = 0; ps < n_pos; ++ps)
                    for (int64_t d = 0; d < c.d_head; ++d) {
                        const int64_t i = ps * c.d_head + d;
                        const int64_t o = ps * c.d_head + kv_swz(d, ps);
                        kb[o] = bf16_bits_rne(k[src + i]);
                        vb[o] = bf16_bits_rne(v[src + i]);
                    }
                const size_t off = kv_offset(m, b, l, h, 0);
                CUDA_TRY(cudaMemcpy(m->kcache + off, kb.data(), 2 * n_pos * c.d_head,
                                    cudaMemcpyHostToDevice));
                CUDA_TRY(cudaMemcpy(m->vcache + off, vb.data(), 2 * n_pos * c.d_head,
                                    cudaMemcpyHostToDevice));
            }
    CUDA_TRY(cudaDeviceSynchronize());  // landed before any stream reads it
    return FFB_OK;
}

ffb_status ffb_kv_set_length(ffb_model* m, int64_t layer, int64_t n) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    if (layer < 0 || layer >= m->cfg.layers) return fail(FFB_VALIDATION, "kv_set_length: bad layer");
    if (n < 0 || n > m->max_seq) return fail(FFB_VALIDATION, "kv_set_length: beyond max_seq_len");
    m->kv_len[layer] = n;
    return FFB_OK;
}

int64_t ffb_kv_length(const ffb_model* m, int64_t layer) {
    if (!m || layer < 0 || layer >= m->cfg.layers) return -1;
    return m->kv_len[layer];
}

ffb_status ffb_set_mode(ffb_model* m, ffb_mode mode) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    if (mode != FFB_MODE_BASELINE && mode != FFB_MODE_FUSED && mode != FFB_MODE_FUSED_OVERLAP &&
        mode != FFB_MODE_BASELINE_NCCL)
        return fail(FFB_USAGE, "unknown mode %d", (int)mode);
    if (mode == FFB_MODE_BASELINE_NCCL && (m->tp_size < 2 || !m->nccl_comm))
        return fail(FFB_USAGE, "BASELINE_NCCL: a tensor-parallel rank after ffb_tp_nccl_init");
    if ((mode == FFB_MODE_BASELINE_NCCL) != (m->mode == FFB_MODE_BASELINE_NCCL)) {
        // the in-kernel exchange flags do not advance in the NCCL mode: every
        // counter restarts from a clean epoch (all ranks switch together)
        CUDA_TRY(cudaSetDevice(m->device));
        CUDA_TRY(cudaStreamSynchronize(m->stream));
        CUDA_TRY(cudaDeviceSynchronize());
        ffb_status s = reset_sync_state(m, m->stream);
        if (s) return s;
        CUDA_TRY(cudaStreamSynchronize(m->stream));
        m->epoch = 0;
    }
    m->mode = mode;
    return FFB_OK;
}

ffb_status ffb_set_debug(ffb_model* m, int32_t flags) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    m->debug = flags;
    return FFB_OK;
}

ffb_status ffb_set_option(ffb_model* m, const char* key, int64_t value) {
    if (!m || !key) return fail(FFB_USAGE, "NULL argument");
    if (std::strcmp(key, "l2_prefetch_bytes") == 0) {
        if (value < 0 || value > (64ll << 20))
            return fail(FFB_USAGE, "l2_prefetch_bytes out of range [0, 64 MiB]");
        m->l2_prefetch = value;
        return FFB_OK;
    }
    const bool plan_key = !std::strcmp(key, "calib_mask") || !std::strcmp(key, "plan_reverse") ||
                          !std::strcmp(key, "attn_group_max");
    if (plan_key && m->tp_size > 1)
        return fail(FFB_UNSUPPORTED, "option '%s' changes the plan; not with tensor parallelism", key);
    if (std::strcmp(key, "calib_mask") == 0) {
        if (value < 0 || value > 0xf) return fail(FFB_USAGE, "calib_mask is a 4-bit mask");
        m->calib_mask = static_cast<int>(value);
        CUDA_TRY(cudaSetDevice(m->device));
        CUDA_TRY(cudaDeviceSynchronize());
        ffb_status s = build_plan(m);
        if (s) return s;
        s = reset_sync_state(m, m->stream);
        if (s) return s;
        CUDA_TRY(cudaStreamSynchronize(m->stream));
        m->epoch = 0;
        return FFB_OK;
    }
    if (std::strcmp(key, "sm_rank") == 0) {
        m->use_sm_rank = value ? 1 : 0;
        return FFB_OK;
    }
    if (std::strcmp(key, "prefill_terms") == 0) {
        if (value != 2 && value != 3) return fail(FFB_USAGE, "prefill_terms: 3 (f32-exact) or 2 (bf16 hi + lo)");
        m->prefill_terms = static_cast<int>(value);
        return FFB_OK;
    }
    if (std::strcmp(key, "stage_mask") == 0) {
        if (value != 0x1f && value != 0x07 && value != 0x18)
            return fail(FFB_USAGE, "stage_mask: 0x1f (decoder), 0x07 (attention blocks) or 0x18 (GLU blocks)");
        if (value != 0x1f && (m->cfg.kind != 0 || m->cfg.batch >= 8 || m->tp_size > 1))
            return fail(FFB_UNSUPPORTED, "stage_mask: single-GPU decoder, batch < 8");
        m->stage_mask = static_cast<int32_t>(value);
        return FFB_OK;
    }
    if (std::strcmp(key, "l2_prefetch_delay_ns") == 0) {
        if (value < 0 || value > 100000) return fail(FFB_USAGE, "l2_prefetch_delay_ns in [0, 100000]");
        m->l2_pf_delay = static_cast<int32_t>(value);
        return FFB_OK;
    }
    if (std::strcmp(key, "l2_prefetch_stages") == 0) {
        if (value < 0 || value > 0x3f) return fail(FFB_USAGE, "l2_prefetch_stages is a 6-bit mask");
        m->l2_pf_stages = static_cast<int32_t>(value);
        return FFB_OK;
    }
    if (std::strcmp(key, "plan_reverse") == 0 || std::strcmp(key, "attn_group_max") == 0) {
        if (key[0] == 'p') {
            m->plan_reverse = value ? 1 : 0;
        } else {
            if (value < 0 || value > kMaxGroup) return fail(FFB_USAGE, "attn_group_max in [0, 32]");
            m->attn_group_max = static_cast<int>(value);
        }
        CUDA_TRY(cudaSetDevice(m->device));
        CUDA_TRY(cudaStreamSynchronize(m->stream));
        CUDA_TRY(cudaDeviceSynchronize());
        ffb_status s = build_plan(m);
        if (s) return s;
        s = reset_sync_state(m, m->stream);
        if (s) return s;
        CUDA_TRY(cudaStreamSynchronize(m->stream));
        m->epoch = 0;
        return FFB_OK;
    }
    return fail(FFB_USAGE, "unknown option '%s'", key);
}

ffb_status ffb_set_trace(ffb_model* m, int enable) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    CUDA_TRY(cudaSetDevice(m->device));
    if (enable && !m->trace) {
        const size_t n = (size_t)m->grid * (m->cfg.layers * kStagesPerLayer + 1) * kTraceSlots;
        ffb_status s = m->alloc(&m->trace, n);
        if (s) return s;
        CUDA_TRY(cudaMemset(m->trace, 0, n * sizeof(uint64_t)));
    } else if (!enable) {
        m->trace = nullptr;  // buffer stays owned by the handle
    }
    return FFB_OK;
}

int64_t ffb_get_trace(ffb_model* m, uint64_t* out, int64_t n) {
    if (!m || !m->trace) return -1;
    const int64_t total = (int64_t)m->grid * (m->cfg.layers * kStagesPerLayer + 1) * kTraceSlots;
    if (out) {
        if (n < total) return -1;
        if (cudaStreamSynchronize(m->stream) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess ||
            cudaMemcpy(out, m->trace, total * sizeof(uint64_t), cudaMemcpyDeviceToHost) !=
                cudaSuccess)
            return -1;
    }
    return total;
}

// The device error latch (DecodeParams::err_flag) was set in an earlier step:
// bit 0 a device-resident token id out of range (decode_kernel.cuh:
// token_row, reported like the reference's ValidationError, reference.hpp:
// 43-53); bit 1 (batch >= 8) an activation outside the fp16 range of the
// tensor-core operands (frag_put).  Clears the latch.
static ffb_status latched_token_error(ffb_model* m, int64_t flag) {
    CUDA_TRY(cudaMemsetAsync(m->greedy + m->cfg.batch, 0, sizeof(int64_t), m->stream));
    CUDA_TRY(cudaStreamSynchronize(m->stream));
    if (flag & 1)
        return fail(FFB_VALIDATION,
                    "decode_step: token id out of range (device-resident tokens; row 0 was used)");
    return fail(FFB_UNSUPPORTED,
                "decode_step: an activation exceeded the fp16 range of the batch >= 8 tensor-core "
                "operands (|v| > 65504); logits of that step are not valid");
}

ffb_status ffb_sync(ffb_model* m) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    if (m->cfg.kind != 0) return FFB_OK;
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaDeviceSynchronize());
    int64_t flag = 0;
    CUDA_TRY(cudaMemcpy(&flag, m->greedy + m->cfg.batch, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (flag != 0) return latched_token_error(m, flag);
    return FFB_OK;
}

static ffb_status check_step(ffb_model* m, const int64_t* tokens, int64_t pos) {
    const auto& c = m->cfg;
    if (m->cfg.kind != 0)
        return fail(FFB_VALIDATION, "decode_step: llama_decoder models only (stacked_linear: "
                                    "ffb_linear_forward)");
    if (!m->tp_connected && !(m->mode == FFB_MODE_BASELINE_NCCL && m->nccl_comm))
        return fail(FFB_USAGE, "tensor-parallel rank not connected (ffb_tp_connect)");
    if (tokens)
        for (int64_t b = 0; b < c.batch; ++b)
            if (tokens[b] < 0 || tokens[b] >= m->gcfg.vocab_size)
                return fail(FFB_VALIDATION, "decode_step: token id out of range");
    for (int64_t l = 0; l < c.layers; ++l)
        if (m->kv_len[l] != pos)
            return fail(FFB_VALIDATION, "decode_step: cache length does not match position");
    if (pos < 0 || pos >= m->max_seq)
        return fail(FFB_VALIDATION, "kv_append: cache capacity reached (max_seq_len)");
    return FFB_OK;
}

ffb_status ffb_decode_step(ffb_model* m, const int64_t* tokens, int64_t pos, float* logits_out,
                           int64_t* greedy_out, void* stream) {
    if (!m || !tokens) return fail(FFB_USAGE, "NULL argument");
    ffb_status st = check_step(m, tokens, pos);
    if (st) return st;
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : m->stream;
    const auto& c = m->cfg;
    std::memcpy(m->tokens_pinned, tokens, sizeof(int64_t) * c.batch);
    CUDA_TRY(cudaMemcpyAsync(m->tokens_dev, m->tokens_pinned, sizeof(int64_t) * c.batch,
                             cudaMemcpyHostToDevice, s));
    // logits straight into pinned host memory (the caller's buffer when it is
    // pinned, else the handle's staging buffer): the LM head's stores cross
    // PCIe while the stage still streams, instead of a D2H copy after the
    // kernel (zero-copy; the device logits buffer is then not written)
    const size_t lbytes = sizeof(float) * c.batch * c.vocab_size;
    const bool direct = logits_out && pinned(logits_out);
    float* d_logits = nullptr;
    if (logits_out) {
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, direct ? static_cast<void*>(logits_out) : m->logits_pinned, 0) ==
            cudaSuccess)
            d_logits = static_cast<float*>(dp);
        else
            cudaGetLastError();  // not mapped: copy after the kernel below
    }
    st = launch_step(m, pos, m->tokens_dev, d_logits, nullptr, s);
    if (st) return st;
    if (logits_out && !d_logits)
        CUDA_TRY(cudaMemcpyAsync(direct ? logits_out : m->logits_pinned, m->logits, lbytes,
                                 cudaMemcpyDeviceToHost, s));
    // greedy ids and the device error latch behind them in one copy
    CUDA_TRY(cudaMemcpyAsync(m->greedy_pinned, m->greedy, sizeof(int64_t) * (c.batch + 1),
                             cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (logits_out && !direct) std::memcpy(logits_out, m->logits_pinned, lbytes);
    if (greedy_out) std::memcpy(greedy_out, m->greedy_pinned, sizeof(int64_t) * c.batch);
    for (auto& n : m->kv_len) n += 1;
    if (m->greedy_pinned[c.batch] != 0) return latched_token_error(m, m->greedy_pinned[c.batch]);
    return FFB_OK;
}

ffb_status ffb_decode_step_device(ffb_model* m, const int64_t* d_tokens, int64_t pos,
                                  float* d_logits, int64_t* d_greedy, void* stream) {
    if (!m || !d_tokens) return fail(FFB_USAGE, "NULL argument");
    ffb_status st = check_step(m, nullptr, pos);
    if (st) return st;
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : m->stream;
    st = launch_step(m, pos, d_tokens, d_logits, d_greedy, s);
    if (st) return st;
    for (auto& n : m->kv_len) n += 1;
    return FFB_OK;
}

ffb_status ffb_decode_loop(ffb_model* m, const int64_t* d_tokens, int64_t pos, int32_t n_steps,
                           int32_t teacher_forced, int64_t* d_out, void* stream) {
    if (!m || !d_tokens || !d_out) return fail(FFB_USAGE, "NULL argument");
    if (n_steps < 1) return fail(FFB_USAGE, "decode_loop: n_steps must be >= 1");
    ffb_status st = check_step(m, nullptr, pos);
    if (st) return st;
    if (pos + n_steps > m->max_seq)
        return fail(FFB_VALIDATION, "kv_append: cache capacity reached (max_seq_len)");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : m->stream;
    const int64_t B = m->cfg.batch;
    for (int32_t i = 0; i < n_steps; ++i) {
        // step i reads its tokens from the prompt (teacher forcing) or from
        // the previous step's greedy output, all on the device
        const int64_t* tok = teacher_forced ? d_tokens + (int64_t)i * B
                                            : (i == 0 ? d_tokens : d_out + (int64_t)(i - 1) * B);
        st = launch_step(m, pos + i, tok, nullptr, d_out + (int64_t)i * B, s);
        if (st) return st;
        for (auto& n : m->kv_len) n += 1;
    }
    return FFB_OK;
}

ffb_status ffb_linear_forward_device(ffb_model* m, const float* d_x_in, float* d_x_out,
                                     void* stream) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    if (m->cfg.kind != 1) return fail(FFB_VALIDATION, "linear_forward: stacked_linear models only");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : m->stream;
    const size_t bytes = sizeof(float) * m->cfg.batch * m->cfg.d_model;
    if (d_x_in) CUDA_TRY(cudaMemcpyAsync(m->xbuf, d_x_in, bytes, cudaMemcpyDeviceToDevice, s));
    ffb_status st = launch_step(m, 0, nullptr, nullptr, nullptr, s);
    if (st) return st;
    if (d_x_out)
        CUDA_TRY(cudaMemcpyAsync(d_x_out, m->xbuf + (m->cfg.layers & 1) * m->cfg.batch * m->cfg.d_model,
                                 bytes, cudaMemcpyDeviceToDevice, s));
    return FFB_OK;
}

ffb_status ffb_linear_forward(ffb_model* m, const float* x_in, float* x_out, void* stream) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    if (m->cfg.kind != 1) return fail(FFB_VALIDATION, "linear_forward: stacked_linear models only");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : m->stream;
    const size_t bytes = sizeof(float) * m->cfg.batch * m->cfg.d_model;
    if (x_in) CUDA_TRY(cudaMemcpyAsync(m->xbuf, x_in, bytes, cudaMemcpyHostToDevice, s));
    ffb_status st = launch_step(m, 0, nullptr, nullptr, nullptr, s);
    if (st) return st;
    if (x_out)
        CUDA_TRY(cudaMemcpyAsync(x_out, m->xbuf + (m->cfg.layers & 1) * m->cfg.batch * m->cfg.d_model,
                                 bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FFB_OK;
}

ffb_status ffb_get_info(const ffb_model* m, ffb_info* out) {
    if (!m || !out) return fail(FFB_USAGE, "NULL argument");
    const auto& c = m->cfg;
    out->grid = m->grid;
    out->threads = m->ops->threads;
    out->smem_bytes = m->ops->smem;
    out->ring_slots = m->ops->nslots;
    out->slot_bytes = m->ops->slot_bytes;
    out->attn_group = m->attn_group;
    out->launches_per_step =
        (m->mode == FFB_MODE_BASELINE || m->mode == FFB_MODE_BASELINE_NCCL)
            ? static_cast<int32_t>(c.layers * kStagesPerLayer + 1) : 1;
    out->mode = m->mode;
    const uint64_t row = static_cast<uint64_t>(m->ops->row_bytes);
    if (c.kind == 1) out->weight_bytes = row * static_cast<uint64_t>(c.layers) * c.d_model;
    else out->weight_bytes = row * (static_cast<uint64_t>(c.layers) * (m->qkv_rows() + 3 * c.d_inter) +
                               c.vocab_size) +
                        static_cast<uint64_t>(m->ops->row_bytes_a) * c.layers * c.d_model;
    out->quant_inexact_groups = m->quant_inexact_groups;
    out->fp16_inexact = m->fp16_inexact;
    out->kc_layout = m->ops->kc_layout;
    out->row_bytes = m->ops->row_bytes;
    out->device_bytes = m->device_bytes;
    return FFB_OK;
}

const float* ffb_logits_device(const ffb_model* m) { return m ? m->logits : nullptr; }

ffb_status ffb_calibrate(ffb_model* m, int32_t iterations) {
    if (!m) return fail(FFB_USAGE, "NULL handle");
    if (m->tp_size > 1)
        return fail(FFB_UNSUPPORTED, "calibrate: per-rank plans would desynchronise TP epochs");
    if (m->cfg.kind != 0) return fail(FFB_UNSUPPORTED, "calibrate: llama_decoder models only");
    if (iterations < 0 || iterations > 16) return fail(FFB_USAGE, "iterations in [0, 16]");
    const auto& c = m->cfg;
    const int G = m->grid;
    if (iterations == 0 || c.layers == 0) {  // back to the uniform plan
        m->sm_weight.assign(G, 1.0);
        m->lm_weight.assign(G, 1.0);
    } else {
        const int64_t pos = m->kv_len[0];
        for (int64_t l = 0; l < c.layers; ++l)
            if (m->kv_len[l] != pos)
                return fail(FFB_VALIDATION, "calibrate: layers have different cache lengths");
        if (pos >= m->max_seq) return fail(FFB_VALIDATION, "calibrate: cache is full");
        if (m->sm_rank == nullptr)
            return fail(FFB_UNSUPPORTED, "calibrate: SM ids unavailable (no per-SM plans)");
        CUDA_TRY(cudaSetDevice(m->device));
        uint64_t* saved_trace = m->trace;
        const ffb_mode saved_mode = m->mode;
        ffb_status st = ffb_set_trace(m, 1);
        if (st) return st;
        m->mode = FFB_MODE_FUSED_OVERLAP;
        const int S = static_cast<int>(c.layers * kStagesPerLayer + 1);
        std::vector<uint64_t> tr((size_t)G * S * kTraceSlots);
        CUDA_TRY(cudaMemsetAsync(m->tokens_dev, 0, sizeof(int64_t) * c.batch, m->stream));
        for (int iter = 0; iter < iterations && !st; ++iter) {
            // steps at the current length: they write K/V at `pos` (beyond
            // the cache length, overwritten by the next real step)
            for (int rep = 0; rep < 3 && !st; ++rep)
                st = launch_step(m, pos, m->tokens_dev, nullptr, nullptr, m->stream);
            if (st) break;
            CUDA_TRY(cudaStreamSynchronize(m->stream));
            CUDA_TRY(cudaMemcpy(tr.data(), m->trace, tr.size() * sizeof(uint64_t),
                                cudaMemcpyDeviceToHost));
            // per CTA (= SM rank): median over layers of the GLU stage time
            std::vector<double> t(G, 0.0);
            for (int i = 0; i < G; ++i) {
                std::vector<double> v;
                for (int64_t l = 0; l < c.layers; ++l) {
                    const uint64_t* r = &tr[((size_t)i * S + l * kStagesPerLayer + S_GLU) * kTraceSlots];
                    if (r[1] && r[2] > r[1]) v.push_back(static_cast<double>(r[2] - r[1]));
                }
                if (v.empty()) { t[i] = 0; continue; }
                std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
                t[i] = v[v.size() / 2];
            }
            double tm = 0;
            int nt = 0;
            for (double x : t) if (x > 0) { tm += x; ++nt; }
            if (nt == 0) break;
            tm /= nt;
            // n_i ~ w_i and t_i ~ n_i / rate_i: equal times need w_i ~ w_i tm / t_i
            double sum = 0;
            for (int i = 0; i < G; ++i) {
                if (t[i] > 0) m->sm_weight[i] *= tm / t[i];
                sum += m->sm_weight[i];
            }
            for (int i = 0; i < G; ++i)
                m->sm_weight[i] = std::min(1.3, std::max(0.7, m->sm_weight[i] * G / sum));
            // LM head (the last trace stage): its own weights, from its own
            // per-CTA times (dependency met -> done)
            {
                std::vector<double> tl(G, 0.0);
                double tlm = 0;
                int nl = 0;
                for (int i = 0; i < G; ++i) {
                    const uint64_t* r = &tr[((size_t)i * S + (S - 1)) * kTraceSlots];
                    if (r[1] && r[2] > r[1]) {
                        tl[i] = static_cast<double>(r[2] - r[1]);
                        tlm += tl[i];
                        ++nl;
                    }
                }
                if (nl == G) {
                    tlm /= nl;
                    double ls = 0;
                    for (int i = 0; i < G; ++i) {
                        m->lm_weight[i] *= tlm / tl[i];
                        ls += m->lm_weight[i];
                    }
                    for (int i = 0; i < G; ++i)
                        m->lm_weight[i] = std::min(1.5, std::max(0.6, m->lm_weight[i] * G / ls));
                }
            }
            // a new plan changes per-head arrival counts: restart the epochs
            st = build_plan(m);
            if (!st) st = reset_sync_state(m, m->stream);
            m->epoch = 0;
        }
        m->mode = saved_mode;
        m->trace = saved_trace;
        if (st) return st;
    }
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaDeviceSynchronize());
    ffb_status st = build_plan(m);
    if (st) return st;
    st = reset_sync_state(m, m->stream);
    if (st) return st;
    CUDA_TRY(cudaStreamSynchronize(m->stream));
    m->epoch = 0;
    return FFB_OK;
}

// ---- tensor parallelism: peer exchange buffers ------------------------------
struct TpBlob {
    uint32_t magic, rank, tp, device;
    uint64_t pid;
    uint64_t xch_ptr, xflag_ptr;  // raw pointers (same process)
    cudaIpcMemHandle_t xch_ipc, xflag_ipc;
};

int64_t ffb_tp_blob_bytes(void) { return sizeof(TpBlob); }

ffb_status ffb_tp_export(ffb_model* m, void* blob) {
    if (!m || !blob) return fail(FFB_USAGE, "NULL argument");
    CUDA_TRY(cudaSetDevice(m->device));
    TpBlob b{};
    b.magic = 0xFFB200u;
    b.rank = static_cast<uint32_t>(m->tp_rank);
    b.tp = static_cast<uint32_t>(m->tp_size);
    b.device = static_cast<uint32_t>(m->device);
    b.pid = static_cast<uint64_t>(getpid());
    b.xch_ptr = reinterpret_cast<uint64_t>(m->xch);
    b.xflag_ptr = reinterpret_cast<uint64_t>(m->xflag);
    // IPC handles (multi-process ranks); may fail in restricted sandboxes,
    // in which case only same-process peers can connect
    if (cudaIpcGetMemHandle(&b.xch_ipc, m->xch) != cudaSuccess ||
        cudaIpcGetMemHandle(&b.xflag_ipc, m->xflag) != cudaSuccess)
        cudaGetLastError();
    std::memcpy(blob, &b, sizeof(b));
    return FFB_OK;
}

ffb_status ffb_tp_connect(ffb_model* m, const void* blobs, int32_t n) {
    if (!m || !blobs) return fail(FFB_USAGE, "NULL argument");
    if (n != m->tp_size) return fail(FFB_USAGE, "tp_connect: expected %d blobs", m->tp_size);
    CUDA_TRY(cudaSetDevice(m->device));
    const auto* bl = static_cast<const TpBlob*>(blobs);
    for (int i = 0; i < n; ++i) {
        const TpBlob& b = bl[i];
        if (b.magic != 0xFFB200u || (int)b.tp != m->tp_size || (int)b.rank != i)
            return fail(FFB_USAGE, "tp_connect: blob %d is not rank %d of %d", i, i, m->tp_size);
        if (i == m->tp_rank) continue;
        if (b.pid == static_cast<uint64_t>(getpid())) {  // same process: one address space
            if ((int)b.device != m->device) {
                cudaError_t e = cudaDeviceEnablePeerAccess(static_cast<int>(b.device), 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return fail(FFB_DEVICE, "peer access to device %u: %s", b.device,
                                cudaGetErrorString(e));
                cudaGetLastError();
            }
            m->peer_xch[i] = reinterpret_cast<float*>(b.xch_ptr);
            m->peer_xflag[i] = reinterpret_cast<uint32_t*>(b.xflag_ptr);
        } else {
            void *px = nullptr, *pf = nullptr;
            CUDA_TRY(cudaIpcOpenMemHandle(&px, b.xch_ipc, cudaIpcMemLazyEnablePeerAccess));
            m->ipc_opened.push_back(px);
            CUDA_TRY(cudaIpcOpenMemHandle(&pf, b.xflag_ipc, cudaIpcMemLazyEnablePeerAccess));
            m->ipc_opened.push_back(pf);
            m->peer_xch[i] = static_cast<float*>(px);
            m->peer_xflag[i] = static_cast<uint32_t*>(pf);
        }
    }
    m->tp_connected = true;
    return FFB_OK;
}

ffb_status ffb_nccl_unique_id(uint8_t id[128]) {
    if (!id) return fail(FFB_USAGE, "NULL argument");
    const auto* nc = nccl_api();
    if (!nc) return fail(FFB_USAGE, "NCCL not available (dlopen libnccl.so.2 failed)");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId");
    ncclUniqueId u;
    NCCL_TRY(nc->get_unique_id(&u));
    std::memcpy(id, &u, 128);
    return FFB_OK;
}

ffb_status ffb_tp_nccl_init(ffb_model* m, const uint8_t id[128]) {
    if (!m || !id) return fail(FFB_USAGE, "NULL argument");
    if (m->tp_size < 2) return fail(FFB_USAGE, "tp_nccl_init: tensor-parallel ranks only");
    const auto* nc = nccl_api();
    if (!nc) return fail(FFB_USAGE, "NCCL not available (dlopen libnccl.so.2 failed)");
    CUDA_TRY(cudaSetDevice(m->device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclComm_t comm = nullptr;
    NCCL_TRY(nc->comm_init_rank(&comm, m->tp_size, u, m->tp_rank));
    if (m->nccl_comm) nc->comm_destroy(static_cast<ncclComm_t>(m->nccl_comm));
    m->nccl_comm = comm;
    m->nccl_destroy = [](void* c) {
        if (const auto* a = nccl_api()) a->comm_destroy(static_cast<ncclComm_t>(c));
    };
    return FFB_OK;
}

int64_t ffb_get_plan_weights(const ffb_model* m, double* out, int64_t n) {
    if (!m) return -1;
    const int64_t G = m->grid;
    if (out) {
        if (n < G) return -1;
        for (int64_t i = 0; i < G; ++i)
            out[i] = i < (int64_t)m->sm_weight.size() ? m->sm_weight[i] : 1.0;
    }
    return G;
}

}  // extern "C"
