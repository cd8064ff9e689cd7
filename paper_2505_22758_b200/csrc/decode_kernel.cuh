// decode_kernel.cuh -- ONE persistent sm_100a kernel for a whole Llama decode
// step (FlashFormer, arxiv 2505.22758), specialised at compile time on the
// model shape.
//
// Reference being replaced: fusesim::execute_program / Interpreter
// (/root/reference/proj/include/fusesim/interpreter.hpp:53-506), i.e. the
// static per-CTA schedule of partition.hpp:266-343 + emit.hpp:214-304 run on
// real hardware.  The math per sublayer follows interpreter.hpp (f32
// accumulation, bf16 weights, bf16 KV cache) and reference.hpp:37-139.
//
// Structure (one CTA per SM, cooperative launch):
//   * warp NCW (the last warp) is the producer: one elected lane walks the
//     same static schedule as the consumers and streams every weight row and
//     every past KV position this CTA needs through an NSLOTS-deep shared
//     memory ring with 1-D TMA bulk copies (cp.async.bulk, L2 evict_first),
//     gated by full/empty mbarriers.  In FusedOverlap mode it never waits at
//     sublayer or layer boundaries (emit.hpp:229-259 "cross" rule): only ring
//     slots gate it.
//   * warps 0..NCW-1 are consumers: column-split GEMV (each thread keeps its
//     slice of the normalised activation vector in registers), warp-shuffle +
//     one named barrier per slot for the row reduction, fused epilogues
//     (RoPE + KV append, residual add, SwiGLU, logits + argmax).
//   * cross-SM dependencies use monotone per-(layer, stage) epoch counters in
//     global memory (release-add / acquire-spin) instead of kernel boundaries.
//
// Per layer the stages are (each ends in a counter arrival; the next waits):
//   S_QKV    RMSNorm(x) -> Wqkv rows -> RoPE -> q (f32), K/V append (bf16)
//   S_ATTN   split-K flash-decoding over KV positions; the last CTA of each
//            (batch row, kv head) group combines the partials (3-stage
//            reduction of numerics.hpp:123-145) -> attn_out
//   S_AOUT   x[rows] += Waout[rows] . attn_out   (row-owned, no atomics)
//   S_GLU    RMSNorm(x) -> paired Wffn1 rows -> h = silu(g)*a -> AXPY with
//            the matching Wffn2^T rows into a per-CTA d_model accumulator
//             -> written as a partial
//   S_RED    x[cols] += sum over CTAs of the GLU partials (fixed order)
// and a tail S_LMHEAD: RMSNorm -> lm_head rows -> logits + fused argmax.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace ffb200 {

enum : int { S_QKV = 0, S_ATTN = 1, S_AOUT = 2, S_GLU = 3, S_RED = 4, kStagesPerLayer = 5 };

// Static per-CTA work ranges, built on the host (runtime.cu: build_cta_plan).
struct CtaPlan {
    int32_t qkv_r0, qkv_r1;    // rows of Wqkv (pair aligned for RoPE)
    int32_t aout_r0, aout_r1;  // rows of Waout
    int32_t glu_t0, glu_t1;    // GLU pair indices: rows 2t,2t+1 of Wffn1, row t of Wffn2^T
    int32_t lm_r0, lm_r1;      // rows of lm_head
    int32_t red_c0, red_c1;    // residual columns this CTA reduces / initialises
    int32_t attn_unit;         // b * NKV + kv_head, or -1 when idle in S_ATTN
    int32_t attn_g;            // slot of this CTA inside its unit's split-K group
    int32_t pad[4];
};

struct DecodeParams {
    // weights, bf16 row-major [out][in] exactly as the reference's Matrix
    const __nv_bfloat16* wqkv;    // [L][QKVR][D]
    const __nv_bfloat16* waout;   // [L][D][D]
    const __nv_bfloat16* wffn1;   // [L][2*DI][D]   rows interleaved in/gate
    const __nv_bfloat16* wffn2t;  // [L][DI][D]     W2 stored transposed
    const float* norm_attn;       // [L][D]  f32 gains (not rounded, tensor_store.hpp:293)
    const float* norm_ffn;        // [L][D]
    const float* final_norm;      // [D]
    const __nv_bfloat16* embedding;  // [V][D]
    const __nv_bfloat16* lm_head;    // [V][D]
    __nv_bfloat16* kcache;        // [L][B][NKV][S][DH] position-major per (l, b, head)
    __nv_bfloat16* vcache;
    // activations / scratch (f32)
    float* x;          // [B][D] residual stream
    float* q;          // [B][NQ*DH] rotated queries
    float* attn_out;   // [B][NQ*DH]
    float* glu_part;   // [grid][RG][B][D]
    float* attn_part;  // [units][grid][QPG][DH+2]  (m, l, o[DH])
    float* logits;     // [B][V]
    float* amax_val;   // [grid][B]
    int32_t* amax_idx; // [grid][B]
    int64_t* greedy;   // [B]
    uint32_t* counters;       // [L*5 + 1] stage counters
    uint32_t* head_counters;  // [L][units]
    uint32_t* amax_counter;   // [1]
    const CtaPlan* plan;      // [grid]
    const int64_t* tokens;    // [B]
    int64_t max_seq;
    int32_t layers, vocab, pos;
    uint32_t epoch;
    int32_t stage_begin, stage_end;
    int32_t overlap;     // 1 = FusedOverlap, 0 = Fused (producer waits at barriers)
    int32_t attn_group;  // G: CTAs per (batch row, kv head)
    int32_t n_units;     // B * NKV
    float eps;
    double rope_theta;
};

template <int D_, int DI_, int DH_, int NQ_, int NKV_, int B_>
struct Shape {
    static constexpr int D = D_, DI = DI_, DH = DH_, NQ = NQ_, NKV = NKV_, B = B_;
    static constexpr int QPG = NQ / NKV;
    static constexpr int QKVR = (NQ + 2 * NKV) * DH;
    static_assert(D == NQ * DH, "d_model must equal n_q_heads * d_head");
    static_assert(NQ % NKV == 0, "GQA grouping");
};

template <class S>
struct KTraits {
    static constexpr int NCW = 8;                   // consumer warps
    static constexpr int NCT = NCW * 32;            // consumer threads
    static constexpr int NTHREADS = NCT + 32;       // + producer warp
    static constexpr int SLOT_BYTES = 32768;
    // GEMV mapping: a row of D bf16 = NV 16-byte vectors split over TPR threads
    static constexpr int NV = S::D / 8;
    static constexpr int TPR = NV < NCT ? NV : NCT;
    static constexpr int VPT = NV / TPR;            // vectors per thread per row
    static constexpr int RG = NCT / TPR;            // row groups working in parallel
    static constexpr int WPR = TPR / 32;            // warps per row
    static constexpr int ROW_BYTES = S::D * 2;
    static constexpr int RPS = SLOT_BYTES / ROW_BYTES;  // rows per slot
    static constexpr int RPT = RPS / RG;            // rows per thread per slot
    static constexpr int KVC = SLOT_BYTES / (2 * S::DH * 2);  // KV positions per slot
    static constexpr int DPL = S::DH / 32;          // attention dims per lane
    static constexpr int TMAX = 160;                // max GLU pairs per CTA (host-checked)
    static_assert(TPR % 32 == 0, "a row must span whole warps");
    static_assert(NV % TPR == 0 && NCT % TPR == 0, "row mapping");
    static_assert(RPS >= 2 && RPS % 2 == 0 && RPS % RG == 0, "slot rows");
    static_assert(RPS * S::B <= NCT, "epilogue threads");
    static_assert(S::DH % 32 == 0 && DPL <= 8, "attention lane split");
    static_assert(KVC >= 1, "kv chunk");

    // ---- shared memory carve-up (bytes) ----
    static constexpr int OFF_RED = 0;  // [2][WPR][RPS][B] f32
    static constexpr int SZ_RED = 2 * WPR * RPS * S::B * 4;
    static constexpr int OFF_H = OFF_RED + SZ_RED;  // [B][TMAX] f32
    static constexpr int SZ_H = S::B * TMAX * 4;
    static constexpr int OFF_ROPE = OFF_H + SZ_H;  // [DH/2][2] f32
    static constexpr int SZ_ROPE = S::DH * 4;
    static constexpr int OFF_NORM = OFF_ROPE + SZ_ROPE;  // [NCW][B] f32
    static constexpr int SZ_NORM = NCW * S::B * 4 + 16;
    static constexpr int OFF_WPART = OFF_NORM + SZ_NORM;  // [NCW][QPG][DH+2] f32
    static constexpr int SZ_WPART = NCW * S::QPG * (S::DH + 2) * 4;
    static constexpr int OFF_AMAX = OFF_WPART + SZ_WPART;  // [NCT] (f32, i32)
    static constexpr int SZ_AMAX = NCT * 8;
    static constexpr int OFF_MISC = OFF_AMAX + SZ_AMAX;  // flags
    static constexpr int SZ_MISC = 64;
    static constexpr int FIXED = ((OFF_MISC + SZ_MISC + 1023) / 1024) * 1024;
    static constexpr int MAX_SMEM = 227 * 1024;
    static constexpr int NSLOTS_RAW = (MAX_SMEM - FIXED - 256) / SLOT_BYTES;
    static constexpr int NSLOTS = NSLOTS_RAW > 8 ? 8 : NSLOTS_RAW;
    static_assert(NSLOTS >= 2, "ring too small");
    static constexpr int OFF_BARS = FIXED;  // full[NSLOTS], empty[NSLOTS]
    static constexpr int OFF_RING = FIXED + 256;
    static constexpr int SMEM_BYTES = OFF_RING + NSLOTS * SLOT_BYTES;
    static_assert(SMEM_BYTES <= MAX_SMEM, "shared memory budget");
};

// ============================================================================
template <class S>
struct DecodeCta {
    using T = KTraits<S>;
    static constexpr int B = S::B, D = S::D, DH = S::DH, QPG = S::QPG, NCT = T::NCT,
                         NCW = T::NCW;

    const DecodeParams& p;
    uint8_t* smem;
    uint64_t* full;
    uint64_t* empty;
    uint8_t* ring;
    CtaPlan pl;
    int cta, grid;

    __device__ DecodeCta(const DecodeParams& p_, uint8_t* smem_) : p(p_), smem(smem_) {
        full = reinterpret_cast<uint64_t*>(smem + T::OFF_BARS);
        empty = full + T::NSLOTS;
        ring = smem + T::OFF_RING;
        cta = blockIdx.x;
        grid = gridDim.x;
        pl = p.plan[cta];
    }

    __device__ float* red_buf(uint32_t it) {
        return reinterpret_cast<float*>(smem + T::OFF_RED) + (it & 1) * (T::WPR * T::RPS * B);
    }
    __device__ float* h_s() { return reinterpret_cast<float*>(smem + T::OFF_H); }
    __device__ float* rope() { return reinterpret_cast<float*>(smem + T::OFF_ROPE); }
    __device__ float* norm_s() { return reinterpret_cast<float*>(smem + T::OFF_NORM); }
    __device__ float* wpart() { return reinterpret_cast<float*>(smem + T::OFF_WPART); }
    __device__ int* misc() { return reinterpret_cast<int*>(smem + T::OFF_MISC); }

    // ------------------------------------------------------------ schedule
    __device__ int n_stages() const { return p.layers * kStagesPerLayer + 1; }

    // counter a stage's consumers wait on before starting, and its target
    __device__ bool dependency(int stage, const uint32_t** ctr, uint32_t* target) const {
        const int l = stage / kStagesPerLayer, s = stage % kStagesPerLayer;
        const uint32_t full_grid = p.epoch * static_cast<uint32_t>(grid);
        if (stage == p.layers * kStagesPerLayer) {  // LM head
            if (p.layers == 0) return false;
            *ctr = p.counters + (p.layers - 1) * kStagesPerLayer + S_RED;
            *target = full_grid;
            return true;
        }
        switch (s) {
            case S_QKV:
                if (l == 0) return false;
                *ctr = p.counters + (l - 1) * kStagesPerLayer + S_RED;
                *target = full_grid;
                return true;
            case S_ATTN:
                *ctr = p.counters + l * kStagesPerLayer + S_QKV;
                *target = full_grid;
                return true;
            case S_AOUT:
                *ctr = p.counters + l * kStagesPerLayer + S_ATTN;
                *target = p.epoch * static_cast<uint32_t>(p.n_units);
                return true;
            case S_GLU:
                *ctr = p.counters + l * kStagesPerLayer + S_AOUT;
                *target = full_grid;
                return true;
            default:  // S_RED
                *ctr = p.counters + l * kStagesPerLayer + S_GLU;
                *target = full_grid;
                return true;
        }
    }

    // attention position range of this CTA: [p0, p1) out of [0, pos]
    __device__ void attn_range(int& p0, int& p1) const {
        const int ctx = p.pos + 1, G = p.attn_group, g = pl.attn_g;
        p0 = static_cast<int>((static_cast<int64_t>(g) * ctx) / G);
        p1 = static_cast<int>((static_cast<int64_t>(g + 1) * ctx) / G);
    }

    __device__ size_t kv_row(int l, int b, int h, int pos) const {
        return ((((size_t)l * B + b) * S::NKV + h) * (size_t)p.max_seq + pos) * DH;
    }

    // ============================================================ producer
    __device__ void produce_rows(uint32_t& it, const __nv_bfloat16* base, int r0, int r1,
                                 uint64_t policy) {
        for (int c0 = r0; c0 < r1; c0 += T::RPS) {
            const int n = min(T::RPS, r1 - c0);
            const uint32_t slot = it % T::NSLOTS, par = ((it / T::NSLOTS) & 1) ^ 1;
            mbar_wait(&empty[slot], par);
            const uint32_t bytes = static_cast<uint32_t>(n) * T::ROW_BYTES;
            mbar_arrive_expect_tx(&full[slot], bytes);
            tma_load_1d(ring + slot * T::SLOT_BYTES, base + (size_t)c0 * D, bytes, &full[slot],
                        policy);
            ++it;
        }
    }

    __device__ void produce_kv(uint32_t& it, int l, int q0, int q1, uint64_t policy) {
        const int unit = pl.attn_unit, b = unit / S::NKV, h = unit % S::NKV;
        for (int c0 = q0; c0 < q1; c0 += T::KVC) {
            const int n = min(T::KVC, q1 - c0);
            const uint32_t slot = it % T::NSLOTS, par = ((it / T::NSLOTS) & 1) ^ 1;
            mbar_wait(&empty[slot], par);
            const uint32_t bytes = static_cast<uint32_t>(n) * DH * 2;
            mbar_arrive_expect_tx(&full[slot], 2 * bytes);
            uint8_t* dst = ring + slot * T::SLOT_BYTES;
            const size_t row = kv_row(l, b, h, c0);
            tma_load_1d(dst, p.kcache + row, bytes, &full[slot], policy);
            tma_load_1d(dst + T::SLOT_BYTES / 2, p.vcache + row, bytes, &full[slot], policy);
            ++it;
        }
    }

    __device__ void producer() {
        const uint64_t policy = policy_evict_first();
        uint32_t it = 0;
        const int last = min(p.stage_end, n_stages());
        for (int stage = p.stage_begin; stage < last; ++stage) {
            if (!p.overlap && stage != p.stage_begin) {
                const uint32_t* ctr;
                uint32_t target;
                if (dependency(stage, &ctr, &target)) spin_until_geq(ctr, target);
            }
            const int l = stage / kStagesPerLayer, s = stage % kStagesPerLayer;
            if (stage == p.layers * kStagesPerLayer) {
                produce_rows(it, p.lm_head, pl.lm_r0, pl.lm_r1, policy);
                continue;
            }
            switch (s) {
                case S_QKV:
                    produce_rows(it, p.wqkv + (size_t)l * S::QKVR * D, pl.qkv_r0, pl.qkv_r1,
                                 policy);
                    break;
                case S_ATTN:
                    if (pl.attn_unit >= 0) {
                        int p0, p1;
                        attn_range(p0, p1);
                        produce_kv(it, l, p0, min(p1, p.pos), policy);
                    }
                    break;
                case S_AOUT:
                    produce_rows(it, p.waout + (size_t)l * D * D, pl.aout_r0, pl.aout_r1, policy);
                    break;
                case S_GLU:
                    produce_rows(it, p.wffn1 + (size_t)l * 2 * S::DI * D, 2 * pl.glu_t0,
                                 2 * pl.glu_t1, policy);
                    produce_rows(it, p.wffn2t + (size_t)l * S::DI * D, pl.glu_t0, pl.glu_t1,
                                 policy);
                    break;
                default:
                    break;
            }
        }
    }

    // ============================================================ consumers
    __device__ static float warp_sum(float v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    }

    __device__ void wait_stage(int stage) {
        const uint32_t* ctr;
        uint32_t target;
        if (dependency(stage, &ctr, &target)) {
            if (threadIdx.x == 0) spin_until_geq(ctr, target);
            consumer_sync(NCT);
        }
    }

    __device__ void arrive(uint32_t* ctr) {
        consumer_sync(NCT);
        if (threadIdx.x == 0) {
            __threadfence();
            red_release_gpu(ctr, 1);
        }
    }

    // Load this thread's activation slice: act[b][j][e] = column (lt + j*TPR)*8 + e.
    // src_emb: layer-0 input taken straight from the embedding (bf16 row per b).
    // gain != nullptr -> RMSNorm with that f32 gain (numerics.hpp:14-24).
    __device__ void load_act(float (&act)[B][T::VPT][8], const float* src, bool from_emb,
                             const float* gain) {
        const int ctid = threadIdx.x, lt = ctid % T::TPR, rg = ctid / T::TPR;
#pragma unroll
        for (int b = 0; b < B; ++b) {
#pragma unroll
            for (int j = 0; j < T::VPT; ++j) {
                const int col = (lt + j * T::TPR) * 8;
                if (from_emb) {
                    const __nv_bfloat16* e = p.embedding + (size_t)p.tokens[b] * D + col;
                    const uint4 w = __ldg(reinterpret_cast<const uint4*>(e));
                    act[b][j][0] = bf_lo(w.x); act[b][j][1] = bf_hi(w.x);
                    act[b][j][2] = bf_lo(w.y); act[b][j][3] = bf_hi(w.y);
                    act[b][j][4] = bf_lo(w.z); act[b][j][5] = bf_hi(w.z);
                    act[b][j][6] = bf_lo(w.w); act[b][j][7] = bf_hi(w.w);
                } else {
                    const float4 a0 = ldcg_f4(src + (size_t)b * D + col);
                    const float4 a1 = ldcg_f4(src + (size_t)b * D + col + 4);
                    act[b][j][0] = a0.x; act[b][j][1] = a0.y; act[b][j][2] = a0.z;
                    act[b][j][3] = a0.w; act[b][j][4] = a1.x; act[b][j][5] = a1.y;
                    act[b][j][6] = a1.z; act[b][j][7] = a1.w;
                }
            }
        }
        if (gain == nullptr) return;
        float ss[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            float s = 0.f;
            if (rg == 0) {
#pragma unroll
                for (int j = 0; j < T::VPT; ++j)
#pragma unroll
                    for (int e = 0; e < 8; ++e) s = fmaf(act[b][j][e], act[b][j][e], s);
            }
            ss[b] = warp_sum(s);
        }
        float* ns = norm_s();
        const int warp = ctid / 32, lane = ctid % 32;
        if (lane == 0)
#pragma unroll
            for (int b = 0; b < B; ++b) ns[warp * B + b] = ss[b];
        consumer_sync(NCT);
        float inv[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            float t = 0.f;
            for (int w = 0; w < NCW; ++w) t += ns[w * B + b];
            inv[b] = 1.0f / sqrtf(t / static_cast<float>(D) + p.eps);
        }
        consumer_sync(NCT);  // ns reusable afterwards
#pragma unroll
        for (int j = 0; j < T::VPT; ++j) {
            const int col = (lt + j * T::TPR) * 8;
            const float4 g0 = __ldg(reinterpret_cast<const float4*>(gain + col));
            const float4 g1 = __ldg(reinterpret_cast<const float4*>(gain + col + 4));
            const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
                for (int e = 0; e < 8; ++e) act[b][j][e] = g[e] * act[b][j][e] * inv[b];
        }
    }

    __device__ static float dot8(const uint4 w, const float (&a)[8], float acc) {
        acc = fmaf(bf_lo(w.x), a[0], acc);
        acc = fmaf(bf_hi(w.x), a[1], acc);
        acc = fmaf(bf_lo(w.y), a[2], acc);
        acc = fmaf(bf_hi(w.y), a[3], acc);
        acc = fmaf(bf_lo(w.z), a[4], acc);
        acc = fmaf(bf_hi(w.z), a[5], acc);
        acc = fmaf(bf_lo(w.w), a[6], acc);
        acc = fmaf(bf_hi(w.w), a[7], acc);
        return acc;
    }

    // GEMV over rows [r0, r1) streamed by the producer.  For every slot the
    // row sums land in red_buf(it)[wr][row][b] and `epi(c0, nrows, red)` runs
    // after the named barrier.
    template <class Epi>
    __device__ void gemv(uint32_t& it, const float (&act)[B][T::VPT][8], int r0, int r1,
                         Epi&& epi) {
        const int ctid = threadIdx.x, lane = ctid % 32;
        const int rg = ctid / T::TPR, lt = ctid % T::TPR, wr = lt / 32;
        for (int c0 = r0; c0 < r1; c0 += T::RPS) {
            const int nrows = min(T::RPS, r1 - c0);
            const uint32_t slot = it % T::NSLOTS, par = (it / T::NSLOTS) & 1;
            mbar_wait(&full[slot], par);
            const uint8_t* base = ring + slot * T::SLOT_BYTES;
            float part[T::RPT][B];
#pragma unroll
            for (int r = 0; r < T::RPT; ++r) {
#pragma unroll
                for (int b = 0; b < B; ++b) part[r][b] = 0.f;
                const int row = rg + r * T::RG;
                if (row < nrows) {
#pragma unroll
                    for (int j = 0; j < T::VPT; ++j) {
                        const uint4 w = lds_u128(base + row * T::ROW_BYTES + (lt + j * T::TPR) * 16);
#pragma unroll
                        for (int b = 0; b < B; ++b) part[r][b] = dot8(w, act[b][j], part[r][b]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            float* red = red_buf(it);
#pragma unroll
            for (int r = 0; r < T::RPT; ++r) {
                const int row = rg + r * T::RG;
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const float v = warp_sum(part[r][b]);
                    if (lane == 0 && row < nrows) red[(wr * T::RPS + row) * B + b] = v;
                }
            }
            consumer_sync(NCT);
            epi(c0, nrows, red);
            ++it;
        }
    }

    __device__ static float row_total(const float* red, int row, int b) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < T::WPR; ++w) t += red[(w * T::RPS + row) * B + b];
        return t;
    }

    // ---------------------------------------------------------- S_QKV
    __device__ void stage_qkv(uint32_t& it, int l) {
        float act[B][T::VPT][8];
        load_act(act, p.x, l == 0, p.norm_attn + (size_t)l * D);
        const float* rp = rope();
        const int ctid = threadIdx.x;
        gemv(it, act, pl.qkv_r0, pl.qkv_r1, [&](int c0, int nrows, const float* red) {
            const int npairs = nrows / 2;
            if (ctid < npairs * B) {
                const int pr = ctid / B, b = ctid % B;
                const int g = c0 + 2 * pr;  // global even row
                const float a = row_total(red, 2 * pr, b), bb = row_total(red, 2 * pr + 1, b);
                constexpr int QR = S::NQ * DH, KR = S::NKV * DH;
                if (g < QR + KR) {  // rotary pair (interleaved, numerics.hpp:27-37)
                    const int dim = g % DH, k = dim / 2;
                    const float c = rp[2 * k], s = rp[2 * k + 1];
                    const float r0 = a * c - bb * s, r1 = a * s + bb * c;
                    if (g < QR) {
                        float* q = p.q + (size_t)b * QR + g;
                        __stcg(q, r0);
                        __stcg(q + 1, r1);
                    } else {
                        const int h = (g - QR) / DH;
                        __nv_bfloat16* k_dst = p.kcache + kv_row(l, b, h, p.pos) + dim;
                        __nv_bfloat162 kv2;
                        kv2.x = __float2bfloat16_rn(r0);
                        kv2.y = __float2bfloat16_rn(r1);
                        *reinterpret_cast<__nv_bfloat162*>(k_dst) = kv2;
                    }
                } else {
                    const int gv = g - QR - KR, h = gv / DH, dim = gv % DH;
                    __nv_bfloat16* v_dst = p.vcache + kv_row(l, b, h, p.pos) + dim;
                    __nv_bfloat162 kv2;
                    kv2.x = __float2bfloat16_rn(a);
                    kv2.y = __float2bfloat16_rn(bb);
                    *reinterpret_cast<__nv_bfloat162*>(v_dst) = kv2;
                }
            }
        });
        arrive(p.counters + l * kStagesPerLayer + S_QKV);
    }

    // ---------------------------------------------------------- S_ATTN
    // One online-softmax state per warp (m, l replicated in all lanes, o
    // split over lanes by head dim), positions dealt round-robin to warps.
    struct AttnState {
        float m[QPG], l[QPG], o[QPG][T::DPL];
    };

    __device__ void attn_update(AttnState& st, const float (&q)[QPG][T::DPL], const float* kf,
                                const float* vf, float alpha) {
        float dot[QPG];
#pragma unroll
        for (int h = 0; h < QPG; ++h) {
            float s = 0.f;
#pragma unroll
            for (int e = 0; e < T::DPL; ++e) s = fmaf(q[h][e], kf[e], s);
            dot[h] = warp_sum(s);
        }
#pragma unroll
        for (int h = 0; h < QPG; ++h) {
            const float s = alpha * dot[h];
            const float m_new = fmaxf(st.m[h], s);
            const float scale = expf(st.m[h] - m_new);
            const float w = expf(s - m_new);
            st.l[h] = st.l[h] * scale + w;
#pragma unroll
            for (int e = 0; e < T::DPL; ++e) st.o[h][e] = st.o[h][e] * scale + w * vf[e];
            st.m[h] = m_new;
        }
    }

    __device__ static void unpack_bf16(const uint32_t* w, float* f, int n) {
        for (int i = 0; i < n / 2; ++i) {
            f[2 * i] = bf_lo(w[i]);
            f[2 * i + 1] = bf_hi(w[i]);
        }
    }

    __device__ void stage_attn(uint32_t& it, int l) {
        if (pl.attn_unit < 0) return;  // idle CTA: no chunks were streamed
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32;
        const int unit = pl.attn_unit, b = unit / S::NKV, kvh = unit % S::NKV;
        const float alpha = 1.0f / sqrtf(static_cast<float>(DH));
        int p0, p1;
        attn_range(p0, p1);
        const int past_end = min(p1, p.pos);

        float q[QPG][T::DPL];
#pragma unroll
        for (int h = 0; h < QPG; ++h)
#pragma unroll
            for (int e = 0; e < T::DPL; ++e)
                q[h][e] = ldcg_f(p.q + (size_t)b * D + (kvh * QPG + h) * DH + lane * T::DPL + e);
        AttnState st;
#pragma unroll
        for (int h = 0; h < QPG; ++h) {
            st.m[h] = -INFINITY;
            st.l[h] = 0.f;
#pragma unroll
            for (int e = 0; e < T::DPL; ++e) st.o[h][e] = 0.f;
        }

        for (int c0 = p0; c0 < past_end; c0 += T::KVC) {
            const int n = min(T::KVC, past_end - c0);
            const uint32_t slot = it % T::NSLOTS, par = (it / T::NSLOTS) & 1;
            mbar_wait(&full[slot], par);
            const uint8_t* kb = ring + slot * T::SLOT_BYTES;
            const uint8_t* vb = kb + T::SLOT_BYTES / 2;
            for (int j = warp; j < n; j += NCW) {
                uint32_t kw[T::DPL / 2], vw[T::DPL / 2];
                const uint8_t* kp = kb + (size_t)j * DH * 2 + lane * T::DPL * 2;
                const uint8_t* vp = vb + (size_t)j * DH * 2 + lane * T::DPL * 2;
#pragma unroll
                for (int i = 0; i < T::DPL / 2; ++i) {
                    kw[i] = lds_u32(kp + 4 * i);
                    vw[i] = lds_u32(vp + 4 * i);
                }
                float kf[T::DPL], vf[T::DPL];
                unpack_bf16(kw, kf, T::DPL);
                unpack_bf16(vw, vf, T::DPL);
                attn_update(st, q, kf, vf, alpha);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            ++it;
        }
        // current token: written by this launch's S_QKV with generic stores,
        // read back at L2 (emit.hpp:148-154 SyncLoadCurrentToken)
        if (p.pos >= p0 && p.pos < p1 && warp == (p.pos - p0) % NCW) {
            const size_t row = kv_row(l, b, kvh, p.pos) + lane * T::DPL;
            uint32_t kw[T::DPL / 2], vw[T::DPL / 2];
#pragma unroll
            for (int i = 0; i < T::DPL / 2; ++i) {
                kw[i] = __ldcg(reinterpret_cast<const unsigned int*>(p.kcache + row) + i);
                vw[i] = __ldcg(reinterpret_cast<const unsigned int*>(p.vcache + row) + i);
            }
            float kf[T::DPL], vf[T::DPL];
            unpack_bf16(kw, kf, T::DPL);
            unpack_bf16(vw, vf, T::DPL);
            attn_update(st, q, kf, vf, alpha);
        }

        // combine the NCW warp states into this CTA's partial (m, l, o)
        float* wp = wpart();
        constexpr int STR = DH + 2;
#pragma unroll
        for (int h = 0; h < QPG; ++h) {
            float* dst = wp + (warp * QPG + h) * STR;
            if (lane == 0) {
                dst[0] = st.m[h];
                dst[1] = st.l[h];
            }
#pragma unroll
            for (int e = 0; e < T::DPL; ++e) dst[2 + lane * T::DPL + e] = st.o[h][e];
        }
        consumer_sync(NCT);
        float* part = p.attn_part + ((size_t)unit * grid + pl.attn_g) * QPG * STR;
        for (int idx = ctid; idx < QPG * DH; idx += NCT) {
            const int h = idx / DH, d = idx % DH;
            float M = -INFINITY;
            for (int w = 0; w < NCW; ++w) {
                const float* s = wp + (w * QPG + h) * STR;
                if (s[1] > 0.f) M = fmaxf(M, s[0]);
            }
            float L = 0.f, O = 0.f;
            for (int w = 0; w < NCW; ++w) {
                const float* s = wp + (w * QPG + h) * STR;
                if (s[1] > 0.f) {
                    const float r = expf(s[0] - M);
                    L += s[1] * r;
                    O += s[2 + d] * r;
                }
            }
            float* dst = part + h * STR;
            __stcg(dst + 2 + d, O);
            if (d == 0) {
                __stcg(dst, M);
                __stcg(dst + 1, L);
            }
        }
        // last arriver of the group combines (numerics.hpp:123-145)
        consumer_sync(NCT);
        int* flag = misc();
        if (ctid == 0) {
            __threadfence();
            const uint32_t old =
                atom_add_acq_rel_gpu(p.head_counters + (size_t)l * p.n_units + unit, 1);
            flag[0] = (old + 1 == p.epoch * static_cast<uint32_t>(p.attn_group)) ? 1 : 0;
            __threadfence();
        }
        consumer_sync(NCT);
        if (flag[0]) {
            const float* base = p.attn_part + (size_t)unit * grid * QPG * STR;
            for (int idx = ctid; idx < QPG * DH; idx += NCT) {
                const int h = idx / DH, d = idx % DH;
                float M = -INFINITY;
                for (int g = 0; g < p.attn_group; ++g) {
                    const float* s = base + ((size_t)g * QPG + h) * STR;
                    if (ldcg_f(s + 1) > 0.f) M = fmaxf(M, ldcg_f(s));
                }
                float L = 0.f;
                for (int g = 0; g < p.attn_group; ++g) {
                    const float* s = base + ((size_t)g * QPG + h) * STR;
                    const float lg = ldcg_f(s + 1);
                    if (lg > 0.f) L += lg * expf(ldcg_f(s) - M);
                }
                float out = 0.f;
                for (int g = 0; g < p.attn_group; ++g) {
                    const float* s = base + ((size_t)g * QPG + h) * STR;
                    const float lg = ldcg_f(s + 1);
                    if (lg > 0.f) out += (expf(ldcg_f(s) - M) / L) * ldcg_f(s + 2 + d);
                }
                __stcg(p.attn_out + (size_t)b * D + (kvh * QPG + h) * DH + d, out);
            }
            arrive(p.counters + l * kStagesPerLayer + S_ATTN);
        }
    }

    // ---------------------------------------------------------- S_AOUT
    __device__ void stage_aout(uint32_t& it, int l) {
        float act[B][T::VPT][8];
        load_act(act, p.attn_out, false, nullptr);
        const int ctid = threadIdx.x;
        gemv(it, act, pl.aout_r0, pl.aout_r1, [&](int c0, int nrows, const float* red) {
            if (ctid < nrows * B) {
                const int r = ctid / B, b = ctid % B;
                float* xp = p.x + (size_t)b * D + c0 + r;
                __stcg(xp, ldcg_f(xp) + row_total(red, r, b));
            }
        });
        arrive(p.counters + l * kStagesPerLayer + S_AOUT);
    }

    // ---------------------------------------------------------- S_GLU
    __device__ void stage_glu(uint32_t& it, int l) {
        const int ctid = threadIdx.x;
        const int t0 = pl.glu_t0, t1 = pl.glu_t1;
        float* hs = h_s();
        {
            float act[B][T::VPT][8];
            load_act(act, p.x, false, p.norm_ffn + (size_t)l * D);
            gemv(it, act, 2 * t0, 2 * t1, [&](int c0, int nrows, const float* red) {
                const int npairs = nrows / 2;
                if (ctid < npairs * B) {
                    const int pr = ctid / B, b = ctid % B;
                    const float a = row_total(red, 2 * pr, b), g = row_total(red, 2 * pr + 1, b);
                    const float silu = g / (1.0f + expf(-g));
                    hs[b * T::TMAX + (c0 / 2 - t0) + pr] = silu * a;
                }
            });
        }
        consumer_sync(NCT);  // h complete
        const int rg = ctid / T::TPR, lt = ctid % T::TPR, lane = ctid % 32;
        float acc[B][T::VPT][8];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int j = 0; j < T::VPT; ++j)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[b][j][e] = 0.f;
        for (int c0 = t0; c0 < t1; c0 += T::RPS) {
            const int nrows = min(T::RPS, t1 - c0);
            const uint32_t slot = it % T::NSLOTS, par = (it / T::NSLOTS) & 1;
            mbar_wait(&full[slot], par);
            const uint8_t* base = ring + slot * T::SLOT_BYTES;
#pragma unroll
            for (int r = 0; r < T::RPT; ++r) {
                const int row = rg + r * T::RG;
                if (row < nrows) {
                    float hb[B];
#pragma unroll
                    for (int b = 0; b < B; ++b) hb[b] = hs[b * T::TMAX + (c0 - t0) + row];
#pragma unroll
                    for (int j = 0; j < T::VPT; ++j) {
                        const uint4 w = lds_u128(base + row * T::ROW_BYTES + (lt + j * T::TPR) * 16);
                        const float wf[8] = {bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y),
                                             bf_lo(w.z), bf_hi(w.z), bf_lo(w.w), bf_hi(w.w)};
#pragma unroll
                        for (int b = 0; b < B; ++b)
#pragma unroll
                            for (int e = 0; e < 8; ++e) acc[b][j][e] = fmaf(hb[b], wf[e], acc[b][j][e]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            ++it;
        }
        // per-(CTA, row group) partial d_model vectors
        float* gp = p.glu_part + ((size_t)cta * T::RG + rg) * B * D;
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int j = 0; j < T::VPT; ++j) {
                const int col = (lt + j * T::TPR) * 8;
                float* dst = gp + (size_t)b * D + col;
                __stcg(reinterpret_cast<float4*>(dst),
                       make_float4(acc[b][j][0], acc[b][j][1], acc[b][j][2], acc[b][j][3]));
                __stcg(reinterpret_cast<float4*>(dst + 4),
                       make_float4(acc[b][j][4], acc[b][j][5], acc[b][j][6], acc[b][j][7]));
            }
        arrive(p.counters + l * kStagesPerLayer + S_GLU);
    }

    // ---------------------------------------------------------- S_RED
    __device__ void stage_red(int l) {
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32;
        const int c0 = pl.red_c0, c1 = pl.red_c1;
        const int nparts = grid * T::RG;
        float* ns = norm_s();  // [NCW][32] scratch reuse would overflow; use wpart
        float* scratch = wpart();
        for (int b = 0; b < B; ++b) {
            for (int cb = c0; cb < c1; cb += 32) {
                const int col = cb + lane;
                float s = 0.f;
                if (col < c1)
                    for (int q = warp; q < nparts; q += NCW)
                        s += ldcg_f(p.glu_part + ((size_t)q * B + b) * D + col);
                scratch[warp * 32 + lane] = s;
                consumer_sync(NCT);
                if (warp == 0 && col < c1) {
                    float t = 0.f;
                    for (int w = 0; w < NCW; ++w) t += scratch[w * 32 + lane];
                    float* xp = p.x + (size_t)b * D + col;
                    __stcg(xp, ldcg_f(xp) + t);
                }
                consumer_sync(NCT);
            }
        }
        (void)ns;
        arrive(p.counters + l * kStagesPerLayer + S_RED);
    }

    // ---------------------------------------------------------- S_LMHEAD
    __device__ void stage_lmhead(uint32_t& it) {
        float act[B][T::VPT][8];
        load_act(act, p.x, p.layers == 0, p.final_norm);
        const int ctid = threadIdx.x;
        float best = -INFINITY;
        int best_i = 0x7fffffff;
        gemv(it, act, pl.lm_r0, pl.lm_r1, [&](int c0, int nrows, const float* red) {
            if (ctid < nrows * B) {
                const int r = ctid / B, b = ctid % B;
                const float v = row_total(red, r, b);
                __stcg(p.logits + (size_t)b * p.vocab + c0 + r, v);
                if (v > best) {
                    best = v;
                    best_i = c0 + r;
                }
            }
        });
        // CTA argmax per batch row (lowest index on ties, numerics.hpp:169-175)
        float* av = reinterpret_cast<float*>(smem + T::OFF_AMAX);
        int* ai = reinterpret_cast<int*>(av + NCT);
        av[ctid] = best;
        ai[ctid] = best_i;
        consumer_sync(NCT);
        if (ctid < B) {
            float bv = -INFINITY;
            int bi = 0x7fffffff;
            for (int t = ctid; t < NCT; t += B) {
                if (av[t] > bv || (av[t] == bv && ai[t] < bi)) {
                    bv = av[t];
                    bi = ai[t];
                }
            }
            __stcg(p.amax_val + (size_t)cta * B + ctid, bv);
            __stcg(p.amax_idx + (size_t)cta * B + ctid, bi);
        }
        consumer_sync(NCT);
        int* flag = misc();
        if (ctid == 0) {
            __threadfence();
            const uint32_t old = atom_add_acq_rel_gpu(p.amax_counter, 1);
            flag[1] = (old + 1 == p.epoch * static_cast<uint32_t>(grid)) ? 1 : 0;
            __threadfence();
        }
        consumer_sync(NCT);
        if (flag[1] && ctid < B) {
            float bv = -INFINITY;
            int bi = 0;
            bool any = false;
            for (int c = 0; c < grid; ++c) {
                const float v = ldcg_f(p.amax_val + (size_t)c * B + ctid);
                const int i = __ldcg(p.amax_idx + (size_t)c * B + ctid);
                if (i == 0x7fffffff) continue;  // CTA without lm_head rows
                if (!any || v > bv || (v == bv && i < bi)) {
                    bv = v;
                    bi = i;
                    any = true;
                }
            }
            p.greedy[ctid] = bi;
        }
    }

    __device__ void consumer() {
        uint32_t it = 0;
        const int last = min(p.stage_end, n_stages());
        for (int stage = p.stage_begin; stage < last; ++stage) {
            wait_stage(stage);  // satisfied immediately after a kernel boundary
            const int l = stage / kStagesPerLayer, s = stage % kStagesPerLayer;
            if (stage == p.layers * kStagesPerLayer) {
                stage_lmhead(it);
                continue;
            }
            switch (s) {
                case S_QKV: stage_qkv(it, l); break;
                case S_ATTN: stage_attn(it, l); break;
                case S_AOUT: stage_aout(it, l); break;
                case S_GLU: stage_glu(it, l); break;
                default: stage_red(l); break;
            }
        }
    }
};

template <class S>
__global__ void __launch_bounds__(KTraits<S>::NTHREADS, 1)
    decode_step_kernel(const __grid_constant__ DecodeParams p) {
    using T = KTraits<S>;
    extern __shared__ __align__(1024) uint8_t smem[];
    DecodeCta<S> cta(p, smem);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int i = 0; i < T::NSLOTS; ++i) {
            mbar_init(&cta.full[i], 1);
            mbar_init(&cta.empty[i], T::NCW);
        }
        fence_mbar_init();
    }
    // RoPE table for this step's position, in f64 (numerics.hpp:27-37 angle)
    if (tid < S::DH / 2) {
        const double freq = pow(p.rope_theta, -static_cast<double>(2 * tid) / S::DH);
        const double ang = static_cast<double>(p.pos) * freq;
        cta.rope()[2 * tid] = static_cast<float>(cos(ang));
        cta.rope()[2 * tid + 1] = static_cast<float>(sin(ang));
    }
    // residual init from the embedding: each CTA owns its reduce columns
    if (p.stage_begin == 0 && tid < T::NCT) {
        for (int b = 0; b < S::B; ++b) {
            const __nv_bfloat16* e = p.embedding + (size_t)p.tokens[b] * S::D;
            for (int c = cta.pl.red_c0 + tid; c < cta.pl.red_c1; c += T::NCT)
                __stcg(p.x + (size_t)b * S::D + c, __bfloat162float(e[c]));
        }
    }
    __syncthreads();
    if (tid >= T::NCT) {
        if (tid == T::NCT) cta.producer();
    } else {
        cta.consumer();
    }
}

}  // namespace ffb200
