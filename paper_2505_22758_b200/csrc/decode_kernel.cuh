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
// (bf16 at batch <= 2, KTraits::F2R: S_GLU stops at h, written to global
// memory, and S_RED is the second GEMV x[rows] += W2[rows] . h.)
// and a tail S_LMHEAD: RMSNorm -> lm_head rows -> logits + fused argmax.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"

namespace ffb200 {

// Debug bits (never set by the public API's production path):
//   kDebugStreamOnly: consumers only wait for / release ring slots (pure TMA
//                     streaming rate of the schedule, no math, no flags)
enum : int { kDebugStreamOnly = 1 };

// per-(CTA, stage) trace record: 0 entry, 1 dependency met, 2 done,
// 3 stage mark, 4 ns starved waiting for ring data, 5-7 spare
constexpr int kTraceSlots = 8;

// most CTAs that split one (batch row, kv head)'s positions (runtime.cu)
constexpr int kMaxGroup = 32;

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
    int32_t qkv_heads;         // bit h: this CTA's Wqkv rows include q/k/v rows of kv head h
    int32_t attn_dep;          // CTAs whose Wqkv rows touch this CTA's kv head (S_ATTN dependency)
    int32_t pad[2];
};

struct DecodeParams {
    // streamed weights, rows [out] of weight_row_bytes(D, QB) bytes each, in
    // the reference's Matrix row order (bf16 or packed int4/int8 rows)
    const uint8_t* wqkv;    // [L][QKVR] rows
    const uint8_t* waout;   // [L][D] rows
    const uint8_t* wffn1;   // [L][2*DI] rows, interleaved in/gate
    const uint8_t* wffn2t;  // [L][DI] rows, W2 stored transposed
    const float* norm_attn;       // [L][D]  f32 gains (not rounded, tensor_store.hpp:293)
    const float* norm_ffn;        // [L][D]
    const float* final_norm;      // [D]
    const __nv_bfloat16* embedding;  // [V][D] bf16 (never quantized)
    const uint8_t* lm_head;          // [V] rows
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
    uint32_t* qkv_head_counters;  // [L][NKV]: arrivals of CTAs holding that head's Wqkv rows
    uint32_t* amax_counter;   // [1]
    const CtaPlan* plan;      // [grid]
    const int64_t* tokens;    // [B]
    uint32_t* err_flag;       // latched bit 0: a device-resident token id was out of range
    int32_t vocab_embed;      // embedding rows (the whole vocabulary, also on a TP shard)
    int64_t max_seq;
    int32_t layers, vocab, pos;
    uint32_t epoch;
    int32_t stage_begin, stage_end;
    int32_t overlap;     // 1 = FusedOverlap, 0 = Fused (producer waits at barriers)
    // component ablation (Table 8, tools/component_bench.py; batch
    // < 8): stage types run per layer, bit s = stage s -- 0x1f the decoder,
    // 0x07 stacked attention blocks (QKV, ATTN, AOUT), 0x18 stacked GLU
    // blocks (GLU, W2 / RED)
    int32_t stage_mask;
    int32_t attn_group;  // G: CTAs per (batch row, kv head)
    int32_t n_units;     // B * NKV
    int32_t debug;       // kDebug* bits; 0 in production
    uint64_t* trace;     // optional [grid][n_stages][8] trace records
    int64_t l2_prefetch; // bytes the L2 prefetch cursor runs ahead of the ring
    int32_t l2_pf_stages; // stage types (bit s % 5, bit 5 = LM head) where the
                          // producer may prefetch while its ring is full
    int32_t l2_pf_delay_ns; // hold the prefetch window this long after the
                            // layer's first K/V chunk is issued (0: no hold)
    // SM id -> dense rank (the CTA's plan index) for persistent launches, so
    // that a per-SM weighted plan (ffb_calibrate) follows the SM whatever
    // block index the launch put there; nullptr -> blockIdx.x
    const int16_t* sm_rank;
    // tensor parallelism (tp_size > 1): the residual deltas of S_AOUT and
    // S_RED and the LM-head argmax are exchanged with the other ranks over
    // peer memory (NVLink P2P / same device).  xch[r]: rank r's exchange
    // buffer [2 stage][2 layer parity][B][D] f32 + [kMaxTP][B] argmax slots;
    // xflag[r]: rank r's arrival flags [L][2][grid] + [1] (argmax).
    int32_t tp_size, tp_rank;
    int32_t tp_host;      // 1 (FFB_MODE_BASELINE_NCCL): deltas / argmax candidates only
                          // written to this rank's own buffer; the host reduces them
    int32_t vocab_base;   // first global vocab row of this rank's lm_head slice
    float* xch[8];
    uint32_t* xflag[8];
    // stacked-linear model kind (reference.hpp:141-152, interpreter.hpp:
    // 227-238): x_{l+1} = W_l x_l, square d_model layers, one stage per layer
    int32_t kind;           // 0 = llama decoder, 1 = stacked linear
    const uint8_t* wlin;    // [L][D] rows
    float* xbuf;            // [2][B][D] ping-pong activations
    float eps;
    double rope_theta;
    // batch >= 8 (Shape::KCP): every GEMV input as MMA A-fragment tables,
    // [K/16 k-steps][hi | lo][32 lanes][4 x f16x2] (1 KiB per
    // k-step; frag_off), written by the producing stage's epilogue and
    // streamed into the ring by TMA one K chunk at a time.  The RMSNorm
    // scale is factored out: tables hold x * gain, the GEMV result is
    // multiplied by 1 / rms from the per-CTA sums of squares.
    uint8_t* xfrag_a;  // x * norm_ffn[l]: S_GLU input (written by S_AOUT)
    uint8_t* xfrag_f;  // x * norm_attn[l] / final_norm: S_QKV / LM-head input
    uint8_t* afrag;    // attn_out: S_AOUT input (attention combine)
    uint8_t* hfrag;    // h = silu(g) * a: S_RED input (S_GLU)
    float* ssq;        // [2][grid][B] sum of squares of each CTA's x rows (0 after S_AOUT, 1 after S_RED)
};

// Embedding row of batch row b.  Host entry points validate token ids like
// reference_forward (reference.hpp:43-53); device-resident ids cannot be
// checked before the launch, so an out-of-range id reads row 0 and latches
// p.err_flag, reported as FFB_VALIDATION by the next synchronous call.
__device__ __forceinline__ int64_t token_row(const DecodeParams& p, int b) {
    int64_t t = p.tokens[b];
    if (t < 0 || t >= p.vocab_embed) {
        atomicOr(p.err_flag, 1u);
        t = 0;
    }
    return t;
}

// Weight storage formats of the streamed matrices (Wqkv, Waout, Wffn1,
// Wffn2^T, lm_head; the embedding is always bf16, tensor_store.hpp:356-361):
//   QB = 0   bf16 row-major [out][in]
//   QB = 4   the reference's weight-only int4 affine scheme (quant.hpp:17-60),
//            groups of 128 along the row: per row [codes: 2 per byte, little
//            nibble first][f32 scale x NG][u8 zero point x NG][pad to 16 B]
//   QB = 8   the same with 8-bit codes (255 levels; the int8 extension)
// The f32 scale and integer zero point make (c - z) * s bit-identical to the
// reference's dequantized f32 weights (the packer re-derives them exactly).
constexpr int kQuantGroup = 128;

// Shape of one tensor-parallel shard (TP = 1: the whole model): the residual
// width D and the norms/embedding are replicated; NQ / NKV are this shard's
// query / kv heads (attention width AD = NQ * DH, = D when TP = 1) and DI its
// slice of d_inter.
constexpr int gcd_(int a, int b) { return b == 0 ? a : gcd_(b, a % b); }
constexpr int pow2_div_(int v, int cap) { return (v % 2 == 0 && cap > 1) ? 2 * pow2_div_(v / 2, cap / 2) : 1; }

template <int D_, int DI_, int DH_, int NQ_, int NKV_, int B_, int QB_ = 0>
struct Shape {
    static constexpr int D = D_, DI = DI_, DH = DH_, NQ = NQ_, NKV = NKV_, B = B_, QB = QB_;
    static constexpr int AD = NQ * DH;
    static constexpr int QPG = NQ / NKV;
    static constexpr int QKVR = (NQ + 2 * NKV) * DH;
    // batch >= 8: every projection is a dense contraction on tensor cores,
    // streamed in K chunks of KC columns (RowMap::KCP, DecodeCta::gemv_kc)
    static constexpr bool KCP = B >= 8;
    static constexpr int KC = pow2_div_(gcd_(D, gcd_(AD, DI)), 512);
    static_assert(!KCP || (QB == 0 && B <= 16 && KC >= 128), "batch >= 8: bf16, K chunks >= 128");
    static_assert(AD <= D && D % AD == 0, "attention width divides d_model");
    static_assert(NQ % NKV == 0, "GQA grouping");
    static_assert(QB == 0 || QB == 4 || QB == 8, "weight format");
    static_assert(QB == 0 || AD % kQuantGroup == 0, "quant groups tile the row");
};

// bytes of one streamed-matrix row of `cols` columns in format qb
__host__ __device__ constexpr int weight_row_bytes(int cols, int qb) {
    return qb == 0 ? cols * 2
                   : ((qb == 4 ? cols / 2 : cols) + 5 * (cols / kQuantGroup) + 15) / 16 * 16;
}

// Ring geometry of the bf16 CUDA-core path (batch < 8): slot bytes and the
// most slots (pipeline depth) the ring may use.  Defaults are the measured
// optimum; other values are built only for the pipeline sweep
// (tools/pipeline_sweep.py, Table 7).
#ifndef FFB_SLOT_BYTES
#define FFB_SLOT_BYTES 32768
#endif
#ifndef FFB_MAX_SLOTS
#define FFB_MAX_SLOTS 16
#endif
constexpr int kSlotBytes = FFB_SLOT_BYTES;
constexpr int kMaxSlots = FFB_MAX_SLOTS;
static_assert(kSlotBytes % 1024 == 0 && kMaxSlots >= 2, "ring geometry");

// batch >= 8 GEMV: mma.sync m16n8k16 (default, layout 2) or tcgen05 with
// TMEM accumulators (-DFFB_KCP_TCGEN05, layout 3)
#ifdef FFB_KCP_TCGEN05
constexpr int kKcLayout = 3;
#else
constexpr int kKcLayout = 2;
#endif

constexpr int kNCW = 8;              // consumer warps
constexpr int kNCT = kNCW * 32;      // consumer threads
constexpr int cmin_(int a, int b) { return a < b ? a : b; }
constexpr int cmax_(int a, int b) { return a > b ? a : b; }
constexpr int pow2_le_(int v) {
    return v >= 32 ? 32 : v >= 16 ? 16 : v >= 8 ? 8 : v >= 4 ? 4 : v >= 2 ? 2 : 1;
}

// GEMV mapping of streamed rows with K columns (K = D for Wqkv / Wffn1 /
// Wffn2^T / lm_head, K = AD for the Waout shard).  bf16: a row = NV 16-byte
// vectors, thread lt of a row takes vectors lt, lt + TPR, ... (CPT = 8 VPT
// columns, strided).  quant: thread lt takes CPT contiguous columns (one
// quant group), so one (scale, zero) per row and thread.
template <class S, int K_>
struct RowMap {
    static constexpr int K = K_;
    static constexpr int QB = S::QB;
    static constexpr int NG = K / kQuantGroup;      // quant groups per row
    static constexpr int CODE_BYTES = QB == 4 ? K / 2 : K;
    static constexpr int ROW_BYTES = weight_row_bytes(K, QB);
    static constexpr int NV = K / 8;
    static constexpr int CPT = QB == 0 ? 8 * (NV / cmin_(NV, kNCT))
                                       : cmin_(cmin_(32, K / 32), 64 / S::B);
    static constexpr int NCH = CPT / 8;             // 8-column chunks per thread per row
    static constexpr int VPT = NCH;
    static constexpr int TPR = K / CPT;             // threads per row
    static constexpr int RG = kNCT / TPR;           // row groups working in parallel
    static constexpr int WPR = TPR / 32;            // warps per row
    // rows per thread per slot: bf16 fills a 32 KiB slot; quant takes the
    // largest power of two with RPT * B <= 32 and a slot <= 32 KiB
    static constexpr int RPT = QB == 0 ? cmin_((kSlotBytes / ROW_BYTES) / RG, 32 / S::B)
                                       : cmax_(2 / RG, cmin_(pow2_le_(32 / S::B),
                                                             pow2_le_(cmax_(1, 32768 / (RG * ROW_BYTES)))));
    // Tensor-core GEMV (quant formats, K a multiple of 8 x 128): the 8 warps
    // split K, each holds its K range of the activations as fp16 hi/lo MMA
    // B fragments in registers and decodes 16-row x 16-column weight tiles
    // straight into mma.sync A fragments (gemv_tc).  Rows of such matrices
    // use the MMA code order (weight_layout_tc); Wffn2^T (CUDA-core AXPY)
    // keeps the plain order.
    static constexpr bool TC = QB != 0 && S::B == 1 && K % (kNCW * kQuantGroup) == 0;
    static constexpr int KW = K / kNCW;             // TC: columns per warp
    static constexpr int KS = TC ? KW / 16 : 1;     // TC: k16 steps per warp
    static constexpr int TC_ROWS = QB == 4 ? 16 : 8;  // TC: rows per M tile (int8: 8 + 8 zero)
    static constexpr int RPS = TC ? TC_ROWS : RG * RPT;  // rows per slot
    static constexpr int EWPR = S::KCP ? 1 : TC ? kNCW : WPR;  // per-row partials in the epilogue
    static constexpr int APT = RPS / RG;            // rows per thread per slot (CUDA-core AXPY)
    // batch >= 8 (KCP): matrices are stored chunk-major, [K / KC][rows][KC]
    // with each row segment's 16-byte units XOR-swizzled by row & 7 (runtime
    // packer, layout 2): a weight slot is one contiguous copy of RW rows x KC
    // columns and the ldmatrix row reads are bank-conflict free.  The
    // activations of a chunk arrive as one slot of MMA A fragments (ATAB
    // bytes); warps split a weight slot as RP row parts (two n8 tiles each)
    // x KP k parts (8 k16 steps each).
    static constexpr bool KCP = S::KCP;
    static constexpr int KC = S::KC;
    static constexpr int RW = KCP ? 16384 / KC : 1;
    static constexpr int NKC = KCP ? K / KC : 1;
    static constexpr int SEG = KC * 2;
    static constexpr int WSTRIDE = SEG;
    static constexpr int ATAB = KC / 16 * 1024;
    static constexpr int RP = KCP ? RW / 16 : 1;
    static constexpr int KP = kNCW / RP;
    static constexpr int SLOT = KCP ? RW * WSTRIDE : (RPS * ROW_BYTES + 127) / 128 * 128;
    // rows per epilogue batch (whole slots; >= 64/B rows so barriers are rare)
    static constexpr int RB = KCP ? 16 : RPS > 64 / S::B ? RPS : ((64 / S::B) / RPS) * RPS;
    // (CUDA-core / quant row mapping; unused at batch >= 8)
    static_assert(KCP || (TPR % 32 == 0 && TPR <= kNCT && kNCT % TPR == 0), "a row must span whole warps");
    static_assert(KCP || (K % CPT == 0 && CPT % 8 == 0), "row mapping");
    static_assert(QB == 0 || kQuantGroup % CPT == 0, "a thread's columns lie in one group");
    static_assert(KCP || (RPS >= 1 && (RPS == 1 || RPS % 2 == 0) && RPS % RG == 0), "slot rows");
    static_assert(RB * S::B <= kNCT && (KCP || RPS * S::B <= kNCT), "epilogue threads");
    static_assert(KCP || TC || (RPT * S::B <= 32 && (RPT & (RPT - 1)) == 0),
                  "one transposed warp reduction per slot");
    static_assert(!TC || (2 * S::B <= 8 && KW % kQuantGroup == 0), "TC: hi/lo columns fit n8");
    static_assert(!KCP || (K % KC == 0 && RP * KP == kNCW && KC / 16 == 8 * KP && ATAB <= SLOT),
                  "K-chunked tensor-core GEMV geometry");
};

template <class S>
struct KTraits : RowMap<S, S::D> {
    using MD = RowMap<S, S::D>;   // rows of d_model columns
    using MA = RowMap<S, S::AD>;  // Waout shard rows (attention width)
    // Two-phase FFN (bf16, batch <= 2, d_model >= 4096, d_inter a multiple
    // of 8 x 256 whose bf16 row fits a slot): S_GLU writes h = silu(g) * a
    // to global memory and S_RED streams W2 rows ([D][DI], row-owned like
    // Waout) against it -- no per-CTA d_model partials and no reduction
    // pass, one more full-grid barrier inside the FFN.  Otherwise Wffn2^T
    // rows are AXPYed into per-CTA partials that S_RED sums.  Same-box A/B:
    // 8B b1 2.725 -> 2.700 ms, b2 3.204 -> 3.176; 1B b1 0.638 -> 0.650
    // (the reduction of 2048-wide partials is cheaper than the barrier).
    static constexpr bool F2R = S::KCP || (S::QB == 0 && S::B <= 2 && S::D >= 4096 &&
                                           S::DI % (8 * kNCT) == 0 && S::DI * 2 <= kSlotBytes);
    using MF = std::conditional_t<F2R, RowMap<S, S::DI>, MD>;
    static constexpr int NCW = kNCW;
    static constexpr int NCT = kNCT;
    // + a producer warpgroup (one active lane): with 12 warps the warpgroups
    // rebalance registers (setmaxnreg) -- the producer gives its registers to
    // the two consumer warpgroups (9 warps would cap everyone at 168)
    static constexpr int NTHREADS = NCT + 128;
    static constexpr int PRODUCER_REGS = 56;
    static constexpr int CONSUMER_REGS = 224;  // 4*32*56 + 8*32*224 <= 64K
    static constexpr int cmin(int a, int b) { return a < b ? a : b; }
    static constexpr int cmax(int a, int b) { return a > b ? a : b; }
    static constexpr int SLOT_BYTES = S::KCP ? MD::SLOT : S::QB == 0 ? kSlotBytes : cmax(MD::SLOT, MA::SLOT);
    // KCP: [KP][RW][B] k-part partials + [RW][B] finished rows (gemv_kc)
    static constexpr int RED_FLOATS =
        S::KCP ? (MD::KP * MD::RW * S::B + MD::RW * S::B + 1) / 2
               : cmax(cmax(MD::EWPR * MD::RB, MA::EWPR * MA::RB), MF::EWPR * MF::RB) * S::B;
    static constexpr int KVC = SLOT_BYTES / (2 * S::DH * 2);  // KV positions per slot
    static constexpr int DPL = S::DH / 32;          // attention dims per lane
    // max GLU pairs / Waout rows per CTA (host-checked): a CTA's share with
    // calibration headroom (weights up to 1.3x the mean), for grids down to
    // 148 / TP CTAs (a TP group co-located on one GPU, TP = D / AD)
    static constexpr int GMIN = 148 / (S::D / S::AD);
    static constexpr int TMAX = cmax(160, (cmax(S::DI, S::D) * 135 / (100 * GMIN) + 15) / 16 * 16);
    static_assert(MD::SLOT <= SLOT_BYTES && MA::SLOT <= SLOT_BYTES && MF::SLOT <= SLOT_BYTES,
                  "slot fits every row map");
    static_assert(S::DH % 32 == 0 && DPL <= 8, "attention lane split");
    static_assert(KVC >= 1 && (SLOT_BYTES / 2) % 16 == 0, "kv chunk");

    // ---- shared memory carve-up (bytes) ----
    static constexpr int R_RED = 0;  // [2][WPR][RB][B] f32 (largest row map)
    static constexpr int SZ_RED = 2 * RED_FLOATS * 4;
    static constexpr int R_H = R_RED + SZ_RED;  // [B][TMAX] f32
    // [B][TMAX] f32 (GLU h slice, S_AOUT / S_RED row results); batch >= 8
    // only stages the current token's K and V rows (attention)
    static constexpr int SZ_H = S::KCP ? (4 * S::DH + 15) / 16 * 16 : S::B * TMAX * 4;
    static constexpr int R_ROPE = R_H + SZ_H;  // [DH/2][2] f32
    static constexpr int SZ_ROPE = S::DH * 4;
    static constexpr int R_NORM = R_ROPE + SZ_ROPE;  // [NCW][B] f32
    static constexpr int SZ_NORM = ((NCW + 1) * S::B * 4 + 16 + 15) / 16 * 16;  // [NCW][B] partials + [B] (KCP inv)
    static constexpr int R_WPART = R_NORM + SZ_NORM;  // attention scratch, f32
    // also reused for: attention combine (3*G*QPG), argmax candidates
    // (2*grid*B) and the GLU reduction (NCW*32); grid <= kMaxGrid
    static constexpr int kMaxGrid = 160;
    // attention: ring slots consumed together in one softmax pass (~128 KiB
    // of K/V), positions per pass (+1 for the current token, rounded to 4)
    // and its scratch: alpha*q [QPG][DH], scores [QPG][ANP], probabilities
    // [ANP][QPG], stats
    // (batch 1 at 4k context fits one pass of 4 slots; batch > 1 runs
    // several passes, the producer filling the next pass's slots while this
    // one computes: 4-slot passes at batch 2 (2 passes at 4k), 2 from batch
    // 4 on -- same-box A/B at 8B, 4k context: b2 3.17 / 3.14 ms for 3 / 4
    // slots; with the per-warp attention b4 3.77 / 3.75, b8 6.41 / 6.38,
    // b16 7.32 / 7.30 ms for 3 / 2 slots (b16 7.65 with 1))
    static constexpr int ATT_SC =
        cmin(S::B == 1 ? cmax(1, (131072 + SLOT_BYTES - 1) / SLOT_BYTES) : S::B == 2 ? 4 : 2, kMaxSlots - 1);
    static constexpr int ANP = ((ATT_SC * KVC + 1) + 15) / 16 * 16;
    // alpha*q f32 [QPG][DH], scores f32 [QPG][ANP], probabilities as bf16
    // hi/lo MMA rows [16][ANP] (tensor-core P.V), stats [QPG][4]
    // per-warp attention (ATT_WARP): alpha*q [QPG][DH], then per warp (m, l)
    // [NCW][QPG][2] and O [NCW][QPG][DH] for the CTA merge.  Same-box A/B
    // against the three-barrier passes (attn_pass_tc), ms/step: 8B b16 8.18
    // -> 7.37, b4 3.93 -> 3.76, b2 3.11 -> 3.10, 1B b1 0.639 -> 0.629; 8B b1
    // (one ~230-position pass per CTA) was 2.700 -> 2.748 in round 1 and,
    // with the producer free of spills (round 2), 2.804 -> 2.789 and int4
    // 1.870 -> 1.833: the per-warp path everywhere.  QPG = 8 (70B) would
    // need 32 KiB of merge scratch: passes.
#ifdef FFB_ATT_PASS
    static constexpr bool ATT_WARP = false;
#else
    static constexpr bool ATT_WARP = S::QPG <= 4;
#endif
    static constexpr int SZ_ATT = ATT_WARP
        ? S::QPG * S::DH + 2 * NCW * S::QPG + NCW * S::QPG * S::DH
        : S::QPG * S::DH + S::QPG * ANP + cmax(S::QPG, 8) * ANP + 4 * S::QPG;
    static constexpr int SZ_WPART =
        4 * cmax(cmax(cmax(cmax(S::QPG * S::DH, 3 * kMaxGrid * S::QPG),
                           // argmax candidates (batch >= 8: in the drained
                           // ring), S_RED scratch + TP delta, TP exchange rows
                           cmax(S::KCP ? 0 : 2 * kMaxGrid * S::B, NCW * 32 + S::B * TMAX)),
                      SZ_ATT),
                 cmax(MD::TC ? S::D + 2 * S::D / kQuantGroup : 0,  // TC activation strips + group words
                      MA::TC ? S::AD + 2 * S::AD / kQuantGroup : 0));
    static_assert(R_H % 16 == 0 && R_NORM % 16 == 0 && R_WPART % 16 == 0,
                  "16-byte aligned scratch (vector smem accesses)");
    static constexpr int R_AMAX = R_WPART + SZ_WPART;  // [NCT] (f32, i32)
    static constexpr int SZ_AMAX = NCT * 8;
    static constexpr int R_MISC = R_AMAX + SZ_AMAX;  // flags
    static constexpr int SZ_MISC = 256;
    static constexpr int FIXED = ((R_MISC + SZ_MISC + 1023) / 1024) * 1024;
    static constexpr int MAX_SMEM = 227 * 1024;
    // batch >= 8 (tcgen05): barriers at 0, the ring at 1024 (128-byte-swizzle
    // atoms need 1024-byte alignment) and the fixed scratch after it, which
    // keeps the M = 128 MMA's reads of the A table's padding rows past the
    // last slot inside shared memory (gemv_kc); otherwise scratch, barriers
    // and the ring in that order
    static constexpr int NSLOTS_RAW = (MAX_SMEM - FIXED - (S::KCP ? 1024 : 256)) / SLOT_BYTES;
    static constexpr int NSLOTS = NSLOTS_RAW > kMaxSlots ? kMaxSlots : NSLOTS_RAW;
    static_assert(NSLOTS >= 2, "ring too small");
    static_assert(NSLOTS >= ATT_SC + 1, "attention pass must leave a slot for streaming");
    static constexpr int OFF_BARS = S::KCP ? 0 : FIXED;  // full[NSLOTS], empty[NSLOTS], (KCP) acc
    static constexpr int OFF_RING = S::KCP ? 1024 : FIXED + 256;
    static constexpr int SHIFT = S::KCP ? OFF_RING + NSLOTS * SLOT_BYTES : 0;
    static constexpr int OFF_RED = SHIFT + R_RED, OFF_H = SHIFT + R_H, OFF_ROPE = SHIFT + R_ROPE,
                         OFF_NORM = SHIFT + R_NORM, OFF_WPART = SHIFT + R_WPART, OFF_AMAX = SHIFT + R_AMAX,
                         OFF_MISC = SHIFT + R_MISC;
    static constexpr int SMEM_BYTES = S::KCP ? SHIFT + FIXED : OFF_RING + NSLOTS * SLOT_BYTES;
    static_assert(!S::KCP || 2 * NSLOTS + 2 <= 128, "tcgen05 barriers below the ring");
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
    // this CTA's plan, staged in shared memory (misc + 128 B): neither role
    // keeps its 14 fields in registers (the 56-register producer spilled them)
    CtaPlan& pl;
    int cta, grid;

    __device__ DecodeCta(const DecodeParams& p_, uint8_t* smem_)
        : p(p_), smem(smem_), pl(*reinterpret_cast<CtaPlan*>(smem_ + T::OFF_MISC + 128)) {
        full = reinterpret_cast<uint64_t*>(smem + T::OFF_BARS);
        empty = full + T::NSLOTS;
        ring = smem + T::OFF_RING;
        cta = blockIdx.x;
        if (p.sm_rank != nullptr) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            cta = p.sm_rank[smid];
        }
        grid = gridDim.x;
        static_assert(sizeof(CtaPlan) % 4 == 0 && 128 + sizeof(CtaPlan) <= T::SZ_MISC, "plan in misc");
        if (threadIdx.x < sizeof(CtaPlan) / 4)  // (read after the kernel's __syncthreads)
            reinterpret_cast<int32_t*>(&pl)[threadIdx.x] =
                reinterpret_cast<const int32_t*>(p.plan + cta)[threadIdx.x];
    }

    __device__ float* red_buf(uint32_t it) {
        return reinterpret_cast<float*>(smem + T::OFF_RED) + (it & 1) * T::RED_FLOATS;
    }
    __device__ float* h_s() { return reinterpret_cast<float*>(smem + T::OFF_H); }
    __device__ float* rope() { return reinterpret_cast<float*>(smem + T::OFF_ROPE); }
    __device__ float* norm_s() { return reinterpret_cast<float*>(smem + T::OFF_NORM); }
    __device__ float* wpart() { return reinterpret_cast<float*>(smem + T::OFF_WPART); }
    __device__ int* misc() { return reinterpret_cast<int*>(smem + T::OFF_MISC); }
    // batch >= 8: TMEM base address (written by tcgen05.alloc) and the
    // accumulator-ready barrier (gemv_kc), one phase per row block
    __device__ uint32_t* tmem_slot() { return reinterpret_cast<uint32_t*>(misc()) + 62; }
    __device__ uint32_t tmem_base() { return *reinterpret_cast<volatile uint32_t*>(tmem_slot()); }
    __device__ uint64_t* accbar() { return full + 2 * T::NSLOTS; }
    __device__ uint64_t* abar() { return full + 2 * T::NSLOTS + 1; }  // TMEM A buffer reusable
    uint32_t acc_phase = 0, a_phase = 0;
    bool a_issued = false;  // an abar commit is outstanding

    // ------------------------------------------------------------ schedule
    __device__ int n_stages() const {
        return p.kind == 1 ? p.layers : p.layers * kStagesPerLayer + 1;
    }

    // counter a stage's consumers wait on before starting, and its target
    __device__ bool dependency(int stage, const uint32_t** ctr, uint32_t* target) const {
        const int l = stage / kStagesPerLayer, s = stage % kStagesPerLayer;
        const uint32_t full_grid = p.epoch * static_cast<uint32_t>(grid);
        if (p.kind == 1) {  // stacked linear: layer l needs every row of layer l - 1
            if (stage == 0) return false;
            *ctr = p.counters + stage - 1;
            *target = full_grid;
            return true;
        }
        const bool red_on = (p.stage_mask >> S_RED) & 1;
        if (stage == p.layers * kStagesPerLayer) {  // LM head
            if (p.layers == 0) {
                if constexpr (!S::KCP) return false;
                *ctr = p.counters + p.layers * kStagesPerLayer + 1;  // init counter
                *target = full_grid;
                return true;
            }
            *ctr = p.counters + (p.layers - 1) * kStagesPerLayer + (red_on ? S_RED : S_AOUT);
            *target = full_grid;
            return true;
        }
        if (!((p.stage_mask >> s) & 1)) return false;  // (component ablation: stage not run)
        switch (s) {
            case S_QKV:
                if (l == 0) {
                    if constexpr (!S::KCP) return false;
                    // KCP: every CTA's initial x rows and A table (kc_publish)
                    *ctr = p.counters + p.layers * kStagesPerLayer + 1;
                    *target = full_grid;
                    return true;
                }
                *ctr = p.counters + (l - 1) * kStagesPerLayer + (red_on ? S_RED : S_AOUT);
                *target = full_grid;
                return true;
            case S_ATTN:  // only the CTAs that computed this kv head's q/k/v rows
                if (pl.attn_unit < 0) return false;
                *ctr = p.qkv_head_counters + l * S::NKV + pl.attn_unit % S::NKV;
                *target = p.epoch * static_cast<uint32_t>(pl.attn_dep);
                return true;
            case S_AOUT:
                *ctr = p.counters + l * kStagesPerLayer + S_ATTN;
                *target = p.epoch * static_cast<uint32_t>(p.n_units);
                return true;
            case S_GLU:
                if (!((p.stage_mask >> S_AOUT) & 1)) {  // stacked GLU blocks: the previous W2
                    if (l == 0) return false;
                    *ctr = p.counters + (l - 1) * kStagesPerLayer + S_RED;
                } else {
                    *ctr = p.counters + l * kStagesPerLayer + S_AOUT;
                }
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

    // KV rows are stored with their 16-byte chunks XOR-swizzled by (pos & 7)
    // (runtime.cu applies the same map on import/export): element `dim` of
    // position `pos` lives at this offset inside the row.
    __device__ static int kv_swz_dim(int dim, int pos) {
        return ((((dim >> 3) ^ (pos & 7))) << 3) | (dim & 7);
    }

    // ============================================================ producer
    // The static schedule walked twice: by the producer lane (DRAIN=false:
    // issue TMA into free slots) and, in the streaming-only debug mode, by the
    // consumer warps (DRAIN=true: wait for each slot and release it).
    template <bool DRAIN>
    __device__ void chunk(uint32_t& it, const void* src0, const void* src1, uint32_t bytes,
                          uint32_t off1, uint64_t policy) {
        const uint32_t slot = it % T::NSLOTS, ph = (it / T::NSLOTS) & 1;
        if (DRAIN) {
            mbar_wait(&full[slot], ph);
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[slot]);
        } else {
            mbar_wait(&empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&full[slot], src1 ? 2 * bytes : bytes);
            uint8_t* dst = ring + slot * T::SLOT_BYTES;
            tma_load_1d(dst, src0, bytes, &full[slot], policy);
            if (src1) tma_load_1d(dst + off1, src1, bytes, &full[slot], policy);
        }
        ++it;
    }

    // One list of the static per-CTA stream: rows [r0, r1) of a matrix (kv =
    // false) or KV positions [r0, r1) of one (layer, batch row, kv head).
    struct List {
        const uint8_t* base;  // matrix rows, or K rows (kv) of one (l, b, head)
        int r0, r1;
        bool kv;
        int row_bytes = T::ROW_BYTES, rps = T::RPS;  // matrix row geometry
        // KCP: per row block, per K chunk: the chunk's A-fragment table (one
        // slot, dependency-gated) then RW-row weight slots of the chunk
        const uint8_t* atab = nullptr;
        int nkc = 0;
        int rows_total = 0;  // KCP: rows of the chunk-major matrix
    };
    // KCP rows per accumulator block: TMEM holds the K chunk's activations
    // (KC / 2 columns, the MMA's A operand) and the block's accumulators (RW
    // columns per weight slot) in 512 columns; the A table is streamed once
    // per block and K chunk
#ifdef FFB_KCP_TCGEN05
    static constexpr int TM_A = 256;  // TMEM columns reserved for the A operand (KC <= 512)
    static constexpr int KC_BLOCK = cmax_(T::MD::RW, (512 - TM_A) / T::MD::RW * T::MD::RW);
#else
    // mma.sync path: per-warp register accumulators for 128 rows (same-box
    // A/B at 8B b16: 7.39 ms with 160-row blocks, 7.32 with 128)
    static constexpr int KC_BLOCK = cmax_(T::MD::RW, cmin_(128, (T::NSLOTS - 1) * T::MD::RW));
#endif

    // The lists of (stage, sub) in consumption order; false past the end.
    __device__ bool list_of(int stage, int sub, List& L) const {
        const int l = stage / kStagesPerLayer, s = stage % kStagesPerLayer;
        if (p.kind == 1) {
            if (sub > 0) return false;
            L = {p.wlin + (size_t)stage * D * T::ROW_BYTES, pl.aout_r0, pl.aout_r1, false};
            return true;
        }
        if (stage == p.layers * kStagesPerLayer) {
            if (sub > 0) return false;
            L = {p.lm_head, pl.lm_r0, pl.lm_r1, false};
            if constexpr (S::KCP) { L.atab = p.xfrag_f; L.nkc = MD::NKC; L.rows_total = p.vocab; }
            return true;
        }
        if (!((p.stage_mask >> s) & 1)) return false;  // (component ablation)
        switch (s) {
            case S_QKV:
                if (sub > 0) return false;
                L = {p.wqkv + (size_t)l * S::QKVR * T::ROW_BYTES, pl.qkv_r0, pl.qkv_r1, false};
                if constexpr (S::KCP) { L.atab = p.xfrag_f; L.nkc = MD::NKC; L.rows_total = S::QKVR; }
                return true;
            case S_ATTN: {
                if (sub > 0 || pl.attn_unit < 0) return false;
                int p0, p1;
                attn_range(p0, p1);
                const int unit = pl.attn_unit;
                L = {reinterpret_cast<const uint8_t*>(p.kcache + kv_row(l, unit / S::NKV,
                                                                        unit % S::NKV, 0)),
                     p0, min(p1, p.pos), true};
                return true;
            }
            case S_AOUT:
                if (sub > 0) return false;
                L = {p.waout + (size_t)l * D * MA::ROW_BYTES, pl.aout_r0, pl.aout_r1, false,
                     MA::ROW_BYTES, MA::RPS};
                if constexpr (S::KCP) { L.atab = p.afrag; L.nkc = MA::NKC; L.rows_total = D; }
                return true;
            case S_GLU:
                if (sub == 0) {
                    L = {p.wffn1 + (size_t)l * 2 * S::DI * T::ROW_BYTES, 2 * pl.glu_t0,
                         2 * pl.glu_t1, false};
                    if constexpr (S::KCP) { L.atab = p.xfrag_a; L.nkc = MD::NKC; L.rows_total = 2 * S::DI; }
                }
                else if (sub == 1 && !T::F2R)
                    L = {p.wffn2t + (size_t)l * S::DI * T::ROW_BYTES, pl.glu_t0, pl.glu_t1, false};
                else return false;
                return true;
            case S_RED:  // two-phase FFN: W2 rows, the CTA's d_model rows (as Waout)
                if (!T::F2R || sub > 0) return false;
                L = {p.wffn2t + (size_t)l * D * MF::ROW_BYTES, pl.aout_r0, pl.aout_r1, false, MF::ROW_BYTES, MF::RPS};
                if constexpr (S::KCP) { L.atab = p.hfrag; L.nkc = MF::NKC; L.rows_total = D; }
                return true;
            default:
                return false;
        }
    }

    // Walks the per-CTA stream chunk by chunk (one ring slot each).
    struct Cursor {
        int stage, sub, c0;
        bool valid;
        List L;
        int kcc, kcj;  // KCP: chunk, slot within the chunk (-1: A table)
        bool out_dep;  // the emitted chunk reads data of this stage's dependency
    };

    __device__ void cursor_init(Cursor& c) const {
        c.stage = p.stage_begin;
        c.sub = 0;
        c.valid = false;
    }

    // Next chunk: K/matrix source, V source (kv only), bytes per source, stage.
    __device__ bool cursor_next(Cursor& c, const void** src0, const void** src1,
                                uint32_t* bytes, int* stage) const {
        const int last = min(p.stage_end, n_stages());
        while (c.stage < last) {
            if (!c.valid) {
                if (!list_of(c.stage, c.sub, c.L)) {
                    ++c.stage;
                    c.sub = 0;
                    continue;
                }
                c.valid = true;
                c.c0 = c.L.r0;
                c.kcc = 0;
                c.kcj = -1;
            }
            if (c.c0 >= c.L.r1) {
                c.valid = false;
                ++c.sub;
                continue;
            }
            *stage = c.stage;
            c.out_dep = false;
            if (c.L.nkc > 0) {  // KCP
                const int blk_end = min(c.c0 + KC_BLOCK, c.L.r1);
                if (c.kcj < 0) {
                    *src0 = c.L.atab + (size_t)c.kcc * MD::ATAB;
                    *src1 = nullptr;
                    *bytes = MD::ATAB;
                    c.out_dep = true;
                    c.kcj = 0;
                    return true;
                }
                const int row0 = c.c0 + c.kcj * MD::RW;
                if (row0 < blk_end) {  // rows [row0, row0 + n) of chunk kcc: contiguous
                    *src0 = c.L.base + ((size_t)c.kcc * c.L.rows_total + row0) * MD::SEG;
                    *src1 = nullptr;
                    *bytes = min(MD::RW, blk_end - row0) * MD::SEG;
                    ++c.kcj;
                    return true;
                }
                c.kcj = -1;
                if (++c.kcc == c.L.nkc) {
                    c.kcc = 0;
                    c.c0 = blk_end;
                }
                continue;
            }
            if (c.L.kv) {
                const int n = min(T::KVC, c.L.r1 - c.c0);
                const size_t off = (size_t)c.c0 * DH * 2;
                *src0 = c.L.base + off;
                *src1 = reinterpret_cast<const uint8_t*>(p.vcache) +
                        (c.L.base - reinterpret_cast<const uint8_t*>(p.kcache)) + off;
                *bytes = static_cast<uint32_t>(n) * DH * 2;
                c.c0 += T::KVC;
            } else {
                const int n = min(c.L.rps, c.L.r1 - c.c0);
                *src0 = c.L.base + (size_t)c.c0 * c.L.row_bytes;
                *src1 = nullptr;
                *bytes = static_cast<uint32_t>(n) * c.L.row_bytes;
                c.c0 += c.L.rps;
            }
            return true;
        }
        return false;
    }

    // Producer: issues every chunk of the stream into the ring (TMA bulk).
    // FusedOverlap: gated only by free slots, plus an L2 prefetch cursor
    // (cp.async.bulk.prefetch.L2) running up to p.l2_prefetch bytes ahead of
    // the ring so HBM keeps streaming through barrier/latency phases.
    // Fused: waits at every stage boundary (emit.hpp:229-235 without hoisting).
    // DRAIN (streaming-only debug): consumers walk the same stream.
    template <bool DRAIN>
    __device__ void producer() {
        const uint64_t policy = policy_evict_first();
        uint32_t it = 0;
        Cursor c, pf;
        cursor_init(c);
        cursor_init(pf);
        // (batch >= 8 never prefetches: the runtime sets no window there)
        const int64_t window = (!DRAIN && p.overlap && !S::KCP) ? p.l2_prefetch : 0;
        int64_t ahead = 0;  // bytes prefetched but not yet loaded into the ring
        int64_t pf_bytes = 0;
        bool pf_live = window > 0;
        int cur_stage = p.stage_begin;
        int dep_stage = -1;  // KCP: last stage whose dependency the producer waited for
        int kv_stage = -1;   // l2_pf_delay_ns: last S_ATTN stage whose first chunk went out
#ifdef FFB_TRACE_PRODUCER
        int pt_stage = -1;
#endif
        uint64_t t_kv = 0;
        const void *s0, *s1;
        uint32_t bytes;
        int stage;
        while (cursor_next(c, &s0, &s1, &bytes, &stage)) {
            if (!DRAIN && !p.overlap && stage != cur_stage) {
                for (int s = cur_stage + 1; s <= stage; ++s) {
                    const uint32_t* ctr;
                    uint32_t target;
                    if (dependency(s, &ctr, &target)) spin_until_geq(ctr, target);
                }
            }
            cur_stage = stage;
            if constexpr (S::KCP) {
                if (c.out_dep && !DRAIN && stage != dep_stage && !(p.debug & kDebugStreamOnly)) {
                    // the A table is written by the previous stage's epilogues
                    // (every mode: the stage-change wait of the non-overlap
                    // modes skips a launch's first stage)
                    const uint32_t* ctr;
                    uint32_t target;
                    if (dependency(stage, &ctr, &target)) spin_until_geq(ctr, target);
                    fence_proxy_async_global();
                    dep_stage = stage;
                }
            }
            const int64_t need = s1 ? 2 * (int64_t)bytes : bytes;
            if (!DRAIN && !S::KCP) {
                // Prefetch into L2 only while the ring is full (this SM cannot
                // load anyway, typically behind a barrier), never more than
                // `window` bytes ahead of the ring: idle HBM time is spent on
                // the bytes the ring will want next.
                const uint32_t slot = it % T::NSLOTS, ph = (it / T::NSLOTS) & 1;
                if (ahead < need) {  // pf cursor must stay ahead of the main one
                    ahead = 0;
                    pf = c;  // restart just past this chunk
                }
                // ring full: issue the whole prefetch window at once (no
                // waiting between prefetches), then block on the slot
                const int stype = stage == p.layers * kStagesPerLayer ? 5 : stage % kStagesPerLayer;
                bool hold = false;
                if (((p.l2_pf_stages >> stype) & 1) && !mbar_test_wait(&empty[slot], ph ^ 1) &&
                    p.l2_pf_delay_ns > 0 && pf_live && ahead < window) {
                    // the layer's own K/V loads (on the attention chain) go
                    // to HBM ahead of the window's bulk: poll for the slot
                    // until the hold time has passed since they were issued
                    while (gtimer() - t_kv < static_cast<uint64_t>(p.l2_pf_delay_ns)) {
                        if (mbar_test_wait(&empty[slot], ph ^ 1)) {
                            hold = true;  // slot free: load it, prefetch at a later chunk
                            break;
                        }
                    }
                }
                if (!hold && ((p.l2_pf_stages >> stype) & 1) && !mbar_test_wait(&empty[slot], ph ^ 1)) {
                    while (pf_live && ahead < window) {
                        const void *q0, *q1;
                        uint32_t qb;
                        int qs;
                        if (!cursor_next(pf, &q0, &q1, &qb, &qs)) {
                            pf_live = false;
                            break;
                        }
                        prefetch_l2(q0, qb);
                        if (q1) prefetch_l2(q1, qb);
                        ahead += q1 ? 2 * (int64_t)qb : qb;
                        pf_bytes += q1 ? 2 * (int64_t)qb : qb;
                    }
                }
                ahead -= need;
            }
#ifdef FFB_TRACE_PRODUCER  // diagnostic build: when the K/V chunks go out (tools/trace_kv_issue.py)
            const bool kvc = !DRAIN && p.trace != nullptr && stage % kStagesPerLayer == S_ATTN &&
                             stage < p.layers * kStagesPerLayer;
            const uint64_t tb = kvc ? gtimer() : 0;
#endif
            chunk<DRAIN>(it, s0, s1, bytes, T::SLOT_BYTES / 2, policy);
#ifdef FFB_TRACE_PRODUCER
            if (kvc) {
                uint64_t* t = p.trace + ((size_t)cta * n_stages() + stage - S_ATTN + S_AOUT) * kTraceSlots;
                const uint64_t ta = gtimer();
                if (stage != pt_stage) {
                    t[5] = tb;
                    t[6] = ta;
                    pt_stage = stage;
                }
                t[7] = ta;
            }
#endif
            if (!DRAIN && p.l2_pf_delay_ns > 0 && stage != kv_stage && stage % kStagesPerLayer == S_ATTN) {
                kv_stage = stage;  // first K/V chunk of this layer issued
                t_kv = gtimer();
            }
        }
        // producer trace: L2-prefetched bytes of this launch (last stage, slot 5)
        // and the SM this CTA ran on (slot 6)
        if (p.trace != nullptr && !DRAIN) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            uint64_t* t = p.trace + ((size_t)cta * n_stages() + n_stages() - 1) * kTraceSlots;
            t[5] = pf_bytes;
            t[6] = smid;
        }
    }

    // ============================================================ consumers
    __device__ static float warp_sum(float v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    }

    __device__ static float warp_max(float v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        return v;
    }

    // per-CTA %globaltimer trace: [grid][n_stages][4] = entry, dependency met,
    // stage done (arrived), spare.  Off (nullptr) in production.
    __device__ static uint64_t gtimer() {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    }

    __device__ void trace_put(int stage, int slot, uint64_t v) {
        if (p.trace != nullptr && threadIdx.x == 0)
            p.trace[((size_t)cta * n_stages() + stage) * kTraceSlots + slot] = v;
    }

    __device__ void trace_mark(int stage, int slot) {
        if (p.trace != nullptr && threadIdx.x == 0) trace_put(stage, slot, gtimer());
    }

    // consumer wait for ring data; with tracing on, thread 0 accumulates the
    // time spent starved (trace slot 4)
    uint64_t ring_wait_ns = 0;
    __device__ void wait_full(uint32_t slot, uint32_t par) {
        if (p.trace != nullptr && threadIdx.x == 0) {
            const uint64_t t0 = gtimer();
            mbar_wait(&full[slot], par);
            ring_wait_ns += gtimer() - t0;
        } else {
            mbar_wait(&full[slot], par);
        }
    }

    __device__ void trace_ring_wait(int stage) {
        trace_put(stage, 4, ring_wait_ns);
        ring_wait_ns = 0;
    }

    // Dependency wait: one thread spins (acquire), the named barrier hands
    // the ordering to the other consumer threads (cf. CUTLASS grid barrier).
    __device__ void wait_stage(int stage) {
        const uint32_t* ctr;
        uint32_t target;
        if (dependency(stage, &ctr, &target)) {
            if (threadIdx.x == 0) spin_until_geq(ctr, target);
            consumer_sync(NCT);
        }
        trace_mark(stage, 1);
    }

    // Stage completion: named barrier orders every consumer's writes before
    // thread 0's gpu-scope release-add (cumulativity); no separate fence.
    __device__ void arrive(uint32_t* ctr, int stage) {
        consumer_sync(NCT);
        if (threadIdx.x == 0) red_release_gpu(ctr, 1);
        trace_mark(stage, 2);
        trace_ring_wait(stage);
    }

    // This thread's activation slice of one GEMV stage: v[b][ci][e] = column
    // col_of(lt, ci) + e.  Quant formats also keep sum[b] = the sum of the
    // thread's (unscaled) activations -- the zero-point term of
    // s * sum_i (c_i - z) a_i = s * (sum_i c_i a_i - z * sum[b]) -- and, for
    // int4, pre-scale column e by q4_scale(e), the inverse of the power of
    // 16 at which the nibble decode (q4_decode) leaves code e.
    using MD = typename T::MD;
    using MA = typename T::MA;
    using MF = typename T::MF;

    template <class M = MD>
    struct Act {
        float v[B][M::TC ? 1 : M::NCH][8];
        float sum[B];
    };

    template <class M = MD>
    __device__ static int col_of(int lt, int ci) {
        return M::QB ? lt * M::CPT + ci * 8 : (lt + ci * M::TPR) * 8;
    }

    // int4 nibble e of a 32-bit code word is decoded in place as c * 16^k(e):
    // e = 0..4 by masking bits 4e..4e+3, e = 5..7 from the word >> 20
    __device__ static constexpr float q4_scale(int e) {
        return e == 0 || e == 5 ? 1.f
               : e == 1 || e == 6 ? 0.0625f
               : e == 2 || e == 7 ? 0.00390625f
               : e == 3 ? 0.000244140625f : 0.0000152587890625f;
    }

    // ---- tensor-core GEMV (quant formats) -----------------------------
    // Activation column k of batch row b (layer-0 input from the embedding).
    template <class M>
    __device__ __forceinline__ float2 act_pair(const float* src, bool from_emb, int b, int k) const {
        if (from_emb) {
            const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(
                p.embedding + (size_t)token_row(p, b) * D + k));
            return make_float2(bf_lo(w), bf_hi(w));
        }
        return __ldcg(reinterpret_cast<const float2*>(src + (size_t)b * M::K + k));
    }

    // MMA B fragments (m16n8k16, "col"): lane (g, q) holds column n = g
    // = batch row g % B as fp16 hi (g < B) or lo (B <= g < 2B) part, rows
    // k = 2q, 2q+1 (bf[j][0]) and 2q+8, 2q+9 (bf[j][1]) of k-step j of the
    // warp's K range.  hi + lo carries 22 bits of each f32 activation; int4
    // pre-scales the second register by 1/16 (see gemv_tc's decode).
    template <class M>
    __device__ __forceinline__ void load_act_tc(Act<M>& act, const float* src, bool from_emb, const float* gain,
                                int stage) {
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32, g = lane / 4, q = lane % 4;
        constexpr int PL = M::KW / 32;  // columns per lane of the warp's K range (16 at d 4096)
        static_assert(PL % 4 == 0, "float4 staging");
        const int col0 = warp * M::KW + lane * PL;
        float gl[PL];
        if (gain != nullptr) {
#pragma unroll
            for (int i = 0; i < PL; i += 4) {
                const float4 g4 = __ldg(reinterpret_cast<const float4*>(gain + col0 + i));
                gl[i] = g4.x; gl[i + 1] = g4.y; gl[i + 2] = g4.z; gl[i + 3] = g4.w;
            }
        }
        wait_stage(stage);
        // coalesced load of the warp's K range (lane: PL consecutive columns)
        float v[B][PL];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            if (from_emb) {
                const __nv_bfloat16* e = p.embedding + (size_t)token_row(p, b) * D + col0;
#pragma unroll
                for (int i = 0; i < PL; i += 8) {
                    const uint4 w = __ldg(reinterpret_cast<const uint4*>(e + i));
                    v[b][i] = bf_lo(w.x); v[b][i + 1] = bf_hi(w.x);
                    v[b][i + 2] = bf_lo(w.y); v[b][i + 3] = bf_hi(w.y);
                    v[b][i + 4] = bf_lo(w.z); v[b][i + 5] = bf_hi(w.z);
                    v[b][i + 6] = bf_lo(w.w); v[b][i + 7] = bf_hi(w.w);
                }
            } else {
#pragma unroll
                for (int i = 0; i < PL; i += 4) {
                    const float4 a4 = ldcg_f4(src + (size_t)b * M::K + col0 + i);
                    v[b][i] = a4.x; v[b][i + 1] = a4.y; v[b][i + 2] = a4.z; v[b][i + 3] = a4.w;
                }
            }
        }
        // RMSNorm statistics over the whole row (numerics.hpp:14-24): the
        // warp partials go to smem now, the row's 1/rms is formed after the
        // table barrier below -- the int8 terms of gain * x do not depend on
        // it (the block scale absorbs it: dq = inv * max|gain * x| / 127)
        float* ns = norm_s();
        if (gain != nullptr) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
                float sq = 0.f;
#pragma unroll
                for (int i = 0; i < PL; ++i) sq = fmaf(v[b][i], v[b][i], sq);
                sq = warp_sum(sq);
                if (lane == 0) ns[warp * B + b] = sq;
            }
        }
        // MMA B fragments (m16n8k32 "col", s8, batch 1): each 128-column
        // group of activations as three int8 terms of one block scale,
        //   x = dq * (x0 + x1 / 254 + x2 / 254^2),  |x0|, |x1|, |x2| <= 127,
        // i.e. 23 bits relative to the group's largest |x| (dq = max / 127);
        // column n = term n, n = 3 zero.  Lane (g, q) of k32-step s needs
        // rows 4q..4q+3 (reg 0) and 16+4q..16+4q+3 (reg 1) of column g.  Each
        // lane quantises its PL columns (a half k32-step per 16) into this
        // warp's strip [step][n][q][reg]; per group, (dq, sum of x0 + x1/254
        // + x2/254^2) for the zero-point term follows the NCW strips.
        static_assert(PL % 16 == 0 && 128 % PL == 0, "half k32-steps per lane, whole lanes per group");
        constexpr int LPG = 128 / PL;  // lanes per quant group
        uint32_t* tab = reinterpret_cast<uint32_t*>(wpart()) + warp * M::KW;
        float2* ginfo = tc_ginfo<M>();
        float x[PL];
        float mx = 0.f;
#pragma unroll
        for (int c = 0; c < PL; ++c) {
            x[c] = gain ? gl[c] * v[0][c] : v[0][c];
            mx = fmaxf(mx, fabsf(x[c]));
        }
#pragma unroll
        for (int o = 1; o < LPG; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float qs = mx > 0.f ? 127.f / mx : 0.f;
        // round-to-nearest through the 1.5 * 2^23 magic: (y + M) holds
        // rint(y) in its low mantissa bits (two's complement in the low byte)
        // and (y + M) - M is rint(y) as a float; sums of the terms in f32
        // (exact: |sum| <= 127 * 128)
        constexpr float kM = 12582912.f;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f;
        uint32_t t0[PL / 4], t1[PL / 4], t2[PL / 4];
#pragma unroll
        for (int c4 = 0; c4 < PL; c4 += 4) {
            uint32_t m0[4], m1[4], m2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float y = x[c4 + e] * qs;
                const float a0 = y + kM, f0 = a0 - kM;
                const float r1 = (y - f0) * 254.f;
                const float a1 = r1 + kM, f1 = a1 - kM;
                const float r2 = (r1 - f1) * 254.f;
                const float a2 = r2 + kM, f2 = a2 - kM;
                s0 += f0;
                s1 += f1;
                s2 += f2;
                m0[e] = __float_as_uint(a0);
                m1[e] = __float_as_uint(a1);
                m2[e] = __float_as_uint(a2);
            }
            auto pack4 = [](const uint32_t (&m)[4]) {  // the four low bytes
                return __byte_perm(__byte_perm(m[0], m[1], 0x0040), __byte_perm(m[2], m[3], 0x0040), 0x5410);
            };
            t0[c4 / 4] = pack4(m0);
            t1[c4 / 4] = pack4(m1);
            t2[c4 / 4] = pack4(m2);
        }
#pragma unroll
        for (int jj = 0; jj < PL / 16; ++jj) {
            const int hs = lane * (PL / 16) + jj, st = hs / 2, h = hs % 2;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                tab[st * 32 + 0 * 8 + qq * 2 + h] = t0[jj * 4 + qq];
                tab[st * 32 + 1 * 8 + qq * 2 + h] = t1[jj * 4 + qq];
                tab[st * 32 + 2 * 8 + qq * 2 + h] = t2[jj * 4 + qq];
            }
        }
#pragma unroll
        for (int o = 1; o < LPG; o <<= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (lane % LPG == 0)
            ginfo[warp * (M::KW / kQuantGroup) + lane / LPG] =
                make_float2(mx / 127.f, s0 + s1 * (1.f / 254.f) + s2 * (1.f / 64516.f));
        consumer_sync(NCT);  // tables (and the norm partials) complete before any warp's first MMA
        act.sum[0] = 1.f;  // the row's 1/rms (1 without a gain): scales every group's dq in tc_slot
        if (gain != nullptr) {
            float t = 0.f;
            for (int w = 0; w < NCW; ++w) t += ns[w * B];
            act.sum[0] = 1.0f / sqrtf(t / static_cast<float>(M::K) + p.eps);
        }
    }

    // per-group (dq, zero-point sum) of the TC activation tables
    template <class M>
    __device__ float2* tc_ginfo() {
        return reinterpret_cast<float2*>(reinterpret_cast<uint32_t*>(wpart()) + NCW * M::KW);
    }

    // u8 codes x s8 activation terms, exact s32 accumulation
    __device__ static void mma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                    uint32_t b0, uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }

    __device__ static void mma_f16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                   uint32_t a3, uint32_t b0, uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }

    // fp16 magic decode: (w & mask) | 0x6400 per half = 1024 + code (int4
    // nibbles at bits 4..7 / 20..23 come out as 1024 + 16 code), then one
    // HSUB2 of (1024 + zero) leaves (code - zero) exactly.
    template <uint32_t MASK>
    __device__ static uint32_t f16_nib(uint32_t w) {
        uint32_t r;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "n"(MASK), "r"(0x64006400u));
        return r;
    }

    __device__ static uint32_t hsub2_u(uint32_t a, uint32_t b) {
        __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
        return *reinterpret_cast<uint32_t*>(&r);
    }

    // One 16-row (int4) / 8-row (int8) slot of a TC matrix against this
    // warp's K range: per 128-column group, the codes of rows g and g + 8
    // (MMA code order, weight_layout_tc) go straight into m16n8k32 u8 A
    // fragments (int4: one LOP3 per 4 codes, int8: as loaded), four MMAs
    // against the three int8 activation terms accumulate exactly in s32,
    // then per row: s * dq * ((t0 + t1/254 + t2/254^2) - z * sum), the
    // zero point folded through the group's activation sum.  out[0] / out[2]
    // = rows g / g + 8 (lanes q == 0), out[1] = out[3] = 0.
    template <class M>
    __device__ __forceinline__ void tc_slot(const uint8_t* base, float inv, float (&out)[4]) {
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32, g = lane / 4, q = lane % 4;
        const uint32_t* tab = reinterpret_cast<const uint32_t*>(wpart()) + warp * M::KW;
        const float2* ginfo = tc_ginfo<M>() + warp * (M::KW / kQuantGroup);
        auto frag = [&](int st) {  // (reg 0, reg 1) of k32-step st for column g (terms 0..2)
            return g < 3 ? *reinterpret_cast<const uint2*>(tab + st * 32 + g * 8 + q * 2) : make_uint2(0u, 0u);
        };
        const uint8_t* rA = base + g * M::ROW_BYTES;
        const uint8_t* rB = base + (g + 8) * M::ROW_BYTES;
#pragma unroll
        for (int e = 0; e < 4; ++e) out[e] = 0.f;
#pragma unroll 2
        for (int gi = 0; gi < M::KW / kQuantGroup; ++gi) {
            const int G = warp * (M::KW / kQuantGroup) + gi;  // group index in the row
            const float sA = *reinterpret_cast<const float*>(rA + M::CODE_BYTES + 4 * G);
            const float zA = static_cast<float>(rA[M::CODE_BYTES + 4 * M::NG + G]);
            int acc[4] = {0, 0, 0, 0};
            if constexpr (M::QB == 4) {
                const uint4 wa = lds_u128(rA + G * 64 + q * 16);
                const uint4 wb = lds_u128(rB + G * 64 + q * 16);
                const uint32_t wA[4] = {wa.x, wa.y, wa.z, wa.w}, wB[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    const uint2 bf = frag(gi * 4 + st);
                    mma_u8s8(acc, wA[st] & 0x0F0F0F0Fu, wB[st] & 0x0F0F0F0Fu, (wA[st] >> 4) & 0x0F0F0F0Fu,
                             (wB[st] >> 4) & 0x0F0F0F0Fu, bf.x, bf.y);
                }
            } else {  // int8: 8 real rows (g), rows g + 8 zero
                const uint4 w0 = lds_u128(rA + G * 128 + q * 32);
                const uint4 w1 = lds_u128(rA + G * 128 + q * 32 + 16);
                const uint32_t wA[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    const uint2 bf = frag(gi * 4 + st);
                    mma_u8s8(acc, wA[2 * st], 0u, wA[2 * st + 1], 0u, bf.x, bf.y);
                }
            }
            // terms 0, 1 in lane q = 0 (columns 0, 1), term 2 in lane q = 1
            const int t2A = __shfl_down_sync(0xffffffffu, acc[0], 1);
            const int t2B = __shfl_down_sync(0xffffffffu, acc[2], 1);
            const float2 gf = ginfo[gi];
            const float dq = gf.x * inv;
            const float xA = fmaf(static_cast<float>(t2A), 1.f / 64516.f,
                                  fmaf(static_cast<float>(acc[1]), 1.f / 254.f, static_cast<float>(acc[0])));
            out[0] = fmaf(sA * dq, fmaf(-zA, gf.y, xA), out[0]);
            if constexpr (M::QB == 4) {
                const float sB = *reinterpret_cast<const float*>(rB + M::CODE_BYTES + 4 * G);
                const float zB = static_cast<float>(rB[M::CODE_BYTES + 4 * M::NG + G]);
                const float xB = fmaf(static_cast<float>(t2B), 1.f / 64516.f,
                                      fmaf(static_cast<float>(acc[3]), 1.f / 254.f, static_cast<float>(acc[2])));
                out[2] = fmaf(sB * dq, fmaf(-zB, gf.y, xB), out[2]);
            } else {
                (void)t2B;
            }
        }
    }

    // Load the activations (RMSNorm'd with `gain` when given,
    // numerics.hpp:14-24).  src_emb: layer-0 input straight from the bf16
    // embedding.  Gains are constants, fetched before the dependency wait.
    template <class M = MD>
    __device__ __forceinline__ void load_act(Act<M>& act, const float* src, bool from_emb, const float* gain,
                             int stage) {
        if constexpr (M::TC) {
            load_act_tc<M>(act, src, from_emb, gain, stage);
            return;
        }
        const int ctid = threadIdx.x, lt = ctid % M::TPR, rg = ctid / M::TPR;
        float g[M::NCH][8];
        if (gain != nullptr) {
#pragma unroll
            for (int j = 0; j < M::NCH; ++j) {
                const int col = col_of<M>(lt, j);
                const float4 g0 = __ldg(reinterpret_cast<const float4*>(gain + col));
                const float4 g1 = __ldg(reinterpret_cast<const float4*>(gain + col + 4));
                g[j][0] = g0.x; g[j][1] = g0.y; g[j][2] = g0.z; g[j][3] = g0.w;
                g[j][4] = g1.x; g[j][5] = g1.y; g[j][6] = g1.z; g[j][7] = g1.w;
            }
        }
        wait_stage(stage);
#pragma unroll
        for (int b = 0; b < B; ++b) {
#pragma unroll
            for (int j = 0; j < M::NCH; ++j) {
                const int col = col_of<M>(lt, j);
                float* a = act.v[b][j];
                if (from_emb) {
                    const __nv_bfloat16* e = p.embedding + (size_t)token_row(p, b) * D + col;
                    const uint4 w = __ldg(reinterpret_cast<const uint4*>(e));
                    a[0] = bf_lo(w.x); a[1] = bf_hi(w.x); a[2] = bf_lo(w.y); a[3] = bf_hi(w.y);
                    a[4] = bf_lo(w.z); a[5] = bf_hi(w.z); a[6] = bf_lo(w.w); a[7] = bf_hi(w.w);
                } else {
                    const float4 a0 = ldcg_f4(src + (size_t)b * M::K + col);
                    const float4 a1 = ldcg_f4(src + (size_t)b * M::K + col + 4);
                    a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
                    a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
                }
            }
        }
        if (gain != nullptr) {
            float ss[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                float s = 0.f;
                if (rg == 0) {
#pragma unroll
                    for (int j = 0; j < M::NCH; ++j)
#pragma unroll
                        for (int e = 0; e < 8; ++e) s = fmaf(act.v[b][j][e], act.v[b][j][e], s);
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
                inv[b] = 1.0f / sqrtf(t / static_cast<float>(M::K) + p.eps);
            }
            consumer_sync(NCT);  // ns reusable afterwards
#pragma unroll
            for (int j = 0; j < M::NCH; ++j)
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                    for (int e = 0; e < 8; ++e) act.v[b][j][e] = g[j][e] * act.v[b][j][e] * inv[b];
        }
        if constexpr (M::QB != 0) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
                float t = 0.f;
#pragma unroll
                for (int j = 0; j < M::NCH; ++j)
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        t += act.v[b][j][e];
                        if constexpr (M::QB == 4) act.v[b][j][e] *= q4_scale(e);
                    }
                act.sum[b] = t;
            }
        }
    }

    // ---- quantized row decode (fused dequant) -------------------------
    // Codes become exact f32 integers with the 2^23 magic: OR the code into
    // the mantissa of 2^23, subtract 2^23 (packed FADD2).  int4: 8 nibbles
    // of a word -> c * 16^k (see q4_scale); int8: PRMT one byte per value.
    // (w & mask) | magic in ONE LOP3 (magic in a register; the compiler
    // otherwise splits the two immediates into two LOP3s)
    template <uint32_t MASK>
    __device__ static float q4_nib(uint32_t w, uint32_t magic) {
        uint32_t r;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "n"(MASK), "r"(magic));
        return __uint_as_float(r);
    }

    __device__ static void q4_decode(uint32_t w, float2 (&d)[4]) {
        const uint32_t M = 0x4B000000u;
        const float2 m2 = make_float2(-8388608.f, -8388608.f);
        const uint32_t h = w >> 20;
        d[0] = __fadd2_rn(make_float2(q4_nib<0xFu>(w, M), q4_nib<0xF0u>(w, M)), m2);
        d[1] = __fadd2_rn(make_float2(q4_nib<0xF00u>(w, M), q4_nib<0xF000u>(w, M)), m2);
        d[2] = __fadd2_rn(make_float2(q4_nib<0xF0000u>(w, M), q4_nib<0xFu>(h, M)), m2);
        d[3] = __fadd2_rn(make_float2(q4_nib<0xF0u>(h, M), q4_nib<0xF00u>(h, M)), m2);
    }

    __device__ static void q8_decode(uint32_t w, float2 (&d)[2]) {
        const float2 m2 = make_float2(-8388608.f, -8388608.f);
        d[0] = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440)),
                                      __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7441))), m2);
        d[1] = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(w, 0x4B000000u, 0x7442)),
                                      __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7443))), m2);
    }

    // This thread's codes of one quantized row (NCH chunks of 8 columns),
    // its group's scale and zero point.
    template <class M = MD>
    struct QRow {
        uint32_t w[M::QB == 4 ? M::NCH : 2 * M::NCH];
        float scale, zero;
    };

    template <class M = MD>
    __device__ static void q_load(const uint8_t* rowp, int lt, QRow<M>& q) {
        constexpr int NW = M::QB == 4 ? M::NCH : 2 * M::NCH;  // 32-bit code words
        const uint8_t* cp = rowp + lt * (NW * 4);
        if constexpr (NW == 4) {
            const uint4 v = lds_u128(cp);
            q.w[0] = v.x; q.w[1] = v.y; q.w[2] = v.z; q.w[3] = v.w;
        } else if constexpr (NW == 2) {
            const uint2 v = lds_u64(cp);
            q.w[0] = v.x; q.w[1] = v.y;
        } else if constexpr (NW == 1) {
            q.w[0] = lds_u32(cp);
        } else {
#pragma unroll
            for (int i = 0; i < NW; i += 4) {
                const uint4 v = lds_u128(cp + 4 * i);
                q.w[i] = v.x; q.w[i + 1] = v.y; q.w[i + 2] = v.z; q.w[i + 3] = v.w;
            }
        }
        const int g = (lt * M::CPT) / kQuantGroup;
        q.scale = *reinterpret_cast<const float*>(rowp + M::CODE_BYTES + 4 * g);
        q.zero = static_cast<float>(rowp[M::CODE_BYTES + 4 * M::NG + g]);
    }

    // decoded 8-column chunk ci of a quantized row: d[k] = columns (2k, 2k+1)
    // as exact f32 integers (int4: times the powers of 16 of q4_scale)
    template <class M>
    __device__ static void q_chunk(const QRow<M>& q, int ci, float2 (&d)[4]) {
        if constexpr (T::QB == 4) {
            q4_decode(q.w[ci], d);
        } else {
            float2 lo[2], hi[2];
            q8_decode(q.w[2 * ci], lo);
            q8_decode(q.w[2 * ci + 1], hi);
            d[0] = lo[0]; d[1] = lo[1]; d[2] = hi[0]; d[3] = hi[1];
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

    // V (power of two <= 32) per-lane values -> lane l ends with the warp sum
    // of value index l >> (5 - log2 V): V-1 + 5-log2(V) shuffles instead of 5V.
    template <int V>
    __device__ static float reduce_multi(float (&v)[V], int lane) {
        static_assert(V >= 1 && V <= 32 && (V & (V - 1)) == 0, "V must be a power of two");
#pragma unroll
        for (int s = V / 2, o = 16; s >= 1; s >>= 1, o >>= 1) {
            const bool upper = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < s; ++i) {
                const float send = upper ? v[i] : v[i + s];
                const float keep = upper ? v[i + s] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        float r = v[0];
#pragma unroll
        for (int o = 16 / V; o >= 1; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        return r;
    }

    static constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }


    // Tensor-core GEMV over rows [r0, r1): per slot every warp runs tc_slot
    // on its K range, the hi/lo columns of each batch row are added (lane
    // pairs), and the per-warp row partials go to red[warp][row][b]; the
    // epilogue (same contract as gemv) sums the 8 warps (row_total).
    template <class M, class Epi>
    __device__ __forceinline__ void gemv_tc(uint32_t& it, const Act<M>& act, int r0, int r1, Epi&& epi) {
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32, g = lane / 4, q = lane % 4;
        int batch_c0 = r0;
        uint32_t nbatch = 0;
        float* red = red_buf(0);
        for (int c0 = r0; c0 < r1; c0 += M::RPS) {
            const int nrows = min(M::RPS, r1 - c0);
            const uint32_t slot = it % T::NSLOTS, par = (it / T::NSLOTS) & 1;
            wait_full(slot, par);
            float c[4];
            tc_slot<M>(ring + slot * T::SLOT_BYTES, act.sum[0], c);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            ++it;
            // columns 2q, 2q+1: batch rows (hi) or their lo parts; fold lo
            // into hi (partner lane q ^ B/2), B = 1 keeps both in one lane
            float v[4];
            if constexpr (B == 1) {
                v[0] = c[0] + c[1];
                v[2] = c[2] + c[3];
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = c[e] + __shfl_xor_sync(0xffffffffu, c[e], B / 2);
            }
            const int base_row = c0 - batch_c0;
            if constexpr (B == 1) {
                if (q == 0) {
                    if (g < nrows) red[(warp * M::RB + base_row + g) * B] = v[0];
                    if (g + 8 < nrows) red[(warp * M::RB + base_row + g + 8) * B] = v[2];
                }
            } else {
                if (q < B / 2) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int b = 2 * q + e;
                        if (g < nrows) red[(warp * M::RB + base_row + g) * B + b] = v[e];
                        if (g + 8 < nrows) red[(warp * M::RB + base_row + g + 8) * B + b] = v[2 + e];
                    }
                }
            }
            const int batch_rows = c0 + nrows - batch_c0;
            if (c0 + M::RPS >= r1 || batch_rows + M::RPS > M::RB) {
                consumer_sync(NCT);
                epi(batch_c0, batch_rows, red);
                batch_c0 = c0 + M::RPS;
                red = red_buf(++nbatch);
            }
        }
    }

    // GEMV over rows [r0, r1) streamed by the producer.  Per slot every warp
    // forms its column-slice partial dots for all RPT x B (row, batch) values
    // (two accumulators per row, no per-row branches), releases the slot, and
    // folds the values with one transposed warp reduction into
    // red[wr][row][b].  Warps never wait for each other inside a batch of RB
    // rows; `epi(c0, nrows, red)` runs once per batch after one named barrier
    // (red is double-buffered across batches).
    template <class M = MD, class Epi>
    __device__ __forceinline__ void gemv(uint32_t& it, const Act<M>& act, int r0, int r1, Epi&& epi) {
        if constexpr (M::TC) {
            gemv_tc<M>(it, act, r0, r1, epi);
            return;
        }
        constexpr int V = M::RPT * B, LV = ilog2(V);
        const int ctid = threadIdx.x, lane = ctid % 32;
        const int rg = ctid / M::TPR, lt = ctid % M::TPR, wr = lt / 32;
        const int vidx = lane >> (5 - LV), vr = vidx / B, vb = vidx % B;
        const bool writer = (lane & ((32 >> LV) - 1)) == 0;
        int batch_c0 = r0;
        uint32_t nbatch = 0;
        float* red = red_buf(0);
        for (int c0 = r0; c0 < r1; c0 += M::RPS) {
            const int nrows = min(M::RPS, r1 - c0);
            const uint32_t slot = it % T::NSLOTS, par = (it / T::NSLOTS) & 1;
            wait_full(slot, par);
            const uint8_t* base = ring + slot * T::SLOT_BYTES;
            float v[V];
#pragma unroll
            for (int r = 0; r < M::RPT; ++r) {
                // rows past nrows read stale (valid) smem; their sums are dropped
                const uint8_t* rowp = base + (rg + r * M::RG) * M::ROW_BYTES;
                if constexpr (M::QB != 0) {  // fused dequant: s * (sum c a - z sum a)
                    QRow<M> q;
                    q_load(rowp, lt, q);
                    float2 acc[B][4];  // 4 independent FFMA2 chains per batch row
#pragma unroll
                    for (int b = 0; b < B; ++b)
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[b][k] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < M::NCH; ++j) {
                        float2 d[4];
                        q_chunk(q, j, d);
#pragma unroll
                        for (int b = 0; b < B; ++b) {
                            const float* a = act.v[b][j];
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                acc[b][k] = __ffma2_rn(d[k], make_float2(a[2 * k], a[2 * k + 1]),
                                                       acc[b][k]);
                        }
                    }
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const float2 t = __fadd2_rn(__fadd2_rn(acc[b][0], acc[b][1]),
                                                    __fadd2_rn(acc[b][2], acc[b][3]));
                        v[r * B + b] = q.scale * ((t.x + t.y) - q.zero * act.sum[b]);
                    }
                    continue;
                }
                // packed f32x2 FMAs on (even, odd) column pairs: one FFMA2
                // per two weights and batch row; two chains per batch row
                float2 a0[B], a1[B];
#pragma unroll
                for (int b = 0; b < B; ++b) a0[b] = a1[b] = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < M::VPT; ++j) {
                    const uint4 w = lds_u128(rowp + (lt + j * M::TPR) * 16);
                    const float2 w0 = make_float2(bf_lo(w.x), bf_hi(w.x));
                    const float2 w1 = make_float2(bf_lo(w.y), bf_hi(w.y));
                    const float2 w2 = make_float2(bf_lo(w.z), bf_hi(w.z));
                    const float2 w3 = make_float2(bf_lo(w.w), bf_hi(w.w));
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const float(&a)[8] = act.v[b][j];
                        a0[b] = __ffma2_rn(w0, make_float2(a[0], a[1]), a0[b]);
                        a1[b] = __ffma2_rn(w1, make_float2(a[2], a[3]), a1[b]);
                        a0[b] = __ffma2_rn(w2, make_float2(a[4], a[5]), a0[b]);
                        a1[b] = __ffma2_rn(w3, make_float2(a[6], a[7]), a1[b]);
                    }
                }
#pragma unroll
                for (int b = 0; b < B; ++b) v[r * B + b] = (a0[b].x + a1[b].x) + (a0[b].y + a1[b].y);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            const float s = reduce_multi<V>(v, lane);
            const int row = rg + vr * M::RG;
            if (writer && row < nrows) red[(wr * M::RB + (c0 - batch_c0) + row) * B + vb] = s;
            ++it;
            const int batch_rows = c0 + nrows - batch_c0;
            if (c0 + M::RPS >= r1 || batch_rows + M::RPS > M::RB) {
                consumer_sync(NCT);
                epi(batch_c0, batch_rows, red);
                batch_c0 = c0 + M::RPS;
                red = red_buf(++nbatch);
            }
        }
    }

    template <class M = MD>
    __device__ static float row_total(const float* red, int row, int b) {
        float t = 0.f;
#pragma unroll
        for (int w = 0; w < M::EWPR; ++w) t += red[(w * M::RB + row) * B + b];
        return t;
    }

    // ================================================ batch >= 8 (KCP)
#ifdef FFB_KCP_TCGEN05
    // tcgen05 operand layouts:
    //  * A table (activations, the MMA's A operand): per K chunk of KC
    //    columns, [KC / 8 units][32 rows][16 B] -- 8 x 16-byte core matrices
    //    -- copied into TMEM columns [4u, 4u + 4) of lanes 0-31 (replicated to
    //    all 128 lanes) by tcgen05.cp.32x128b.warpx4; row m = t * 16 + b
    //    holds term t (0: fp16 hi, 1: fp16 lo) of batch row b (rows b >= B
    //    stay zero)
    //  * weights (B operand, N = RW rows per slot, K-major, 128-byte
    //    swizzle: 8-row x 128-byte atoms, 16-byte unit u of row r at u ^
    //    (r & 7)): [K / KC][rows / 8][KC / 64][8 rows][128 B] (runtime
    //    packer, layout 3): a slot of rows is one contiguous copy, atom
    //    column j of it at j * 1 KiB with KC / 64 KiB between 8-row groups
    __device__ static size_t frag_off(int k, int m) {
        const int c = k / S::KC, kk = k % S::KC;
        return (size_t)c * MD::ATAB + (kk >> 3) * 512 + m * 16 + (kk & 7) * 2;
    }
#else
    // A-fragment table offset of activation column k, batch row b (m16n8k16
    // row-major A: lane (g, q) holds rows g / g + 8, columns 2q, 2q + 1 and
    // 2q + 8, 2q + 9 of each k16 step; registers a0..a3 = (g, lo k), (g + 8,
    // lo k), (g, hi k), (g + 8, hi k)); per k-step the 32 lanes' hi parts
    // (16 bytes each, conflict-free LDS.128) then the lo parts (+512).
    __device__ static size_t frag_off(int k, int b) {
        const int kst = k >> 4, kk = k & 15;
        const int lane = (b & 7) * 4 + ((kk & 7) >> 1);
        const int reg = (kk >> 3) * 2 + (b >> 3);
        return (size_t)kst * 1024 + lane * 16 + reg * 4 + (kk & 1) * 2;
    }
#endif
    // v as fp16 hi + lo (22 bits of mantissa); the bf16 weights are stored as
    // fp16 by the packer.  |v| beyond the fp16 range latches err_flag bit 1
    // (reported as FFB_NUMERIC by the next synchronous call) instead of
    // silently turning into inf.
    __device__ void frag_put(uint8_t* tab, int k, int b, float v) const {
        const __half hi = __float2half_rn(v);
        const __half lo = __float2half_rn(v - __half2float(hi));
        if (!(fabsf(v) <= 65504.f)) atomicOr(p.err_flag, 2u);
#ifdef FFB_KCP_TCGEN05
        *reinterpret_cast<__half*>(tab + frag_off(k, b)) = hi;
        *reinterpret_cast<__half*>(tab + frag_off(k, 16 + b)) = lo;
#else
        uint8_t* d = tab + frag_off(k, b);
        *reinterpret_cast<__half*>(d) = hi;
        *reinterpret_cast<__half*>(d + 512) = lo;
#endif
    }
    // After this CTA updated x rows [c0, c1): their A-table entries x * gain
    // and this CTA's per-batch-row sum of squares (ssq_out[cta][b]).  Ends
    // with a proxy fence: the tables are read by TMA (async proxy).
    __device__ void kc_publish(int c0, int c1, const float* gain, uint8_t* tab, float* ssq_out) {
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32;
        static_assert(kNCT % B == 0, "a thread's batch row is fixed");
        float sq = 0.f;
        for (int i = ctid; i < (c1 - c0) * B; i += NCT) {
            const int c = c0 + i / B, b = i % B;
            const float v = ldcg_f(p.x + (size_t)b * D + c);
            sq = fmaf(v, v, sq);
            frag_put(tab, c, b, v * __ldg(gain + c));
        }
#pragma unroll
        for (int off = B; off < 32; off <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
        float* ns = norm_s();
        if (lane < B) ns[warp * B + lane] = sq;
        fence_proxy_async_global();
        consumer_sync(NCT);
        if (ctid < B) {
            float t = 0.f;
            for (int w = 0; w < NCW; ++w) t += ns[w * B + ctid];
            __stcg(ssq_out + (size_t)cta * B + ctid, t);
        }
        consumer_sync(NCT);
    }

    // 1 / rms of every batch row from the CTAs' sums of squares (fixed order)
    // -> norm_s()[NCW * B + b]
    __device__ const float* kc_inv(const float* ssq_in) {
        float* inv = norm_s() + NCW * B;
        if (threadIdx.x < B) {
            float t = 0.f;
            for (int c = 0; c < grid; ++c) t += ldcg_f(ssq_in + (size_t)c * B + threadIdx.x);
            inv[threadIdx.x] = 1.0f / sqrtf(t / static_cast<float>(D) + p.eps);
        }
        consumer_sync(NCT);
        return inv;
    }

#ifdef FFB_KCP_TCGEN05
    // K-chunked tcgen05 GEMV, rows [r0, r1) (8-aligned), in row blocks of
    // KC_BLOCK: per K chunk the ring delivers the A table (activations of
    // all batch rows, fp16 hi / lo) then weight slots of RW rows.  One lane
    // of warp 0 copies the A table into TMEM (tcgen05.cp; the ring slot is
    // released as soon as the copies complete) and issues, per weight slot,
    // the chunk's KC / 16 MMAs (A from TMEM, M = 128: the 32 table rows
    // replicated four times; B = the slot's RW weight rows from shared
    // memory, K = 16) into that slot's TMEM accumulator columns,
    // accumulating across K chunks; a tcgen05.commit releases each weight
    // slot once its MMAs have read it (copies and MMAs execute in issue
    // order, so the next chunk's copy cannot overtake them).  The epilogue
    // (warps 0 and 4: TMEM lanes 0-31) adds the hi and lo rows, scales by
    // inv[b] (normed inputs) and hands 16-row groups to epi(c0, nrows,
    // red[row][b]) like gemv's epilogues.  The MMA's f32 accumulation order
    // is fixed by the hardware: deterministic.
    template <class M, class Epi>
    __device__ void gemv_kc(uint32_t& it, int r0, int r1, const float* inv, Epi&& epi) {
        constexpr int RW = M::RW, NKA = S::KC / 64;
        constexpr uint32_t IDESC = umma_idesc_f16(128, RW);
        static_assert(RW % 16 == 0 && RW <= 256 && S::KC % 64 == 0 && S::KC / 2 <= TM_A, "UMMA tile");
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32;
        float* fin = reinterpret_cast<float*>(smem + T::OFF_RED);  // [2][32][B] finished rows
        static_assert(2 * 32 * B <= 2 * T::RED_FLOATS && RW % 32 == 0, "epilogue staging");
        const uint32_t tbase = tmem_base();
        for (int blk = r0; blk < r1; blk += KC_BLOCK) {
            const int blk_end = min(blk + KC_BLOCK, r1);
            const int nj = (blk_end - blk + RW - 1) / RW;
            if (warp == 0) {
                for (int c = 0; c < M::NKC; ++c) {
                    const uint32_t sa = it % T::NSLOTS;
                    wait_full(sa, (it / T::NSLOTS) & 1);
                    ++it;
                    // the previous chunk's MMAs have read the TMEM A buffer
                    if (a_issued) {
                        mbar_wait(abar(), a_phase & 1);
                        ++a_phase;
                        tc05_fence_after();
                    }
                    {  // lane m: its A-table row of the chunk -> TMEM lane m, columns [0, KC / 2)
                        const uint8_t* arow = ring + sa * T::SLOT_BYTES + lane * 16;
#pragma unroll 1
                        for (int q = 0; q < S::KC / 128; ++q) {
                            uint32_t r[64];
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const uint4 v = lds_u128(arow + (q * 16 + u) * 512);
                                r[4 * u] = v.x; r[4 * u + 1] = v.y; r[4 * u + 2] = v.z; r[4 * u + 3] = v.w;
                            }
                            tmem_st_32x32b_x64(tbase + q * 64, r);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cnt(&empty[sa], NCW);  // A slot read: free
                    tc05_fence_before();
                    __syncwarp();
                    tc05_fence_after();
                    for (int j = 0; j < nj; ++j) {
                        const uint32_t sw = it % T::NSLOTS;
                        wait_full(sw, (it / T::NSLOTS) & 1);
                        ++it;
                        tc05_fence_after();
                        if (lane == 0) {
                            const uint32_t wbase = smem_u32(ring + sw * T::SLOT_BYTES);
#pragma unroll
                            for (int ka = 0; ka < NKA; ++ka)
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    umma_f16_ts(tbase + TM_A + j * RW, tbase + (ka * 4 + kk) * 8,
                                                umma_desc_sw128(wbase + ka * 1024 + kk * 32, NKA * 1024), IDESC,
                                                (c | ka | kk) != 0);
                            umma_commit(&empty[sw]);  // one arrival when these MMAs have read the slot
                            mbar_arrive_cnt(&empty[sw], NCW - 1);
                        }
                        __syncwarp();
                    }
                    if (lane == 0) umma_commit(abar());  // A buffer free once these MMAs are done
                    a_issued = true;
                }
                if (lane == 0) umma_commit(accbar());
                __syncwarp();
            } else {
                it += M::NKC * (1 + nj);  // the same slots, consumed by warp 0
            }
            const bool reader = warp == 0 || warp == 4;
            if (reader) {
                mbar_wait(accbar(), acc_phase & 1);
                tc05_fence_after();
            }
            ++acc_phase;
            // 32-row tiles of the block's accumulators (32 TMEM columns each),
            // two at a time: warp 0 the even tile, warp 4 the odd one
            const int ntile = (blk_end - blk + 31) / 32;
            for (int t0 = 0; t0 < ntile; t0 += 2) {
                const int t = t0 + warp / 4;
                if (reader && t < ntile) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tbase + TM_A + t * 32, r);  // lane l: D[row l][cols t * 32 ..]
                    float* f = fin + (warp / 4) * 32 * B;
#pragma unroll
                    for (int n = 0; n < 32; ++n) {
                        float v = __uint_as_float(r[n]);
                        v += __shfl_down_sync(0xffffffffu, v, 16);  // hi row b + lo row 16 + b
                        if (lane < B) f[n * B + lane] = inv != nullptr ? v * inv[lane] : v;
                    }
                }
                consumer_sync(NCT);
                for (int tt = t0; tt < min(t0 + 2, ntile); ++tt) {
                    const int g0 = blk + tt * 32, nrows = min(32, blk_end - g0);
                    for (int e0 = 0; e0 < nrows; e0 += 16)
                        epi(g0 + e0, min(16, nrows - e0), fin + ((tt - t0) * 32 + e0) * B);
                }
                consumer_sync(NCT);
            }
            if (reader) tc05_fence_before();  // TMEM reads done before the next block's MMAs
        }
    }

#else
    // K-chunked tensor-core GEMV, rows [r0, r1), in row blocks of KC_BLOCK:
    // per K chunk the ring delivers the A table (activations of all batch
    // rows, fp16 hi/lo) then weight slots of RW rows; warp (rp, kp) runs the
    // mma.sync m16n8k16 of its two n8 row tiles over its 8 k-steps into
    // per-block accumulators (M = batch: the 16 MMA rows are the batch
    // rows).  At the block end the KP k-part partials are summed in a fixed
    // order (deterministic), scaled by inv[b] (normed inputs) and handed to
    // epi(c0, nrows <= 16, red[row][b]) like gemv's epilogues (EWPR = 1).
    template <class M, class Epi>
    __device__ void gemv_kc(uint32_t& it, int r0, int r1, const float* inv, Epi&& epi) {
        constexpr int RW = M::RW, NJ = KC_BLOCK / RW;
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32, g = lane / 4, q4 = lane % 4;
        const int rp = warp % M::RP, kp = warp / M::RP;
        float* R = reinterpret_cast<float*>(smem + T::OFF_RED);  // [KP][RW][B]
        float* fin = R + M::KP * RW * B;                          // [RW][B]
        // this lane's ldmatrix row (two n8 tiles x two k halves) in a weight
        // slot; 16-byte unit u of a row segment sits at u ^ (matrix row & 7)
        const int lrow = rp * 16 + (lane >> 4) * 8 + (lane & 7);
        const int lhalf = (lane >> 3) & 1;
        for (int blk = r0; blk < r1; blk += KC_BLOCK) {
            const int blk_end = min(blk + KC_BLOCK, r1);
            const int nj = (blk_end - blk + RW - 1) / RW;
            float acc[NJ][2][4];
#pragma unroll
            for (int j = 0; j < NJ; ++j)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[j][nt][e] = 0.f;
            for (int c = 0; c < M::NKC; ++c) {
                uint4 afh[8], afl[8];
                const uint32_t sa = it % T::NSLOTS;
                wait_full(sa, (it / T::NSLOTS) & 1);
                const uint8_t* atab = ring + sa * T::SLOT_BYTES + kp * 8 * 1024 + lane * 16;
                ++it;
                // this warp's A fragments of the chunk into registers, then the
                // A-table slot is released: the ring refills it with weights
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    afh[ks] = lds_u128(atab + ks * 1024);
                    afl[ks] = lds_u128(atab + ks * 1024 + 512);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[sa]);
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    if (j < nj) {
                        const uint32_t sw = it % T::NSLOTS;
                        wait_full(sw, (it / T::NSLOTS) & 1);
                        const uint8_t* wrow = ring + sw * T::SLOT_BYTES + lrow * M::SEG;
                        const int key = (blk + j * RW + lrow) & 7;
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks) {
                            const uint4 ah = afh[ks];
                            const uint4 al = afl[ks];
                            uint32_t b0, b1, b2, b3;
                            ldsm_x4(wrow + ((((kp * 8 + ks) * 2 + lhalf) ^ key) << 4), b0, b1, b2, b3);
                            mma_f16(acc[j][0], ah.x, ah.y, ah.z, ah.w, b0, b1);
                            mma_f16(acc[j][1], ah.x, ah.y, ah.z, ah.w, b2, b3);
                            mma_f16(acc[j][0], al.x, al.y, al.z, al.w, b0, b1);
                            mma_f16(acc[j][1], al.x, al.y, al.z, al.w, b2, b3);
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[sw]);
                        ++it;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                if (j < nj) {
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int row = rp * 16 + nt * 8 + 2 * q4 + (e & 1);
                            const int b = g + 8 * (e >> 1);
                            if (b < B) R[(kp * RW + row) * B + b] = acc[j][nt][e];
                        }
                    consumer_sync(NCT);
                    for (int i = ctid; i < RW * B; i += NCT) {
                        float t = 0.f;
#pragma unroll
                        for (int k = 0; k < M::KP; ++k) t += R[k * RW * B + i];
                        fin[i] = inv != nullptr ? t * inv[i % B] : t;
                    }
                    consumer_sync(NCT);
                    const int g0 = blk + j * RW, nrows = min(RW, blk_end - g0);
                    for (int e0 = 0; e0 < nrows; e0 += 16) epi(g0 + e0, min(16, nrows - e0), fin + e0 * B);
                    consumer_sync(NCT);
                }
            }
        }
    }

#endif

    // One GEMV stage's activation + rows: CUDA-core / quant path (load_act +
    // gemv) or, at batch >= 8, gemv_kc (inputs already in the A tables;
    // ssq_in = the sums of squares of a normed input, else nullptr).
    template <class M, class Epi>
    __device__ void run_gemv(uint32_t& it, const float* src, bool from_emb, const float* gain,
                             const float* ssq_in, int stage, int r0, int r1, Epi&& epi) {
        if constexpr (S::KCP) {
            wait_stage(stage);
            const float* inv = ssq_in != nullptr ? kc_inv(ssq_in) : nullptr;
            trace_mark(stage, 3);
            gemv_kc<M>(it, r0, r1, inv, epi);
        } else {
            Act<M> act;
            load_act<M>(act, src, from_emb, gain, stage);
            trace_mark(stage, 3);
            gemv<M>(it, act, r0, r1, epi);
        }
    }

    // ---------------------------------------------------------- S_QKV
    __device__ void stage_qkv(uint32_t& it, int l) {
        const float* rp = rope();
        const int ctid = threadIdx.x;
        run_gemv<MD>(it, p.x, l == 0, p.norm_attn + (size_t)l * D,
                     S::KCP ? p.ssq + (size_t)grid * B : nullptr, l * kStagesPerLayer + S_QKV,
                     pl.qkv_r0, pl.qkv_r1, [&](int c0, int nrows, const float* red) {
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
                        __nv_bfloat16* k_dst =
                            p.kcache + kv_row(l, b, h, p.pos) + kv_swz_dim(dim, p.pos);
                        __nv_bfloat162 kv2;
                        kv2.x = __float2bfloat16_rn(r0);
                        kv2.y = __float2bfloat16_rn(r1);
                        *reinterpret_cast<__nv_bfloat162*>(k_dst) = kv2;
                    }
                } else {
                    const int gv = g - QR - KR, h = gv / DH, dim = gv % DH;
                    __nv_bfloat16* v_dst =
                        p.vcache + kv_row(l, b, h, p.pos) + kv_swz_dim(dim, p.pos);
                    __nv_bfloat162 kv2;
                    kv2.x = __float2bfloat16_rn(a);
                    kv2.y = __float2bfloat16_rn(bb);
                    *reinterpret_cast<__nv_bfloat162*>(v_dst) = kv2;
                }
            }
        });
        // fine-grained release: one arrival per kv head whose rows this CTA
        // holds (S_ATTN of that head waits for exactly those CTAs)
        consumer_sync(NCT);
        if (threadIdx.x < S::NKV && ((pl.qkv_heads >> threadIdx.x) & 1))
            red_release_gpu(p.qkv_head_counters + l * S::NKV + threadIdx.x, 1);
        trace_mark(l * kStagesPerLayer + S_QKV, 2);
        trace_ring_wait(l * kStagesPerLayer + S_QKV);
    }

    // ---------------------------------------------------------- S_ATTN
    // Split-K flash-decoding (numerics.hpp:64-145).  A CTA's positions
    // [p0, p1) are consumed in passes of up to ATT_SC ring slots (plus the
    // current token in the last pass), three barriers per pass:
    //   A  scores: tensor-core K . (alpha log2e q) over 16-position tiles
    //   B  softmax: warp h takes the pass max, rescales its running (m, l)
    //      (online softmax across passes) and writes P (bf16 hi/lo rows)
    //   C  P.V on tensor cores, warp w owning dims [w DH/8, (w+1) DH/8)
    // K/V rows keep their 16-byte chunks XOR-swizzled by pos & 7, so the
    // per-lane ldmatrix row addresses are bank-conflict free.  At ctx 4096 on
    // the 8B shape a CTA owns ~228 positions: one pass.
    static constexpr int DC = DH / 8;   // 16-byte chunks per K/V row
    static constexpr int PG = NCT / DC;  // position groups in phase C
    static constexpr int ANP = T::ANP;
    static_assert(DC >= 8 && NCT % DC == 0, "attention mapping");
    static_assert(32 % DC == 0, "attention mapping: a position's chunks share one warp");
    static_assert(QPG <= DC, "attention score fold: QPG <= DH / 8");

    __device__ float* att_q() { return wpart(); }                 // [QPG][DH]
    __device__ float* att_sc() { return att_q() + QPG * DH; }     // [QPG][ANP]
    __device__ float* att_p() { return att_sc() + QPG * ANP; }    // [ANP][QPG]
    __device__ float* att_st() { return att_p() + ANP * (QPG > 8 ? QPG : 8); }  // [QPG][4] m l scale
    __device__ __nv_bfloat16* att_pt() { return reinterpret_cast<__nv_bfloat16*>(att_p()); }  // [16][ANP]

    // K (kv = 0) or V (kv = 1) row of pass position j: ring slot (it0 + j /
    // KVC) for j < nring, else the current token staged in h_s
    __device__ const uint8_t* att_row(uint32_t it0, int j, int nring, int kv) {
        if (j < nring) {
            const uint32_t slot = (it0 + j / T::KVC) % T::NSLOTS;
            return ring + slot * T::SLOT_BYTES + kv * (T::SLOT_BYTES / 2) + (j % T::KVC) * DH * 2;
        }
        return reinterpret_cast<const uint8_t*>(h_s()) + kv * DH * 2;
    }

    // ---- tensor-core attention pass (mma.sync m16n8k16 bf16, f32 accumulate)
    // GQA groups QPG query heads on one kv head, so the decode step is two
    // small contractions per pass: S[pos][h] = K[pos][:] . (alpha q_h) with
    // K tiles as A (ldmatrix from the swizzled ring rows) and q as B, and
    // O[h][dim] = P[h][pos] V[pos][dim] with P as A and V tiles as B
    // (ldmatrix.trans).  q and P enter as bf16 hi + lo (two MMA columns /
    // rows per head: 16 bits of mantissa), K and V are bf16 already.
    static constexpr int NTS = (2 * QPG + 7) / 8;  // score n-tiles (hi/lo columns)
    static constexpr int DPW = DH / NCW;           // P.V output dims per warp
    static constexpr int NTW = DPW / 8;            // P.V n-tiles per warp
    static_assert(2 * QPG <= 16 && DPW % 8 == 0 && (NTW == 1 || NTW == 2), "TC attention shape");

    __device__ static uint32_t bf2_pack(float lo_elem, float hi_elem) {
        __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
        return *reinterpret_cast<uint32_t*>(&v);
    }

    __device__ static void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                    uint32_t a3, uint32_t b0, uint32_t b1) {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }

    __device__ static void ldsm_x4(const void* p, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                   uint32_t& r3) {
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                     : "r"(smem_u32(p)));
    }

    __device__ static void ldsm_x4_t(const void* p, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                     uint32_t& r3) {
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                     : "r"(smem_u32(p)));
    }

    __device__ static void ldsm_x2_t(const void* p, uint32_t& r0, uint32_t& r1) {
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                     : "=r"(r0), "=r"(r1)
                     : "r"(smem_u32(p)));
    }

    // o[NTW][4]: this warp's P.V accumulator (rows = heads hi/lo, columns =
    // its dims), carried across passes (online softmax rescale per row).
    __device__ void attn_pass_tc(uint32_t it0, int nring, int n, int pos0, float (&o)[NTW][4]) {
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32, g = lane / 4, q4 = lane % 4;
        float* sc = att_sc();
        const float* qs = att_q();
        float* st = att_st();
        __nv_bfloat16* pt = att_pt();
        const int ntiles = (n + 15) / 16;
        {  // A: scores, warps over 16-position tiles
            uint32_t qb[DH / 16][NTS][2];  // q B fragments (column = head hi / lo)
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)
#pragma unroll
                for (int nt = 0; nt < NTS; ++nt) {
                    const int col = nt * 8 + g;
                    const int h = col % QPG;
                    const bool live = col < 2 * QPG, lo = col >= QPG;
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const int d = kk * 16 + 2 * q4 + 8 * r;
                        uint32_t v = 0u;
                        if (live) {
                            const float x0 = qs[h * DH + d], x1 = qs[h * DH + d + 1];
                            if (lo) {
                                const float h0 = __bfloat162float(__float2bfloat16_rn(x0));
                                const float h1 = __bfloat162float(__float2bfloat16_rn(x1));
                                v = bf2_pack(x0 - h0, x1 - h1);
                            } else {
                                v = bf2_pack(x0, x1);
                            }
                        }
                        qb[kk][nt][r] = v;
                    }
                }
            for (int t = warp; t < ntiles; t += NCW) {
                // this lane's ldmatrix row: position t*16 + (lane & 7) + 8 * ((lane >> 3) & 1)
                const int jr = min(t * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), n - 1);
                const uint8_t* row = att_row(it0, jr, nring, 0);
                const int key = (pos0 + jr) & 7;
                float c[NTS][4];
#pragma unroll
                for (int nt = 0; nt < NTS; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) c[nt][e] = 0.f;
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4(row + (((2 * kk + (lane >> 4)) ^ key) << 4), a0, a1, a2, a3);
#pragma unroll
                    for (int nt = 0; nt < NTS; ++nt)
                        mma_bf16(c[nt], a0, a1, a2, a3, qb[kk][nt][0], qb[kk][nt][1]);
                }
                // C[pos][col]: fold the lo column into the hi one
#pragma unroll
                for (int nt = 0; nt < NTS; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int col = nt * 8 + 2 * q4 + (e & 1);
                        const int j = t * 16 + g + 8 * (e >> 1);
                        if (QPG >= 4) {
                            // lo of column col sits at col + QPG: same n-tile for QPG = 4
                            // (lane q4 + 2), next n-tile for QPG = 8 (same lane)
                            float partner;
                            if constexpr (QPG == 8) partner = nt == 0 ? c[NTS - 1][e] : 0.f;
                            else partner = __shfl_xor_sync(0xffffffffu, c[nt][e], QPG / 2);
                            if (col < QPG && j < n) sc[col * ANP + j] = c[nt][e] + partner;
                        } else {  // QPG 2: lo columns 2, 3 at lane q4 + 1
                            const float partner = __shfl_xor_sync(0xffffffffu, c[nt][e], 1);
                            if (col < QPG && j < n) sc[col * ANP + j] = c[nt][e] + partner;
                        }
                    }
            }
        }
        consumer_sync(NCT);
        for (int h = warp; h < QPG; h += NCW) {  // B: online softmax of head h -> P hi/lo rows
            // 8 consecutive positions per lane (16-byte smem accesses), held
            // in registers between the max and the exp pass
            constexpr int PIT = (ANP + 255) / 256;
            float v[PIT][8];
            float cmax = -INFINITY;
#pragma unroll
            for (int i = 0; i < PIT; ++i) {
                const int j0 = i * 256 + lane * 8;
#pragma unroll
                for (int e = 0; e < 8; ++e) v[i][e] = -INFINITY;
                if (j0 < n) {
                    const float4 x0 = *reinterpret_cast<const float4*>(sc + h * ANP + j0);
                    const float4 x1 = *reinterpret_cast<const float4*>(sc + h * ANP + j0 + 4);
                    const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) v[i][e] = j0 + e < n ? xs[e] : -INFINITY;
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) cmax = fmaxf(cmax, v[i][e]);
            }
            cmax = warp_max(cmax);
            const float m_old = st[h * 4 + 0];
            const float m_new = fmaxf(m_old, cmax);
            const float scale = exp2f(m_old - m_new);  // 0 for the first pass
            float psum = 0.f;
#pragma unroll
            for (int i = 0; i < PIT; ++i) {
                const int j0 = i * 256 + lane * 8;
                if (j0 < ntiles * 16) {
                    uint32_t hw[4], lw[4];
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        const float p0 = j0 + e < n ? exp2f(v[i][e] - m_new) : 0.f;
                        const float p1 = j0 + e + 1 < n ? exp2f(v[i][e + 1] - m_new) : 0.f;
                        const __nv_bfloat16 h0 = __float2bfloat16_rn(p0), h1 = __float2bfloat16_rn(p1);
                        hw[e / 2] = bf2_pack(__bfloat162float(h0), __bfloat162float(h1));
                        lw[e / 2] = bf2_pack(p0 - __bfloat162float(h0), p1 - __bfloat162float(h1));
                        psum += p0 + p1;
                    }
                    *reinterpret_cast<uint4*>(pt + h * ANP + j0) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    *reinterpret_cast<uint4*>(pt + (QPG + h) * ANP + j0) =
                        make_uint4(lw[0], lw[1], lw[2], lw[3]);
                }
            }
            psum = warp_sum(psum);
            if (lane == 0) {
                st[h * 4 + 0] = m_new;
                st[h * 4 + 1] = st[h * 4 + 1] * scale + psum;
                st[h * 4 + 2] = scale;
            }
        }
        consumer_sync(NCT);
        {  // C: P.V, warp w owns dims [w DPW, (w+1) DPW) over every position
            const int r0 = g, r1 = g + 8;  // A rows (heads hi/lo) of this lane
            const float s0 = r0 < 2 * QPG ? st[(r0 % QPG) * 4 + 2] : 0.f;
            const float s1 = r1 < 2 * QPG ? st[(r1 % QPG) * 4 + 2] : 0.f;
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) {
                o[nt][0] *= s0;
                o[nt][1] *= s0;
                o[nt][2] *= s1;
                o[nt][3] *= s1;
            }
            const int c0 = warp * (DPW / 8);  // first 16-byte dim chunk of this warp
            // software-pipelined: tile t + 1's fragments are loaded before
            // tile t's MMAs; even / odd tiles accumulate into two sets (two
            // independent MMA chains)
            float o2[NTW][4];
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) o2[nt][e] = 0.f;
            struct Frag {
                uint32_t a[4], b[2 * NTW];
            };
            const uint8_t* cur_v = reinterpret_cast<const uint8_t*>(h_s()) + DH * 2;
            auto load = [&](int t, Frag& f) {
                const __nv_bfloat16* p0 = pt + r0 * ANP + t * 16 + 2 * q4;
                const __nv_bfloat16* p1 = pt + r1 * ANP + t * 16 + 2 * q4;
                f.a[0] = r0 < 2 * QPG ? *reinterpret_cast<const uint32_t*>(p0) : 0u;
                f.a[2] = r0 < 2 * QPG ? *reinterpret_cast<const uint32_t*>(p0 + 8) : 0u;
                f.a[1] = r1 < 2 * QPG ? *reinterpret_cast<const uint32_t*>(p1) : 0u;
                f.a[3] = r1 < 2 * QPG ? *reinterpret_cast<const uint32_t*>(p1 + 8) : 0u;
                // ldmatrix.trans rows: position t*16 + (lane & 7) + 8*((lane>>3)&1), chunk c0 + (lane>>4)
                const int jr = min(t * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), n - 1);
                const uint32_t slot = (it0 + jr / T::KVC) % T::NSLOTS;
                const uint8_t* rr = ring + slot * T::SLOT_BYTES + T::SLOT_BYTES / 2 + (jr % T::KVC) * DH * 2;
                const uint8_t* row = jr < nring ? rr : cur_v;  // (att_row, branch-free)
                const int key = (pos0 + jr) & 7;
                if constexpr (NTW == 2)
                    ldsm_x4_t(row + (((c0 + (lane >> 4)) ^ key) << 4), f.b[0], f.b[1], f.b[2], f.b[3]);
                else
                    ldsm_x2_t(row + ((c0 ^ key) << 4), f.b[0], f.b[1]);
            };
            auto mma_f = [&](const Frag& f, float (&acc)[NTW][4]) {
#pragma unroll
                for (int nt = 0; nt < NTW; ++nt)
                    mma_bf16(acc[nt], f.a[0], f.a[1], f.a[2], f.a[3], f.b[2 * nt], f.b[2 * nt + 1]);
            };
            Frag f0, f1;
            load(0, f0);
            int t = 0;
            for (; t + 2 <= ntiles; t += 2) {
                load(t + 1, f1);
                mma_f(f0, o);
                if (t + 2 < ntiles) load(t + 2, f0);
                mma_f(f1, o2);
            }
            if (t < ntiles) mma_f(f0, o);
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) o[nt][e] += o2[nt][e];
        }
        consumer_sync(NCT);  // sc / pt / stats reusable by the next pass
    }

    // ---- per-warp flash decoding (T::ATT_WARP) -------------------------
    // Every warp runs its own online softmax over the 16-position tiles
    // t = warp, warp + NCW, ... of each pass (no CTA barrier per pass):
    // S[head row][pos] = (alpha q as A: rows = heads hi / lo) x (K rows as B,
    // ldmatrix), folded hi + lo, exp2 against the warp's running max; the
    // score accumulators are re-packed in registers as the A operand (P
    // hi / lo rows) of O += P V (V tiles as B, ldmatrix.trans).  At the end
    // the NCW warp states are merged in smem (attn_warp_merge).
    struct WarpAtt {
        uint32_t qa[DH / 16][4];  // A fragments of alpha * log2e * q (bf16 hi / lo rows)
        float o[DH / 8][4];       // O accumulators: rows g (and g + 8) x dims
        float m, l;               // running max / sum of the head of row g
    };

    __device__ void attn_warp_init(WarpAtt& w) {
        const int lane = threadIdx.x % 32, g = lane / 4, q4 = lane % 4;
        const float* qs = att_q();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int row = g + 8 * (r & 1), d = kk * 16 + 2 * q4 + 8 * (r >> 1);
                uint32_t v = 0u;
                if (row < 2 * QPG) {
                    const int h = row % QPG;
                    const float x0 = qs[h * DH + d], x1 = qs[h * DH + d + 1];
                    if (row >= QPG) {
                        const float h0 = __bfloat162float(__float2bfloat16_rn(x0));
                        const float h1 = __bfloat162float(__float2bfloat16_rn(x1));
                        v = bf2_pack(x0 - h0, x1 - h1);
                    } else {
                        v = bf2_pack(x0, x1);
                    }
                }
                w.qa[kk][r] = v;
            }
#pragma unroll
        for (int c = 0; c < DH / 8; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e) w.o[c][e] = 0.f;
        w.m = -INFINITY;
        w.l = 0.f;
    }

    // this warp's tiles of one pass: positions [0, n) of the pass (ring rows
    // j < nring, the current token at j == nring), pass start pos0
    __device__ void attn_warp_pass(WarpAtt& w, uint32_t it0, int nring, int n, int pos0) {
        const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, q4 = lane % 4;
        const int ntiles = (n + 15) / 16;
        for (int t = warp; t < ntiles; t += NCW) {
            const int tb = t * 16;
            // scores: 2 n8 tiles of positions, K rows via ldmatrix (non-trans)
            float sc[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) sc[nt][e] = 0.f;
            {
                const int jr = min(tb + (lane & 7) + 8 * (lane >> 4), n - 1);
                const uint8_t* krow = att_row(it0, jr, nring, 0);
                const int key = (pos0 + jr) & 7, kh = (lane >> 3) & 1;
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk) {
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(krow + (((2 * kk + kh) ^ key) << 4), b0, b1, b2, b3);
                    mma_bf16(sc[0], w.qa[kk][0], w.qa[kk][1], w.qa[kk][2], w.qa[kk][3], b0, b1);
                    mma_bf16(sc[1], w.qa[kk][0], w.qa[kk][1], w.qa[kk][2], w.qa[kk][3], b2, b3);
                }
            }
            // fold hi + lo rows -> the score of row g's head; mask past n
            float f[2][2];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    float v;
                    if constexpr (QPG == 8) v = sc[nt][e] + sc[nt][e + 2];
                    else v = sc[nt][e] + __shfl_xor_sync(0xffffffffu, sc[nt][e], 4 * QPG);
                    f[nt][e] = tb + nt * 8 + 2 * q4 + e < n ? v : -INFINITY;
                }
            float mx = fmaxf(fmaxf(f[0][0], f[0][1]), fmaxf(f[1][0], f[1][1]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(w.m, mx);
            const float scale = exp2f(w.m - m_new);  // 0 on the first tile
            float pv[2][2], ps = 0.f;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    pv[nt][e] = exp2f(f[nt][e] - m_new);
                    ps += pv[nt][e];
                }
            ps += __shfl_xor_sync(0xffffffffu, ps, 1);
            ps += __shfl_xor_sync(0xffffffffu, ps, 2);
            w.m = m_new;
            w.l = w.l * scale + ps;
#pragma unroll
            for (int c = 0; c < DH / 8; ++c)
#pragma unroll
                for (int e = 0; e < 4; ++e) w.o[c][e] *= scale;
            // P as A fragments: row g = P hi (g < QPG) / P lo (QPG <= g < 2 QPG);
            // QPG = 8: rows g hi, g + 8 lo
            uint32_t pa[4];
            {
                auto hi2 = [](float a, float b) { return bf2_pack(__bfloat162float(__float2bfloat16_rn(a)),
                                                                   __bfloat162float(__float2bfloat16_rn(b))); };
                auto lo2 = [](float a, float b) {
                    return bf2_pack(a - __bfloat162float(__float2bfloat16_rn(a)),
                                    b - __bfloat162float(__float2bfloat16_rn(b)));
                };
                if constexpr (QPG == 8) {
                    pa[0] = hi2(pv[0][0], pv[0][1]);
                    pa[1] = lo2(pv[0][0], pv[0][1]);
                    pa[2] = hi2(pv[1][0], pv[1][1]);
                    pa[3] = lo2(pv[1][0], pv[1][1]);
                } else {
                    const bool lo_row = g >= QPG, live = g < 2 * QPG;
                    pa[0] = !live ? 0u : lo_row ? lo2(pv[0][0], pv[0][1]) : hi2(pv[0][0], pv[0][1]);
                    pa[2] = !live ? 0u : lo_row ? lo2(pv[1][0], pv[1][1]) : hi2(pv[1][0], pv[1][1]);
                    pa[1] = 0u;
                    pa[3] = 0u;
                }
            }
            // O += P V: V rows of the tile via ldmatrix.trans, 16 dims per x4
            {
                const int jr = min(tb + (lane & 7) + 8 * ((lane >> 3) & 1), n - 1);
                const uint8_t* vrow = att_row(it0, jr, nring, 1);
                const int key = (pos0 + jr) & 7;
#pragma unroll
                for (int c = 0; c < DH / 16; ++c) {
                    uint32_t b00, b01, b10, b11;
                    ldsm_x4_t(vrow + (((2 * c + (lane >> 4)) ^ key) << 4), b00, b01, b10, b11);
                    mma_bf16(w.o[2 * c], pa[0], pa[1], pa[2], pa[3], b00, b01);
                    mma_bf16(w.o[2 * c + 1], pa[0], pa[1], pa[2], pa[3], b10, b11);
                }
            }
        }
    }

    // merge the NCW warp states -> ro [QPG][DH] (unnormalised O), mlc [QPG][2]
    // (max, sum): the same CTA partial the pass path produces
    __device__ void attn_warp_merge(const WarpAtt& w, float* ro, float* mlc) {
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32, g = lane / 4, q4 = lane % 4;
        float* wml = att_q() + QPG * DH;        // [NCW][QPG][2]
        float* wo = wml + 2 * NCW * QPG;        // [NCW][QPG][DH]
        float ov[DH / 8][2];
#pragma unroll
        for (int c = 0; c < DH / 8; ++c)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if constexpr (QPG == 8) ov[c][e] = w.o[c][e] + w.o[c][e + 2];
                else ov[c][e] = w.o[c][e] + __shfl_xor_sync(0xffffffffu, w.o[c][e], 4 * QPG);
            }
        if (g < QPG) {
            float* dst = wo + (warp * QPG + g) * DH;
#pragma unroll
            for (int c = 0; c < DH / 8; ++c)
#pragma unroll
                for (int e = 0; e < 2; ++e) dst[c * 8 + 2 * q4 + e] = ov[c][e];
            if (q4 == 0) {
                wml[(warp * QPG + g) * 2] = w.m;
                wml[(warp * QPG + g) * 2 + 1] = w.l;
            }
        }
        consumer_sync(NCT);
        for (int idx = ctid; idx < QPG * DH; idx += NCT) {
            const int h = idx / DH, d = idx % DH;
            float M = -INFINITY;
#pragma unroll
            for (int v = 0; v < NCW; ++v)
                if (wml[(v * QPG + h) * 2 + 1] > 0.f) M = fmaxf(M, wml[(v * QPG + h) * 2]);
            float O = 0.f, L = 0.f;
#pragma unroll
            for (int v = 0; v < NCW; ++v) {
                const float lv = wml[(v * QPG + h) * 2 + 1];
                if (lv > 0.f) {
                    const float r = exp2f(wml[(v * QPG + h) * 2] - M);
                    O += r * wo[(v * QPG + h) * DH + d];
                    L += r * lv;
                }
            }
            ro[idx] = O;
            if (d == 0) {
                mlc[2 * h] = M;
                mlc[2 * h + 1] = L;
            }
        }
        consumer_sync(NCT);
    }

    __device__ void stage_attn(uint32_t& it, int l) {
        if (pl.attn_unit < 0) return;  // idle CTA: no chunks were streamed
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32;
        const int unit = pl.attn_unit, b = unit / S::NKV, kvh = unit % S::NKV;
        int p0, p1;
        attn_range(p0, p1);
        const int past_end = max(p0, min(p1, p.pos));
        const bool has_cur = p.pos >= p0 && p.pos < p1;
        float* st = att_st();  // (pass path only: outside the per-warp path's scratch)
        if (!T::ATT_WARP && ctid < QPG) {
            st[ctid * 4 + 0] = -INFINITY;
            st[ctid * 4 + 1] = 0.f;
            st[ctid * 4 + 2] = 0.f;
        }
        wait_stage(l * kStagesPerLayer + S_ATTN);
        {  // alpha * log2(e) * q of this kv head's QPG query heads -> smem
           // (alpha = 1/sqrt(dh); scores in log2 units, see attn_pass)
            const float alpha = 1.4426950408889634f / sqrtf(static_cast<float>(DH));
            float* qs = att_q();
            for (int i = ctid; i < QPG * DH; i += NCT)
                qs[i] = alpha * ldcg_f(p.q + (size_t)b * D + kvh * QPG * DH + i);
            // the current token's K/V rows (this launch's S_QKV wrote them with
            // generic stores; read at L2, emit.hpp:148-154 SyncLoadCurrentToken)
            if (has_cur) {
                uint8_t* cur = reinterpret_cast<uint8_t*>(h_s());  // [K row][V row]
                const size_t row = kv_row(l, b, kvh, p.pos);
                constexpr int V16 = DH * 2 / 16;
                if (ctid < 2 * V16) {
                    const __nv_bfloat16* src = (ctid < V16 ? p.kcache : p.vcache) + row;
                    const uint4 w = __ldcg(reinterpret_cast<const uint4*>(src) + ctid % V16);
                    *reinterpret_cast<uint4*>(cur + ctid * 16) = w;
                }
            }
        }
        constexpr int STR = DH + 2;
        float* mlc = reinterpret_cast<float*>(misc()) + 4;  // [QPG][2]
        float* ro = wpart();                                  // [QPG][DH]
        constexpr int PASS = T::ATT_SC * T::KVC;
        if constexpr (T::ATT_WARP) {
            consumer_sync(NCT);
            trace_mark(l * kStagesPerLayer + S_ATTN, 5);
            WarpAtt wa;
            attn_warp_init(wa);
            for (int c0 = p0; c0 < past_end || (c0 == p0 && has_cur); c0 += PASS) {
                const int nring = min(PASS, past_end - c0);
                const int nslots = (nring + T::KVC - 1) / T::KVC;
                const bool last = c0 + PASS >= past_end;
                const int n = nring + ((last && has_cur) ? 1 : 0);
                const uint32_t it0 = it;
                for (int s = 0; s < nslots; ++s, ++it)
                    wait_full(it % T::NSLOTS, (it / T::NSLOTS) & 1);
                trace_mark(l * kStagesPerLayer + S_ATTN, 6);
                attn_warp_pass(wa, it0, nring, n, c0);
                __syncwarp();
                if (lane == 0)
                    for (uint32_t i = it0; i < it; ++i) mbar_arrive(&empty[i % T::NSLOTS]);
                if (last) break;
            }
            trace_mark(l * kStagesPerLayer + S_ATTN, 3);
            attn_warp_merge(wa, ro, mlc);
        } else {
            float o[NTW][4];
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) o[nt][e] = 0.f;
            consumer_sync(NCT);
            trace_mark(l * kStagesPerLayer + S_ATTN, 5);

            for (int c0 = p0; c0 < past_end || (c0 == p0 && has_cur); c0 += PASS) {
                const int nring = min(PASS, past_end - c0);
                const int nslots = (nring + T::KVC - 1) / T::KVC;
                const bool last = c0 + PASS >= past_end;
                const int n = nring + ((last && has_cur) ? 1 : 0);
                const uint32_t it0 = it;
                for (int s = 0; s < nslots; ++s, ++it)
                    wait_full(it % T::NSLOTS, (it / T::NSLOTS) & 1);
                trace_mark(l * kStagesPerLayer + S_ATTN, 6);
                attn_pass_tc(it0, nring, n, c0, o);
                if (lane == 0)
                    for (uint32_t i = it0; i < it; ++i) mbar_arrive(&empty[i % T::NSLOTS]);
                if (last) break;
            }
            trace_mark(l * kStagesPerLayer + S_ATTN, 3);
            // CTA partial straight from the registers / stats to global (no
            // smem staging, no barrier): (m, l) from st, o summed over the
            // hi / lo rows of P
            float* part = p.attn_part + ((size_t)unit * grid + pl.attn_g) * QPG * STR;
            if (ctid < QPG) {
                __stcg(part + ctid * STR, st[ctid * 4 + 0]);
                __stcg(part + ctid * STR + 1, st[ctid * 4 + 1]);
            }
            // O[h][dim] = C[row h][dim] + C[row QPG + h][dim] (hi + lo of P):
            // QPG = 8: rows g / g + 8 of the same lane; QPG < 8: row g + QPG is
            // lane + 4 QPG.  Each (h, d) is owned by one lane: no cross-warp sum.
            float ov[NTW][2];
            {
#pragma unroll
                for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        if constexpr (QPG == 8) ov[nt][e] = o[nt][e] + o[nt][e + 2];
                        else ov[nt][e] = o[nt][e] + __shfl_xor_sync(0xffffffffu, o[nt][e], 4 * QPG);
                    }
            }
            {
                const int g = lane / 4, q4 = lane % 4;
                if (g < QPG)
#pragma unroll
                    for (int nt = 0; nt < NTW; ++nt)
                        __stcg(reinterpret_cast<float2*>(part + g * STR + 2 + warp * DPW + nt * 8 + 2 * q4),
                               make_float2(ov[nt][0], ov[nt][1]));
            }
        }
        if constexpr (T::ATT_WARP) {
            float* part = p.attn_part + ((size_t)unit * grid + pl.attn_g) * QPG * STR;
            for (int idx = ctid; idx < QPG * DH; idx += NCT) {
                const int h = idx / DH, d = idx % DH;
                const float O = ro[h * DH + d];
                float* dst = part + h * STR;
                __stcg(dst + 2 + d, O);
                if (d == 0) {
                    __stcg(dst, mlc[2 * h]);
                    __stcg(dst + 1, mlc[2 * h + 1]);
                }
            }
        }
        // The group's first CTA (attn_g == 0) combines (numerics.hpp:123-145):
        // the others publish their partial with one release arrival and move
        // on (no round trip); the combiner polls for the G - 1 arrivals
        // instead of a last-arriver acq_rel atomic, saving one L2 round trip
        // on the chain to S_AOUT.
        consumer_sync(NCT);
        trace_mark(l * kStagesPerLayer + S_ATTN, 7);
        uint32_t* hc = p.head_counters + (size_t)l * p.n_units + unit;
        if (pl.attn_g != 0) {
            if (ctid == 0) red_release_gpu(hc, 1);
            return;
        }
        if (ctid == 0)
            spin_until_geq(hc, p.epoch * static_cast<uint32_t>(p.attn_group - 1));
        consumer_sync(NCT);
        {
            // One L2 round trip: every thread first issues the G o-values of
            // its (first two) outputs into registers, then the (m, l) of the
            // whole group go to smem; per head (one warp): M = max m,
            // r_g = e^{m_g - M} / L; out = sum_g r_g o_g.
            const int G = p.attn_group;  // <= kMaxGroup (host-checked)
            const float* base = p.attn_part + (size_t)unit * grid * QPG * STR;
            constexpr int NO = (QPG * DH + NCT - 1) / NCT;  // outputs per thread
            constexpr int NV = NO < 2 ? NO : 2;             // held in registers at once
            float v[NV][kMaxGroup];
            auto load_o = [&](int k0) {
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int idx = ctid + (k0 + k) * NCT;
                    const int h = idx / DH, d = idx % DH;
                    const float* o = base + (size_t)h * STR + 2 + d;
#pragma unroll
                    for (int g = 0; g < kMaxGroup; ++g)
                        v[k][g] = (g < G && k0 + k < NO && idx < QPG * DH)
                                      ? ldcg_f(o + (size_t)g * QPG * STR)
                                      : 0.f;
                }
            };
            load_o(0);
            float* ml = wpart();  // [G][QPG][2]; free again after the barrier above
            for (int i = ctid; i < G * QPG; i += NCT) {
                const float* s = base + (size_t)i * STR;
                ml[2 * i] = ldcg_f(s);
                ml[2 * i + 1] = ldcg_f(s + 1);
            }
            consumer_sync(NCT);
            float* rr = ml + 2 * G * QPG;  // [QPG][G] combine weights
            for (int h = warp; h < QPG; h += NCW) {
                float M = -INFINITY;
                for (int g = lane; g < G; g += 32)
                    if (ml[2 * (g * QPG + h) + 1] > 0.f) M = fmaxf(M, ml[2 * (g * QPG + h)]);
                M = warp_max(M);
                float L = 0.f;
                for (int g = lane; g < G; g += 32) {
                    const float lg = ml[2 * (g * QPG + h) + 1];
                    if (lg > 0.f) L += lg * exp2f(ml[2 * (g * QPG + h)] - M);
                }
                L = warp_sum(L);
                for (int g = lane; g < G; g += 32) {
                    const float lg = ml[2 * (g * QPG + h) + 1];
                    rr[h * G + g] = lg > 0.f ? exp2f(ml[2 * (g * QPG + h)] - M) / L : 0.f;
                }
            }
            consumer_sync(NCT);
            for (int k0 = 0; k0 < NO; k0 += NV) {
                if (k0 > 0) load_o(k0);
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int idx = ctid + (k0 + k) * NCT;
                    if (k0 + k >= NO || idx >= QPG * DH) continue;
                    const int h = idx / DH, d = idx % DH;
                    float out = 0.f;
#pragma unroll
                    for (int g = 0; g < kMaxGroup; ++g)
                        if (g < G) out += rr[h * G + g] * v[k][g];
                    __stcg(p.attn_out + (size_t)b * D + (kvh * QPG + h) * DH + d, out);
                    if constexpr (S::KCP) frag_put(p.afrag, (kvh * QPG + h) * DH + d, b, out);
                }
            }
            if constexpr (S::KCP) fence_proxy_async_global();  // afrag is read by TMA
            arrive(p.counters + l * kStagesPerLayer + S_ATTN, l * kStagesPerLayer + S_ATTN);
        }
    }

    // ---------------------------------------------------------- TP exchange
    // Cross-rank sum of a residual delta: every rank's CTA i owns the same
    // slice [c0, c1) of d_model (identical plans), writes its delta into its
    // own exchange buffer, releases one arrival on CTA i's flag of every rank
    // (system scope: peers on other GPUs), waits for TP arrivals on its own
    // flag, then adds sum_r delta_r (fixed rank order: bit-identical x on
    // every rank).  delta: [B][cnt] in smem, slot 0 (S_AOUT) or 1 (S_RED).
    __device__ float* xch_slot(int r, int slot, int l) const {
        return p.xch[r] + ((size_t)(slot * 2 + (l & 1)) * B) * D;
    }

    __device__ void tp_exchange_add(const float* delta, int c0, int cnt, int slot, int l) {
        const int ctid = threadIdx.x;
        float* mine = xch_slot(p.tp_rank, slot, l);
        for (int i = ctid; i < cnt * B; i += NCT) {
            const int b = i / cnt, c = i % cnt;
            __stcg(mine + (size_t)b * D + c0 + c, delta[b * cnt + c]);
        }
        if (p.tp_host) return;  // host ncclAllReduce + apply between the launches
        consumer_sync(NCT);
        const size_t fi = ((size_t)l * 2 + slot) * grid + cta;
        if (ctid < p.tp_size) red_release_sys(p.xflag[ctid] + fi, 1);
        if (ctid == 0) spin_until_geq_sys(p.xflag[p.tp_rank] + fi, p.epoch * p.tp_size);
        consumer_sync(NCT);
        for (int i = ctid; i < cnt * B; i += NCT) {
            const int b = i / cnt, c = i % cnt;
            float t = 0.f;
            for (int r = 0; r < p.tp_size; ++r)
                t += ldcg_f(xch_slot(r, slot, l) + (size_t)b * D + c0 + c);
            float* xp = p.x + (size_t)b * D + c0 + c;
            __stcg(xp, ldcg_f(xp) + t);
        }
    }

    // ---------------------------------------------------------- S_AOUT
    // x[rows] += Waout[rows] . attn_out.  TP: Waout is split by input
    // columns (this rank's q heads, AD = NQ * DH of them), each rank holds a
    // partial of every row, summed across ranks (tp_exchange_add).
    __device__ void stage_aout(uint32_t& it, int l) {
        const int ctid = threadIdx.x;
        const int r0 = pl.aout_r0, nr = pl.aout_r1 - pl.aout_r0;
        float* acc = h_s();  // [B][TMAX] row results; x updated once at the end
        run_gemv<MA>(it, p.attn_out, false, nullptr, nullptr, l * kStagesPerLayer + S_AOUT, r0,
                     pl.aout_r1, [&](int c0, int nrows, const float* red) {
            if (ctid < nrows * B) {
                const int r = ctid / B, b = ctid % B;
                if constexpr (S::KCP) {  // (no TP at batch >= 8) x rows owned: update now
                    float* xp = p.x + (size_t)b * D + c0 + r;
                    __stcg(xp, ldcg_f(xp) + row_total<MA>(red, r, b));
                } else {
                    acc[b * T::TMAX + c0 - r0 + r] = row_total<MA>(red, r, b);
                }
            }
        });
        consumer_sync(NCT);
        if (p.tp_size > 1) {
            float* d = wpart();  // [B][nr] compact copy for the exchange
            for (int i = ctid; i < nr * B; i += NCT) {
                const int b = i / nr, r = i % nr;
                d[b * nr + r] = acc[b * T::TMAX + r];
            }
            consumer_sync(NCT);
            tp_exchange_add(d, r0, nr, 0, l);
        } else if constexpr (S::KCP) {  // x already updated: S_GLU's A table and norm statistics
            kc_publish(r0, pl.aout_r1, p.norm_ffn + (size_t)l * D, p.xfrag_a, p.ssq);
        } else {
            for (int i = ctid; i < nr * B; i += NCT) {  // one L2 round trip for all rows
                const int r = i / B, b = i % B;
                float* xp = p.x + (size_t)b * D + r0 + r;
                __stcg(xp, ldcg_f(xp) + acc[b * T::TMAX + r]);
            }
        }
        arrive(p.counters + l * kStagesPerLayer + S_AOUT, l * kStagesPerLayer + S_AOUT);
    }

    // ---------------------------------------------------------- S_GLU
    // in/gate rows [2 t0, 2 t1) of Wffn1 -> h[t - t0] = silu(gate) * in (smem)
    // act: the normalised activations (CUDA-core / quant GEMV); batch >= 8
    // passes nullptr and kc_inv_b (the A table is in the ring)
    __device__ void glu_ffn1(uint32_t& it, const Act<>* act, int t0, int t1,
                             const float* kc_inv_b = nullptr) {
        const int ctid = threadIdx.x;
        float* hs = h_s();
        auto epi = [&](int c0, int nrows, const float* red) {
            const int npairs = nrows / 2;
            if (ctid < npairs * B) {
                const int pr = ctid / B, b = ctid % B;
                const float a = row_total(red, 2 * pr, b), g = row_total(red, 2 * pr + 1, b);
                const float silu = g / (1.0f + expf(-g));
                if constexpr (S::KCP)
                    frag_put(p.hfrag, c0 / 2 + pr, b, silu * a);
                else if constexpr (T::F2R)
                    __stcg(p.glu_part + (size_t)b * S::DI + c0 / 2 + pr, silu * a);
                else
                    hs[b * T::TMAX + (c0 / 2 - t0) + pr] = silu * a;
            }
        };
        if constexpr (S::KCP) {
            gemv_kc<MD>(it, 2 * t0, 2 * t1, kc_inv_b, epi);
            fence_proxy_async_global();  // h is read by TMA in S_RED
        } else {
            gemv(it, *act, 2 * t0, 2 * t1, epi);
        }
        consumer_sync(NCT);  // h complete
    }

    // d_model partial of pairs [t0, t1) (Wffn2^T rows, AXPY) written to dst
    // ([RG][B][D] block of glu_part)
    __device__ void glu_ffn2(uint32_t& it, int t0, int t1, float* dst_part) {
        const int ctid = threadIdx.x;
        const float* hs = h_s();
        const int rg = ctid / T::TPR, lt = ctid % T::TPR, lane = ctid % 32;
        float acc[B][T::VPT][8];
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int j = 0; j < T::VPT; ++j)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[b][j][e] = 0.f;
        // quant: acc[col] = sum_r c_r,col s_r h_r (int4: times 16^k), and the
        // zero-point term sum_r z_r s_r h_r is the same for all of the
        // thread's columns (one group per row): one scalar per batch row
        float zs[B];
#pragma unroll
        for (int b = 0; b < B; ++b) zs[b] = 0.f;
        for (int c0 = t0; c0 < t1; c0 += T::RPS) {
            const int nrows = min(T::RPS, t1 - c0);
            const uint32_t slot = it % T::NSLOTS, par = (it / T::NSLOTS) & 1;
            wait_full(slot, par);
            const uint8_t* base = ring + slot * T::SLOT_BYTES;
            auto axpy_row = [&](int row) {
                float hb[B];
#pragma unroll
                for (int b = 0; b < B; ++b) hb[b] = hs[b * T::TMAX + (c0 - t0) + row];
                if constexpr (T::QB != 0) {
                    QRow<> q;
                    q_load(base + row * T::ROW_BYTES, lt, q);
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        hb[b] *= q.scale;
                        zs[b] = fmaf(q.zero, hb[b], zs[b]);
                    }
#pragma unroll
                    for (int j = 0; j < T::NCH; ++j) {
                        float2 d[4];
                        q_chunk(q, j, d);
#pragma unroll
                        for (int b = 0; b < B; ++b) {
                            const float2 h2 = make_float2(hb[b], hb[b]);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                float2 a2 = make_float2(acc[b][j][2 * k], acc[b][j][2 * k + 1]);
                                a2 = __ffma2_rn(d[k], h2, a2);
                                acc[b][j][2 * k] = a2.x;
                                acc[b][j][2 * k + 1] = a2.y;
                            }
                        }
                    }
                    return;
                }
#pragma unroll
                for (int j = 0; j < T::VPT; ++j) {
                    const uint4 w = lds_u128(base + row * T::ROW_BYTES + (lt + j * T::TPR) * 16);
                    const float2 wf[4] = {make_float2(bf_lo(w.x), bf_hi(w.x)),
                                          make_float2(bf_lo(w.y), bf_hi(w.y)),
                                          make_float2(bf_lo(w.z), bf_hi(w.z)),
                                          make_float2(bf_lo(w.w), bf_hi(w.w))};
#pragma unroll
                    for (int b = 0; b < B; ++b) {
                        const float2 h2 = make_float2(hb[b], hb[b]);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            float2 a2 = make_float2(acc[b][j][2 * k], acc[b][j][2 * k + 1]);
                            a2 = __ffma2_rn(wf[k], h2, a2);
                            acc[b][j][2 * k] = a2.x;
                            acc[b][j][2 * k + 1] = a2.y;
                        }
                    }
                }
            };
            if (nrows == T::RPS) {  // full slot: straight-line, no per-row branches
#pragma unroll
                for (int r = 0; r < T::APT; ++r) axpy_row(rg + r * T::RG);
            } else {
#pragma unroll
                for (int r = 0; r < T::APT; ++r)
                    if (rg + r * T::RG < nrows) axpy_row(rg + r * T::RG);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            ++it;
        }
        if constexpr (T::QB != 0) {  // undo the int4 decode scale, subtract the zero term
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
                for (int j = 0; j < T::NCH; ++j)
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        acc[b][j][e] = (T::QB == 4 ? acc[b][j][e] * q4_scale(e) : acc[b][j][e]) - zs[b];
        }
        // per-row-group partial d_model vectors
        float* gp = dst_part + (size_t)rg * B * D;
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int j = 0; j < T::VPT; ++j) {
                const int col = col_of(lt, j);
                float* dst = gp + (size_t)b * D + col;
                __stcg(reinterpret_cast<float4*>(dst),
                       make_float4(acc[b][j][0], acc[b][j][1], acc[b][j][2], acc[b][j][3]));
                __stcg(reinterpret_cast<float4*>(dst + 4),
                       make_float4(acc[b][j][4], acc[b][j][5], acc[b][j][6], acc[b][j][7]));
            }
    }

    // ---------------------------------------------------------- S_GLU
    // Static slice [glu_t0, glu_t1) into glu_part[cta].
    __device__ void stage_glu(uint32_t& it, int l) {
        if constexpr (S::KCP) {
            wait_stage(l * kStagesPerLayer + S_GLU);
            const float* inv = kc_inv(p.ssq);
            trace_mark(l * kStagesPerLayer + S_GLU, 3);
            glu_ffn1(it, nullptr, pl.glu_t0, pl.glu_t1, inv);
            arrive(p.counters + l * kStagesPerLayer + S_GLU, l * kStagesPerLayer + S_GLU);
            return;
        }
        Act<> act;
        load_act(act, p.x, false, p.norm_ffn + (size_t)l * D, l * kStagesPerLayer + S_GLU);
        glu_ffn1(it, &act, pl.glu_t0, pl.glu_t1);
        trace_mark(l * kStagesPerLayer + S_GLU, 3);  // (trace only: FFN1 done)
        if constexpr (T::F2R) {  // h is in glu_part; S_RED applies W2
            arrive(p.counters + l * kStagesPerLayer + S_GLU, l * kStagesPerLayer + S_GLU);
            return;
        }
        glu_ffn2(it, pl.glu_t0, pl.glu_t1, p.glu_part + (size_t)cta * T::RG * B * D);
        arrive(p.counters + l * kStagesPerLayer + S_GLU, l * kStagesPerLayer + S_GLU);
    }

    // ---------------------------------------------------------- S_RED
    // Two-phase FFN: x[rows] += W2[rows] . h (h = [B][DI] in glu_part, written
    // by every CTA's S_GLU); rows are this CTA's Waout rows.  TP: W2 is split
    // by input columns (this rank's d_inter slice), partials summed across
    // ranks in exchange slot 1.
    __device__ void stage_ffn2(uint32_t& it, int l) {
        const int ctid = threadIdx.x;
        const int r0 = pl.aout_r0, nr = pl.aout_r1 - pl.aout_r0;
        float* acc = h_s();  // [B][TMAX]
        run_gemv<MF>(it, p.glu_part, false, nullptr, nullptr, l * kStagesPerLayer + S_RED, r0,
                     pl.aout_r1, [&](int c0, int nrows, const float* red) {
            if (ctid < nrows * B) {
                const int r = ctid / B, b = ctid % B;
                if constexpr (S::KCP) {  // (no TP at batch >= 8) x rows owned: update now
                    float* xp = p.x + (size_t)b * D + c0 + r;
                    __stcg(xp, ldcg_f(xp) + row_total<MF>(red, r, b));
                } else {
                    acc[b * T::TMAX + c0 - r0 + r] = row_total<MF>(red, r, b);
                }
            }
        });
        consumer_sync(NCT);
        if (p.tp_size > 1) {
            float* d = wpart();
            for (int i = ctid; i < nr * B; i += NCT) {
                const int b = i / nr, r = i % nr;
                d[b * nr + r] = acc[b * T::TMAX + r];
            }
            consumer_sync(NCT);
            tp_exchange_add(d, r0, nr, 1, l);
        } else if constexpr (S::KCP) {  // x already updated: next S_QKV's (or the LM head's) A table
            kc_publish(r0, pl.aout_r1,
                       l + 1 < p.layers ? p.norm_attn + (size_t)(l + 1) * D : p.final_norm,
                       p.xfrag_f, p.ssq + (size_t)grid * B);
        } else {
            for (int i = ctid; i < nr * B; i += NCT) {
                const int r = i / B, b = i % B;
                float* xp = p.x + (size_t)b * D + r0 + r;
                __stcg(xp, ldcg_f(xp) + acc[b * T::TMAX + r]);
            }
        }
        arrive(p.counters + l * kStagesPerLayer + S_RED, l * kStagesPerLayer + S_RED);
    }

    __device__ void stage_red(int l) {
        wait_stage(l * kStagesPerLayer + S_RED);
        const int ctid = threadIdx.x, warp = ctid / 32, lane = ctid % 32;
        const int c0 = pl.red_c0, c1 = pl.red_c1;
        // CTA partials in a fixed order -> deterministic sums
        const int nparts = grid * T::RG;
        float* scratch = wpart();          // [NCW][32]
        float* delta = wpart() + NCW * 32;  // [B][c1 - c0] (TP)
        for (int b = 0; b < B; ++b) {
            for (int cb = c0; cb < c1; cb += 32) {
                const int col = cb + lane;
                float s = 0.f;
                if (col < c1) {
                    // partials warp, warp+NCW, ... summed in that fixed order,
                    // 8 independent L2 loads in flight per thread
                    constexpr int U = 32;  // independent L2 loads in flight per thread
                    for (int q0 = warp; q0 < nparts; q0 += U * NCW) {
                        float v[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int q = q0 + u * NCW;
                            const float* src = p.glu_part + (size_t)q * B * D;
                            v[u] = q < nparts ? ldcg_f(src + (size_t)b * D + col) : 0.f;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) s += v[u];
                    }
                }
                scratch[warp * 32 + lane] = s;
                consumer_sync(NCT);
                if (warp == 0 && col < c1) {
                    float t = 0.f;
                    for (int w = 0; w < NCW; ++w) t += scratch[w * 32 + lane];
                    if (p.tp_size > 1) {
                        delta[b * (c1 - c0) + col - c0] = t;  // exchanged below
                    } else {
                        float* xp = p.x + (size_t)b * D + col;
                        __stcg(xp, ldcg_f(xp) + t);
                    }
                }
                consumer_sync(NCT);
            }
        }
        if (p.tp_size > 1) tp_exchange_add(delta, c0, c1 - c0, 1, l);
        arrive(p.counters + l * kStagesPerLayer + S_RED, l * kStagesPerLayer + S_RED);
    }

    // ---------------------------------------------------------- S_LMHEAD
    __device__ void stage_lmhead(uint32_t& it) {
        const int ctid = threadIdx.x;
        float best = -INFINITY;
        int best_i = 0x7fffffff;
        run_gemv<MD>(it, p.x, p.layers == 0, p.final_norm,
                     S::KCP ? p.ssq + (size_t)grid * B : nullptr, p.layers * kStagesPerLayer,
                     pl.lm_r0, pl.lm_r1, [&](int c0, int nrows, const float* red) {
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
            const uint32_t old = atom_add_acq_rel_gpu(p.amax_counter, 1);
            flag[1] = (old + 1 == p.epoch * static_cast<uint32_t>(grid)) ? 1 : 0;
        }
        consumer_sync(NCT);
        if (flag[1]) {
            // all CTA candidates into smem in one parallel pass, then scan in
            // CTA (= ascending row) order
            // (batch >= 8: the ring, drained after the last stage's GEMV)
            float* cv = S::KCP ? reinterpret_cast<float*>(ring) : wpart();
            int* ci = reinterpret_cast<int*>(cv + grid * B);
            for (int i = ctid; i < grid * B; i += NCT) {
                cv[i] = ldcg_f(p.amax_val + i);
                ci[i] = __ldcg(p.amax_idx + i);
            }
            consumer_sync(NCT);
            if (ctid < B) {
                float bv = -INFINITY;
                int bi = 0;
                bool any = false;
                for (int c = 0; c < grid; ++c) {
                    const float v = cv[c * B + ctid];
                    const int i = ci[c * B + ctid];
                    if (i == 0x7fffffff) continue;  // CTA without lm_head rows
                    if (!any || v > bv || (v == bv && i < bi)) {
                        bv = v;
                        bi = i;
                        any = true;
                    }
                }
                if (p.tp_size == 1) {
                    p.greedy[ctid] = bi;
                } else {  // this rank's candidate, as a global vocab index
                    cv[ctid] = any ? bv : -INFINITY;
                    ci[ctid] = bi + p.vocab_base;
                }
            }
            if (p.tp_size > 1) {
                // exchange (value, index) with every rank; ranks own ascending
                // vocab slices, so scanning ranks in order keeps the lowest
                // index on ties (numerics.hpp:169-175)
                consumer_sync(NCT);
                const size_t amax_off = (size_t)4 * B * D;
                if (p.tp_host) {  // this rank's candidates, ncclAllGather'ed by the host
                    if (ctid < B) {
                        float* dst = p.xch[p.tp_rank] + amax_off + ((size_t)p.tp_rank * B + ctid) * 2;
                        __stcg(dst, cv[ctid]);
                        __stcg(dst + 1, __int_as_float(ci[ctid]));
                    }
                    return;
                }
                const size_t fi = (size_t)p.layers * 2 * grid;
                if (ctid < B * p.tp_size) {
                    const int r = ctid / B, b = ctid % B;
                    float* dst = p.xch[r] + amax_off + ((size_t)p.tp_rank * B + b) * 2;
                    __stcg(dst, cv[b]);
                    __stcg(dst + 1, __int_as_float(ci[b]));
                }
                consumer_sync(NCT);
                if (ctid < p.tp_size) red_release_sys(p.xflag[ctid] + fi, 1);
                if (ctid == 0) spin_until_geq_sys(p.xflag[p.tp_rank] + fi, p.epoch * p.tp_size);
                consumer_sync(NCT);
                if (ctid < B) {
                    float bv = -INFINITY;
                    int bi = 0;
                    for (int r = 0; r < p.tp_size; ++r) {
                        const float* src = p.xch[p.tp_rank] + amax_off + ((size_t)r * B + ctid) * 2;
                        const float v = ldcg_f(src);
                        const int i = __float_as_int(ldcg_f(src + 1));
                        if (r == 0 || v > bv) {
                            bv = v;
                            bi = i;
                        }
                    }
                    p.greedy[ctid] = bi;
                }
            }
        }
        trace_mark(p.layers * kStagesPerLayer, 2);  // (trace only: LM-head end)
    }

    // ---------------------------------------------------------- linear
    // x_out[rows] = W_l[rows] . x_in (no residual, no norm; f32 accumulation,
    // interpreter.hpp:227-238)
    __device__ void stage_linear(uint32_t& it, int l) {
        Act<> act;
        const float* xin = p.xbuf + (size_t)(l & 1) * B * D;
        float* xout = p.xbuf + (size_t)((l + 1) & 1) * B * D;
        load_act(act, xin, false, nullptr, l);
        const int ctid = threadIdx.x;
        gemv(it, act, pl.aout_r0, pl.aout_r1, [&](int c0, int nrows, const float* red) {
            if (ctid < nrows * B) {
                const int r = ctid / B, b = ctid % B;
                __stcg(xout + (size_t)b * D + c0 + r, row_total(red, r, b));
            }
        });
        arrive(p.counters + l, l);
    }

    __device__ void consumer() {
        uint32_t it = 0;
        const int last = min(p.stage_end, n_stages());
        for (int stage = p.stage_begin; stage < last; ++stage) {
            trace_mark(stage, 0);
            if (p.kind == 1) {
                if constexpr (!S::KCP) stage_linear(it, stage);  // (host: kind 1 is batch < 8)
                continue;
            }
            const int l = stage / kStagesPerLayer, s = stage % kStagesPerLayer;
            if (stage == p.layers * kStagesPerLayer) {
                stage_lmhead(it);
                continue;
            }
            if (!((p.stage_mask >> s) & 1)) continue;  // (component ablation)
            switch (s) {
                case S_QKV: stage_qkv(it, l); break;
                case S_ATTN: stage_attn(it, l); break;
                case S_AOUT: stage_aout(it, l); break;
                case S_GLU: stage_glu(it, l); break;
                default:
                    if constexpr (T::F2R) stage_ffn2(it, l);
                    else stage_red(l);
                    break;
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
#ifdef FFB_KCP_TCGEN05
        if constexpr (S::KCP) {
            mbar_init(cta.accbar(), 1);
            mbar_init(cta.abar(), 1);
        }
#endif
        fence_mbar_init();
    }
    // batch >= 8: 512 TMEM columns (the whole SM's, one CTA per SM) for the
    // tcgen05 GEMV accumulators (DecodeCta::gemv_kc)
#ifdef FFB_KCP_TCGEN05
    if constexpr (S::KCP) {
        if (tid < 32) tmem_alloc(cta.tmem_slot(), 512);
        tc05_fence_before();
    }
#endif
    // RoPE table for this step's position, in f64 (numerics.hpp:27-37 angle)
    if (tid < S::DH / 2) {
        const double freq = pow(p.rope_theta, -static_cast<double>(2 * tid) / S::DH);
        const double ang = static_cast<double>(p.pos) * freq;
        cta.rope()[2 * tid] = static_cast<float>(cos(ang));
        cta.rope()[2 * tid + 1] = static_cast<float>(sin(ang));
    }
    // residual init from the embedding: each CTA owns its reduce columns
    if (p.kind == 0 && p.stage_begin == 0 && tid < T::NCT) {
        for (int b = 0; b < S::B; ++b) {
            const __nv_bfloat16* e = p.embedding + (size_t)token_row(p, b) * S::D;
            for (int c = p.plan[cta.cta].red_c0 + tid; c < p.plan[cta.cta].red_c1; c += T::NCT)
                __stcg(p.x + (size_t)b * S::D + c, __bfloat162float(e[c]));
        }
    }
    __syncthreads();
    if (tid >= T::NCT) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(T::PRODUCER_REGS));
        if (tid == T::NCT) cta.template producer<false>();
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(T::CONSUMER_REGS));
#ifdef FFB_KCP_TCGEN05
    if constexpr (S::KCP) tc05_fence_after();
#endif
    if constexpr (S::KCP) {
        // the initial x rows' A-table entries and norm statistics; the first
        // S_QKV (or the LM head) waits for every CTA's arrival
        if (p.kind == 0 && p.stage_begin == 0 && !(p.debug & kDebugStreamOnly)) {
            cta.kc_publish(cta.pl.red_c0, cta.pl.red_c1,
                           p.layers > 0 ? p.norm_attn : p.final_norm, p.xfrag_f,
                           p.ssq + (size_t)gridDim.x * S::B);
            if (tid == 0) red_release_gpu(p.counters + p.layers * kStagesPerLayer + 1, 1);
        }
    }
    if (p.debug & kDebugStreamOnly) {
        cta.template producer<true>();  // streaming-only measurement
    } else {
        cta.consumer();
    }
#ifdef FFB_KCP_TCGEN05
    if constexpr (S::KCP) {  // every MMA was waited for (accbar) and every TMEM load completed
        tc05_fence_before();
        consumer_sync(T::NCT);
        tc05_fence_after();
        if (tid < 32) tmem_dealloc(cta.tmem_base(), 512);
    }
#endif
}

}  // namespace ffb200
