// prefill.cu -- prompt ingestion as GEMMs ("a real
// prefill GEMM path is the step before decode").
//
// The reference ingests a prompt one position at a time (decode-as-prefill,
// reference.hpp:60-61: reference_forward at pos, pos + 1, ...).  Here n
// prompt positions of every batch row go through each layer together: the
// projections are GEMMs over M = n * B activation rows on the tensor cores,
// the rest (RMSNorm, RoPE + K/V append, causal attention over the cache,
// SiLU, residual adds) are small kernels of this file; the K/V cache and the
// cache lengths end exactly where n decode steps would leave them, so decoding
// continues with the persistent kernel at pos0 + n.
//
// Numerics.  The bf16 weights are exact in bf16; every GEMM input activation
// (f32) is split into three bf16 terms (hi + mid + lo carry 24 bits, the
// f32 mantissa) and the GEMM runs three bf16 x bf16 products accumulated in
// f32 (cublasGemmEx, CUBLAS_COMPUTE_32F) -- f32-accurate products on the
// bf16 tensor cores.  Attention and everything elementwise is f32 (the
// online softmax in f32, like the decode kernel); K/V are rounded to bf16 at
// append, as reference.hpp / KVCache::append do.
//
// cuBLAS is loaded at run time (dlopen "libcublas.so.12"): plain library
// GEMMs only, the decode path never touches it.  bf16 weights in the
// row-major layout only (batch < 8, no quantisation, one GPU).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/flashformer_b200.h"
#include "model.cuh"

namespace ffb200 {
ffb_status fail(ffb_status s, const char* fmt, ...);  // runtime.cu
}  // namespace ffb200

using namespace ffb200;

namespace {

// ---- cuBLAS, loaded at run time ----------------------------------------
// (the subset of cublas_api.h this file uses; values from that header)
typedef void* cublasHandle_t;
enum { CUBLAS_OP_N = 0, CUBLAS_OP_T = 1 };
enum { kCUDA_R_32F = 0, kCUDA_R_16BF = 14 };
enum { kCUBLAS_COMPUTE_32F = 68 };
enum { kCUBLAS_GEMM_DEFAULT = -1 };

struct CublasApi {
    int (*create)(cublasHandle_t*);
    int (*set_stream)(cublasHandle_t, cudaStream_t);
    int (*destroy)(cublasHandle_t);
    int (*gemm_ex)(cublasHandle_t, int, int, int, int, int, const void*, const void*, int, int,
                   const void*, int, int, const void*, void*, int, int, int, int);
};

const CublasApi* cublas() {
    static CublasApi api{};
    static bool ok = [] {
        void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        api.create = reinterpret_cast<decltype(api.create)>(dlsym(h, "cublasCreate_v2"));
        api.set_stream = reinterpret_cast<decltype(api.set_stream)>(dlsym(h, "cublasSetStream_v2"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "cublasDestroy_v2"));
        api.gemm_ex = reinterpret_cast<decltype(api.gemm_ex)>(dlsym(h, "cublasGemmEx"));
        return api.create && api.set_stream && api.destroy && api.gemm_ex;
    }();
    return ok ? &api : nullptr;
}

// ---- kernels --------------------------------------------------------------
__global__ void k_embed(float* __restrict__ x, const __nv_bfloat16* __restrict__ emb,
                        const int64_t* __restrict__ tok, int rows, int D) {
    const int r = blockIdx.x;
    if (r >= rows) return;
    const __nv_bfloat16* e = emb + (size_t)tok[r] * D;
    for (int c = threadIdx.x; c < D; c += blockDim.x) x[(size_t)r * D + c] = __bfloat162float(e[c]);
}

__device__ __forceinline__ void split3(float v, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
    a = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(a);
    b = __float2bfloat16_rn(r1);
    c = __float2bfloat16_rn(r1 - __bfloat162float(b));
}

// one element of a split-term GEMM result: (hi + mid) + lo planes
__device__ __forceinline__ float ld3(const float* c, size_t plane, size_t i) {
    return (c[i] + c[plane + i]) + c[2 * plane + i];
}

// y = gain * x / sqrt(mean(x^2) + eps) (numerics.hpp:14-24; gain == nullptr:
// y = x), split into three bf16 terms [3][rows][K]
__global__ void k_norm_split(const float* __restrict__ src, const float* __restrict__ gain, float eps,
                             __nv_bfloat16* __restrict__ y3, int rows, int K) {
    const int r = blockIdx.x;
    const float* x = src + (size_t)r * K;
    float inv = 1.f;
    if (gain != nullptr) {
        __shared__ float part[32];
        float s = 0.f;
        for (int c = threadIdx.x; c < K; c += blockDim.x) s = fmaf(x[c], x[c], s);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
        __syncthreads();
        float t = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        inv = 1.0f / sqrtf(t / static_cast<float>(K) + eps);
    }
    const size_t plane = (size_t)rows * K;
    for (int c = threadIdx.x; c < K; c += blockDim.x) {
        const float v = gain != nullptr ? gain[c] * x[c] * inv : x[c];
        __nv_bfloat16 a, b, d;
        split3(v, a, b, d);
        y3[(size_t)r * K + c] = a;
        y3[plane + (size_t)r * K + c] = b;
        y3[2 * plane + (size_t)r * K + c] = d;
    }
}

__device__ __forceinline__ int swz(int d, int64_t pos) { return ((((d >> 3) ^ (int)(pos & 7))) << 3) | (d & 7); }

// RoPE (interleaved pairs, f64 angle as numerics.hpp:27-37 / the decode
// kernel) on q and k rows of the QKV output; K and V rounded to bf16 and
// appended at position pos0 + t of batch row b; q (f32) kept for attention.
// Activation row r = t * B + b.
__global__ void k_qkv_epilogue(const float* __restrict__ qkv, size_t plane, float* __restrict__ q, __nv_bfloat16* kc,
                               __nv_bfloat16* vc, int rows, int B, int NQ, int NKV, int DH, int64_t pos0,
                               double theta, int64_t layer_off, int64_t max_seq) {
    const int r = blockIdx.x;
    const int t = r / B, b = r % B;
    const int64_t pos = pos0 + t;
    const int QR = NQ * DH, KR = NKV * DH, QKVR = QR + 2 * KR;
    const size_t base = (size_t)r * QKVR;
    for (int i = threadIdx.x; i < QKVR / 2; i += blockDim.x) {
        const int g = 2 * i;
        const float a = ld3(qkv, plane, base + g), c2 = ld3(qkv, plane, base + g + 1);
        if (g < QR + KR) {
            const int dim = g % DH, k = dim / 2;
            const double freq = pow(theta, -static_cast<double>(2 * k) / DH);
            const double ang = static_cast<double>(pos) * freq;
            const float cs = static_cast<float>(cos(ang)), sn = static_cast<float>(sin(ang));
            const float r0 = a * cs - c2 * sn, r1 = a * sn + c2 * cs;
            if (g < QR) {
                q[(size_t)r * QR + g] = r0;
                q[(size_t)r * QR + g + 1] = r1;
            } else {
                const int h = (g - QR) / DH;
                __nv_bfloat16* row = kc + layer_off + (((size_t)b * NKV + h) * max_seq + pos) * DH;
                row[swz(dim, pos)] = __float2bfloat16_rn(r0);
                row[swz(dim + 1, pos)] = __float2bfloat16_rn(r1);
            }
        } else {
            const int gv = g - QR - KR, h = gv / DH, dim = gv % DH;
            __nv_bfloat16* row = vc + layer_off + (((size_t)b * NKV + h) * max_seq + pos) * DH;
            row[swz(dim, pos)] = __float2bfloat16_rn(a);
            row[swz(dim + 1, pos)] = __float2bfloat16_rn(c2);
        }
    }
}

// Causal attention, tiled: one block per (query tile, kv head, batch row)
// holds kPairs (query position, q head) pairs of one GQA group -- TQ =
// kPairs / QPG consecutive prompt positions x the group's QPG heads -- and
// walks the keys [0, last position of the tile] in tiles of kKeys staged in
// shared memory (un-swizzled, K rows padded so lane-per-row reads are bank-
// conflict free), shared by all pairs.  Warp w owns pairs [8w, 8w + 8):
// scores lane-per-key (keys j, j + 32 of the tile), online softmax per pair
// in f32 (two warp reductions per tile), P through shared memory, then P.V
// lane-per-dims.  Everything f32; only the order of the sums differs from
// the decode kernel's.
constexpr int kPairs = 64, kKeys = 64, kPPW = 8;  // pairs per block / keys per tile / pairs per warp

template <int DH>
struct AttnSmem {
    static constexpr int KSTRIDE = DH + 8;  // bf16 elements per staged K row
    static constexpr int Q_OFF = 0;                                   // f32 [kPairs][DH]
    static constexpr int K_OFF = Q_OFF + kPairs * DH * 4;             // bf16 [kKeys][KSTRIDE]
    static constexpr int V_OFF = K_OFF + kKeys * KSTRIDE * 2;         // bf16 [kKeys][DH]
    static constexpr int P_OFF = V_OFF + kKeys * DH * 2;              // f32 [8 warps][kPPW][kKeys]
    static constexpr int BYTES = P_OFF + 8 * kPPW * kKeys * 4;
};

template <int DH>
__global__ void __launch_bounds__(256, 1) k_attention(const float* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                                                   const __nv_bfloat16* __restrict__ vc, float* __restrict__ out,
                                                   int B, int NQ, int NKV, int n, int64_t pos0,
                                                   int64_t layer_off, int64_t max_seq) {
    using SM = AttnSmem<DH>;
    constexpr int DPL = DH / 32, CH = DH / 8;  // dims per lane (P.V), 16-byte chunks per row
    extern __shared__ __align__(16) uint8_t sm[];
    float* Qs = reinterpret_cast<float*>(sm + SM::Q_OFF);
    __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(sm + SM::K_OFF);
    __nv_bfloat16* Vs = reinterpret_cast<__nv_bfloat16*>(sm + SM::V_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* Ps = reinterpret_cast<float*>(sm + SM::P_OFF) + warp * kPPW * kKeys;
    const int qpg = NQ / NKV, tq = kPairs / qpg;
    const int t0 = blockIdx.x * tq, kvh = blockIdx.y, b = blockIdx.z;
    const float alpha = 1.0f / sqrtf(static_cast<float>(DH));
    // stage the tile's queries, pre-scaled (pairs past the prompt: zeros)
    for (int i = threadIdx.x; i < kPairs * DH; i += blockDim.x) {
        const int pr = i / DH, d = i % DH, t = t0 + pr / qpg, h = kvh * qpg + pr % qpg;
        Qs[i] = t < n ? alpha * q[((size_t)t * B + b) * NQ * DH + (size_t)h * DH + d] : 0.f;
    }
    const __nv_bfloat16* kb = kc + layer_off + ((size_t)b * NKV + kvh) * max_seq * DH;
    const __nv_bfloat16* vb = vc + layer_off + ((size_t)b * NKV + kvh) * max_seq * DH;
    const int tlast = min(t0 + tq, n) - 1;
    const int64_t kend = pos0 + tlast + 1;  // keys of the whole tile
    // this warp's pairs: positions qpos[i], the warp's last key
    int64_t qpos[kPPW];
#pragma unroll
    for (int i = 0; i < kPPW; ++i) qpos[i] = pos0 + min(t0 + (warp * kPPW + i) / qpg, tlast);
    const int64_t wend = qpos[kPPW - 1] + 1;
    float mx[kPPW], sum[kPPW], o[kPPW][DPL];
#pragma unroll
    for (int i = 0; i < kPPW; ++i) {
        mx[i] = -INFINITY;
        sum[i] = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[i][e] = 0.f;
    }
    for (int64_t k0 = 0; k0 < kend; k0 += kKeys) {
        __syncthreads();  // previous tile consumed (and Q staged, first time)
        for (int i = threadIdx.x; i < kKeys * CH; i += blockDim.x) {
            const int j = i / CH, c = i % CH;
            const int64_t pos = k0 + j;
            uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
            if (pos < kend) {
                const int cs = c ^ (int)(pos & 7);  // the cache's chunk swizzle (kv_swz)
                kv = *reinterpret_cast<const uint4*>(kb + pos * DH + cs * 8);
                vv = *reinterpret_cast<const uint4*>(vb + pos * DH + cs * 8);
            }
            *reinterpret_cast<uint4*>(Ks + j * SM::KSTRIDE + c * 8) = kv;
            *reinterpret_cast<uint4*>(Vs + j * DH + c * 8) = vv;
        }
        __syncthreads();
        if (k0 >= wend) continue;  // every key of this tile is after the warp's positions
        // scores: lane owns keys k0 + lane and k0 + lane + 32
        float sc[kPPW][2];
#pragma unroll
        for (int i = 0; i < kPPW; ++i) sc[i][0] = sc[i][1] = 0.f;
        const float* qw = Qs + warp * kPPW * DH;
#pragma unroll 2
        for (int c = 0; c < CH; ++c) {
            float ka[8], kb2[8];
            const uint4 r0 = *reinterpret_cast<const uint4*>(Ks + lane * SM::KSTRIDE + c * 8);
            const uint4 r1 = *reinterpret_cast<const uint4*>(Ks + (lane + 32) * SM::KSTRIDE + c * 8);
            const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&r0);
            const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&r1);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f0 = __bfloat1622float2(h0[e]), f1 = __bfloat1622float2(h1[e]);
                ka[2 * e] = f0.x;
                ka[2 * e + 1] = f0.y;
                kb2[2 * e] = f1.x;
                kb2[2 * e + 1] = f1.y;
            }
#pragma unroll
            for (int i = 0; i < kPPW; ++i) {
                const float4 qa = *reinterpret_cast<const float4*>(qw + i * DH + c * 8);
                const float4 qb = *reinterpret_cast<const float4*>(qw + i * DH + c * 8 + 4);
                const float qq[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    sc[i][0] = fmaf(qq[e], ka[e], sc[i][0]);
                    sc[i][1] = fmaf(qq[e], kb2[e], sc[i][1]);
                }
            }
        }
        // online softmax per pair, P to shared memory
#pragma unroll
        for (int i = 0; i < kPPW; ++i) {
            const float s0 = k0 + lane <= qpos[i] ? sc[i][0] : -INFINITY;
            const float s1 = k0 + lane + 32 <= qpos[i] ? sc[i][1] : -INFINITY;
            float tm = fmaxf(s0, s1);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, off));
            const float mn = fmaxf(mx[i], tm);  // finite: key 0 <= every position
            const float p0 = expf(s0 - mn), p1 = expf(s1 - mn), scale = expf(mx[i] - mn);
            float ts = p0 + p1;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) ts += __shfl_xor_sync(0xffffffffu, ts, off);
            sum[i] = sum[i] * scale + ts;
            mx[i] = mn;
#pragma unroll
            for (int e = 0; e < DPL; ++e) o[i][e] *= scale;
            Ps[i * kKeys + lane] = p0;
            Ps[i * kKeys + lane + 32] = p1;
        }
        __syncwarp();
        // P.V: lane owns dims [lane * DPL, lane * DPL + DPL)
        const int jn = wend - k0 < kKeys ? (int)(wend - k0) : kKeys;
        for (int j = 0; j < jn; j += 4) {
            float v[4][DPL];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
#pragma unroll
                for (int e = 0; e < DPL; ++e) v[u][e] = __bfloat162float(Vs[(j + u) * DH + lane * DPL + e]);
            }
#pragma unroll
            for (int i = 0; i < kPPW; ++i) {
                const float4 p4 = *reinterpret_cast<const float4*>(Ps + i * kKeys + j);
#pragma unroll
                for (int e = 0; e < DPL; ++e)
                    o[i][e] = fmaf(p4.w, v[3][e], fmaf(p4.z, v[2][e], fmaf(p4.y, v[1][e], fmaf(p4.x, v[0][e], o[i][e]))));
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < kPPW; ++i) {
        const int pr = warp * kPPW + i, t = t0 + pr / qpg, h = kvh * qpg + pr % qpg;
        if (t >= n) continue;
        float* dst = out + ((size_t)t * B + b) * NQ * DH + (size_t)h * DH + lane * DPL;
#pragma unroll
        for (int e = 0; e < DPL; ++e) dst[e] = o[i][e] / sum[i];
    }
}

// h[t] = silu(gate) * in over the interleaved (in, gate) rows of Wffn1
__global__ void k_silu(const float* __restrict__ c, size_t plane, float* __restrict__ h, int rows, int DI) {
    const size_t n = (size_t)rows * DI;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t r = i / DI, k = i % DI;
        const float a = ld3(c, plane, r * 2 * DI + 2 * k), g = ld3(c, plane, r * 2 * DI + 2 * k + 1);
        h[i] = g / (1.0f + expf(-g)) * a;
    }
}

__global__ void k_add(float* __restrict__ x, const float* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        x[i] += ld3(d, n, i);
}

// logits of the last positions: the three planes summed in place
__global__ void k_sum3(float* __restrict__ c, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        c[i] = ld3(c, n, i);
}

// lowest index of the maximum (numerics.hpp:169-175), one block per row
__global__ void k_argmax(const float* __restrict__ lg, int V, int64_t* __restrict__ out) {
    const float* x = lg + (size_t)blockIdx.x * V;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < V; i += blockDim.x)
        if (x[i] > bv) {
            bv = x[i];
            bi = i;
        }
    __shared__ float sv[256];
    __shared__ int si[256];
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int t = 1; t < (int)blockDim.x; ++t)
            if (sv[t] > bv || (sv[t] == bv && si[t] < bi)) {
                bv = sv[t];
                bi = si[t];
            }
        out[blockIdx.x] = bi;
    }
}

// C3[3][rows][N] (f32, row-major) = Y3[3][rows][K] . W^T: ONE GEMM over the
// 3 * rows stacked split-term rows, so W is read once; consumers add the
// three planes (ld3).  W bf16 row-major [N][K] (w_kn = false) or [K][N]
// (w_kn = true: Wffn2^T stored [DI][D])
ffb_status gemm3(cublasHandle_t h, const __nv_bfloat16* y3, int rows, int K, const void* W, int N, bool w_kn,
                 float* C3) {
    const float one = 1.f, zero = 0.f;
    // column-major view: C'[N][3 rows] = op(W') . Y'[K][3 rows]
    const int st = cublas()->gemm_ex(h, w_kn ? CUBLAS_OP_N : CUBLAS_OP_T, CUBLAS_OP_N, N, 3 * rows, K, &one, W,
                                     kCUDA_R_16BF, w_kn ? N : K, y3, kCUDA_R_16BF, K, &zero, C3, kCUDA_R_32F, N,
                                     kCUBLAS_COMPUTE_32F, kCUBLAS_GEMM_DEFAULT);
    if (st != 0) return fail(FFB_DEVICE, "prefill: cublasGemmEx failed (status %d)", st);
    return FFB_OK;
}

}  // namespace

extern "C" ffb_status ffb_prefill(ffb_model* m, const int64_t* tokens, int64_t n, int64_t pos0, float* logits,
                                  int64_t* greedy) {
    if (!m || !tokens || n <= 0) return fail(FFB_USAGE, "prefill: NULL argument or n <= 0");
    const auto& c = m->cfg;
    if (c.kind != 0 || m->ops->QB != 0 || m->ops->kc != 0 || m->tp_size != 1)
        return fail(FFB_UNSUPPORTED, "prefill: bf16 decoder, batch < 8, one GPU");
    if (!cublas()) return fail(FFB_UNSUPPORTED, "prefill: cuBLAS not available (dlopen libcublas.so.12)");
    for (int64_t l = 0; l < c.layers; ++l)
        if (m->kv_len[l] != pos0)
            return fail(FFB_VALIDATION, "prefill: cache length does not match position");
    if (pos0 + n > m->max_seq) return fail(FFB_VALIDATION, "prefill: positions exceed the KV cache");
    const int64_t B = c.batch, rows = n * B;
    for (int64_t i = 0; i < rows; ++i)
        if (tokens[i] < 0 || tokens[i] >= m->gcfg.vocab_size)
            return fail(FFB_VALIDATION, "prefill: token id out of range");
    if (rows > 1024) return fail(FFB_USAGE, "prefill: at most 1024 activation rows per call (n * batch)");
    const int D = (int)c.d_model, DI = (int)c.d_inter, DH = (int)c.d_head, NQ = (int)c.n_q_heads,
              NKV = (int)c.n_kv_heads, V = (int)c.vocab_size;
    const int QR = NQ * DH, QKVR = (int)m->qkv_rows(), AD = QR;
    if ((DH != 32 && DH != 64 && DH != 128) || kPairs % (NQ / NKV) != 0)
        return fail(FFB_UNSUPPORTED, "prefill: head shape (d_head 32 / 64 / 128, q heads per kv head dividing 64)");
    CUDA_TRY(cudaSetDevice(m->device));
    cudaStream_t s = m->stream;
    // scratch (kept; sized for the largest call so far)
    const int Kmax = std::max({D, AD, DI});
    const size_t Cn = 3 * std::max<size_t>((size_t)rows * std::max({QKVR, 2 * DI, D}), (size_t)B * V);
    const size_t need = ((size_t)rows * (D + QR + AD + DI) + Cn) * 4 + (size_t)3 * rows * Kmax * 2 + rows * 8 + 256;
    if (m->pf_bytes < need) {
        if (m->pf_buf) cudaFree(m->pf_buf);
        m->pf_buf = nullptr;
        m->pf_bytes = 0;
        CUDA_TRY(cudaMalloc(&m->pf_buf, need));
        m->pf_bytes = need;
    }
    auto* X = static_cast<float*>(m->pf_buf);
    float* Q = X + (size_t)rows * D;
    float* A = Q + (size_t)rows * QR;
    float* H = A + (size_t)rows * AD;
    float* C = H + (size_t)rows * DI;
    auto* Y3 = reinterpret_cast<__nv_bfloat16*>(C + Cn);
    auto* tok = reinterpret_cast<int64_t*>(
        (reinterpret_cast<uintptr_t>(Y3 + (size_t)3 * rows * Kmax) + 15) & ~uintptr_t(15));
    static bool attn_attr = [] {
        cudaFuncSetAttribute(k_attention<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<32>::BYTES);
        cudaFuncSetAttribute(k_attention<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<64>::BYTES);
        cudaFuncSetAttribute(k_attention<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, AttnSmem<128>::BYTES);
        return true;
    }();
    (void)attn_attr;
    if (!m->cublas) {
        cublasHandle_t h = nullptr;
        if (cublas()->create(&h) != 0) return fail(FFB_DEVICE, "prefill: cublasCreate failed");
        m->cublas = h;
        m->cublas_destroy = [](void* hd) { cublas()->destroy(static_cast<cublasHandle_t>(hd)); };
    }
    auto h = static_cast<cublasHandle_t>(m->cublas);
    cublas()->set_stream(h, s);
    CUDA_TRY(cudaMemcpyAsync(tok, tokens, sizeof(int64_t) * rows, cudaMemcpyHostToDevice, s));
    const auto* RB = m->ops;
    k_embed<<<(int)rows, 256, 0, s>>>(X, m->embedding, tok, (int)rows, D);
    const float eps = static_cast<float>(c.rmsnorm_eps);
    for (int64_t l = 0; l < c.layers; ++l) {
        const int64_t layer_off = l * B * NKV * m->max_seq * DH;
        k_norm_split<<<(int)rows, 256, 0, s>>>(X, m->norm_attn + l * D, eps, Y3, (int)rows, D);
        ffb_status st = gemm3(h, Y3, (int)rows, D, m->wqkv + (size_t)l * QKVR * RB->row_bytes, QKVR, false, C);
        if (st) return st;
        k_qkv_epilogue<<<(int)rows, 256, 0, s>>>(C, (size_t)rows * QKVR, Q, m->kcache, m->vcache, (int)rows, (int)B, NQ, NKV, DH,
                                                  pos0, c.rope_theta, layer_off, m->max_seq);
        const int tq = kPairs / (NQ / NKV);
        const dim3 ag((unsigned)((n + tq - 1) / tq), (unsigned)NKV, (unsigned)B);
        if (DH == 64)
            k_attention<64><<<ag, 256, AttnSmem<64>::BYTES, s>>>(Q, m->kcache, m->vcache, A, (int)B, NQ, NKV,
                                                                 (int)n, pos0, layer_off, m->max_seq);
        else if (DH == 128)
            k_attention<128><<<ag, 256, AttnSmem<128>::BYTES, s>>>(Q, m->kcache, m->vcache, A, (int)B, NQ, NKV,
                                                                   (int)n, pos0, layer_off, m->max_seq);
        else
            k_attention<32><<<ag, 256, AttnSmem<32>::BYTES, s>>>(Q, m->kcache, m->vcache, A, (int)B, NQ, NKV,
                                                                 (int)n, pos0, layer_off, m->max_seq);
        k_norm_split<<<(int)rows, 256, 0, s>>>(A, nullptr, 0.f, Y3, (int)rows, AD);
        st = gemm3(h, Y3, (int)rows, AD, m->waout + (size_t)l * D * RB->row_bytes_a, D, false, C);
        if (st) return st;
        k_add<<<592, 256, 0, s>>>(X, C, (size_t)rows * D);
        k_norm_split<<<(int)rows, 256, 0, s>>>(X, m->norm_ffn + l * D, eps, Y3, (int)rows, D);
        st = gemm3(h, Y3, (int)rows, D, m->wffn1 + (size_t)l * 2 * DI * RB->row_bytes, 2 * DI, false, C);
        if (st) return st;
        k_silu<<<592, 256, 0, s>>>(C, (size_t)rows * 2 * DI, H, (int)rows, DI);
        k_norm_split<<<(int)rows, 256, 0, s>>>(H, nullptr, 0.f, Y3, (int)rows, DI);
        // W2: [D][DI] rows (two-phase FFN shapes) or Wffn2^T [DI][D]
        st = gemm3(h, Y3, (int)rows, DI, m->wffn2t + (size_t)l * D * DI * 2, D, !RB->ffn2_rows, C);
        if (st) return st;
        k_add<<<592, 256, 0, s>>>(X, C, (size_t)rows * D);
    }
    // LM head on the last position of every batch row
    const float* xl = X + (size_t)(n - 1) * B * D;
    k_norm_split<<<(int)B, 256, 0, s>>>(xl, m->final_norm, eps, Y3, (int)B, D);
    ffb_status st = gemm3(h, Y3, (int)B, D, m->lm_head, V, false, C);
    if (st) return st;
    k_sum3<<<592, 256, 0, s>>>(C, (size_t)B * V);
    k_argmax<<<(int)B, 256, 0, s>>>(C, V, tok);
    CUDA_TRY(cudaGetLastError());
    if (logits) CUDA_TRY(cudaMemcpyAsync(logits, C, sizeof(float) * B * V, cudaMemcpyDeviceToHost, s));
    if (greedy) CUDA_TRY(cudaMemcpyAsync(greedy, tok, sizeof(int64_t) * B, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t l = 0; l < c.layers; ++l) m->kv_len[l] = pos0 + n;
    return FFB_OK;
}
