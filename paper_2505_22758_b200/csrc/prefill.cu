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
// Numerics.  Every GEMM input activation (f32) is split into three bf16
// terms (hi + mid + lo carry 24 bits, the f32 mantissa; option
// "prefill_terms" = 2 keeps hi + lo) and ONE GEMM over the stacked terms runs
// the bf16 x bf16 products with f32 accumulation (cublasGemmEx,
// CUBLAS_COMPUTE_32F) -- f32-accurate products on the bf16 tensor cores; the
// consumers add the term planes.  The weights enter exactly: bf16 as stored;
// int4 / int8 expanded per projection into three bf16 planes of
// (code - zero) * scale (k_dequant3; three accumulated GEMMs); batch >= 8
// unpacked from the decode kernel's fp16 tensor-core layouts (k_unpack_kc).
// Attention (mma.sync, q and P as bf16 hi + lo like the decode kernel's) and
// everything elementwise is f32; K/V are rounded to bf16 at append, as
// reference.hpp / KVCache::append do.
//
// cuBLAS is loaded at run time (dlopen "libcublas.so.12"): plain library
// GEMMs only, the decode path never touches it.  One GPU (tensor-parallel
// shards return FFB_UNSUPPORTED).
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
    const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(emb + (size_t)tok[r] * D);
    float2* xr = reinterpret_cast<float2*>(x + (size_t)r * D);
    for (int c = threadIdx.x; c < D / 2; c += blockDim.x) xr[c] = __bfloat1622float2(e[c]);
}

__device__ __forceinline__ void split3(float v, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
    a = __float2bfloat16_rn(v);
    const float r1 = v - __bfloat162float(a);
    b = __float2bfloat16_rn(r1);
    c = __float2bfloat16_rn(r1 - __bfloat162float(b));
}

// four consecutive values split into the three bf16 planes (8-byte stores)
__device__ __forceinline__ void put_split4(__nv_bfloat16* y3, size_t plane, size_t i, float4 v) {
    __nv_bfloat16 h[4], m[4], l[4];
    split3(v.x, h[0], m[0], l[0]);
    split3(v.y, h[1], m[1], l[1]);
    split3(v.z, h[2], m[2], l[2]);
    split3(v.w, h[3], m[3], l[3]);
    *reinterpret_cast<uint2*>(y3 + i) = *reinterpret_cast<const uint2*>(h);
    *reinterpret_cast<uint2*>(y3 + plane + i) = *reinterpret_cast<const uint2*>(m);
    *reinterpret_cast<uint2*>(y3 + 2 * plane + i) = *reinterpret_cast<const uint2*>(l);
}

// one element of a split-term GEMM result: (hi + mid) + lo planes
// (nt = 2: the two-term split, option "prefill_terms", no lo plane)
__device__ __forceinline__ float ld3(const float* c, size_t plane, size_t i, int nt) {
    return (c[i] + c[plane + i]) + (nt == 3 ? c[2 * plane + i] : 0.f);
}
__device__ __forceinline__ float4 ld3x4(const float* c, size_t plane, size_t i, int nt) {
    const float4 a = *reinterpret_cast<const float4*>(c + i);
    const float4 b = *reinterpret_cast<const float4*>(c + plane + i);
    const float4 d = nt == 3 ? *reinterpret_cast<const float4*>(c + 2 * plane + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    return make_float4((a.x + b.x) + d.x, (a.y + b.y) + d.y, (a.z + b.z) + d.z, (a.w + b.w) + d.w);
}

// Residual row update + RMSNorm + split, one block (256 threads) per row:
// x += c3 (the three planes of a projection, when c3 != nullptr), then
// y = gain * x / sqrt(mean(x^2) + eps) (numerics.hpp:14-24) split into the
// three bf16 planes of the next GEMM's input.  K % 4 == 0, K <= 8192.
constexpr int kRowThreads = 256, kRowVec = 8;  // float4 per thread: K <= 256 * 4 * 8
__global__ void __launch_bounds__(kRowThreads) k_residual_norm_split(float* __restrict__ x, const float* __restrict__ c3,
                                                                     size_t cplane, const float* __restrict__ gain,
                                                                     float eps, __nv_bfloat16* __restrict__ y3,
                                                                     int rows, int K, int nt) {
    const int r = blockIdx.x;
    float4* xr = reinterpret_cast<float4*>(x + (size_t)r * K);
    const int nv = K / 4;
    float4 v[kRowVec];
    float ss = 0.f;
#pragma unroll
    for (int u = 0; u < kRowVec; ++u) {
        const int c = threadIdx.x + u * kRowThreads;
        if (c < nv) {
            float4 a = xr[c];
            if (c3 != nullptr) {
                const float4 d = ld3x4(c3, cplane, (size_t)r * K + 4 * c, nt);
                a = make_float4(a.x + d.x, a.y + d.y, a.z + d.z, a.w + d.w);
                xr[c] = a;
            }
            v[u] = a;
            ss = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, ss))));
        }
    }
    __shared__ float part[kRowThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kRowThreads / 32; ++w) t += part[w];
    const float inv = 1.0f / sqrtf(t / static_cast<float>(K) + eps);
    const size_t plane = (size_t)rows * K;
#pragma unroll
    for (int u = 0; u < kRowVec; ++u) {
        const int c = threadIdx.x + u * kRowThreads;
        if (c < nv) {
            const float4 g = reinterpret_cast<const float4*>(gain)[c];
            put_split4(y3, plane, (size_t)r * K + 4 * c,
                       make_float4(g.x * v[u].x * inv, g.y * v[u].y * inv, g.z * v[u].z * inv, g.w * v[u].w * inv));
        }
    }
}

// h = silu(gate) * in over the interleaved (in, gate) columns of the Wffn1
// output (three planes), split straight into the W2 GEMM's input planes
__global__ void k_silu_split(const float* __restrict__ c3, size_t cplane, __nv_bfloat16* __restrict__ y3, int rows,
                             int DI, int nt) {
    const size_t n4 = (size_t)rows * DI / 4, plane = (size_t)rows * DI;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const float4 a = ld3x4(c3, cplane, 8 * i, nt), b = ld3x4(c3, cplane, 8 * i + 4, nt);
        const float4 h = make_float4(a.y / (1.0f + expf(-a.y)) * a.x, a.w / (1.0f + expf(-a.w)) * a.z,
                                     b.y / (1.0f + expf(-b.y)) * b.x, b.w / (1.0f + expf(-b.w)) * b.z);
        put_split4(y3, plane, 4 * i, h);
    }
}

// RoPE table of the call's positions: (cos, sin) of pos * theta^(-2k/dh),
// angle in f64 as numerics.hpp:27-37 / the decode kernel; [n][dh / 2]
__global__ void k_rope_table(float2* __restrict__ tab, int n, int64_t pos0, int DH, double theta) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * (DH / 2)) return;
    const int t = i / (DH / 2), k = i % (DH / 2);
    const double freq = pow(theta, -static_cast<double>(2 * k) / DH);
    const double ang = static_cast<double>(pos0 + t) * freq;
    tab[i] = make_float2(static_cast<float>(cos(ang)), static_cast<float>(sin(ang)));
}

__device__ __forceinline__ int swz(int d, int64_t pos) { return ((((d >> 3) ^ (int)(pos & 7))) << 3) | (d & 7); }

// RoPE (interleaved pairs) on the q and k columns of the QKV output; K and V
// rounded to bf16 and appended at position pos0 + t of batch row b; q (f32)
// kept for attention.  Activation row r = t * B + b; one thread per 4
// columns (two rotary pairs, one half 16-byte chunk of a K/V row).
__global__ void k_qkv_epilogue(const float* __restrict__ qkv, size_t plane, const float2* __restrict__ rope,
                               float* __restrict__ q, __nv_bfloat16* kc, __nv_bfloat16* vc, int rows, int B, int NQ,
                               int NKV, int DH, int64_t pos0, int64_t layer_off, int64_t max_seq, int nt) {
    const int QR = NQ * DH, KR = NKV * DH, QKVR = QR + 2 * KR;
    const size_t n4 = (size_t)rows * QKVR / 4;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const size_t r = 4 * i / QKVR;
        const int g = (int)(4 * i - r * QKVR);
        const int t = (int)(r / B), b = (int)(r % B);
        const int64_t pos = pos0 + t;
        float4 v = ld3x4(qkv, plane, 4 * i, nt);
        const int dim = g % DH;
        if (g < QR + KR) {
            const float2 cs0 = rope[t * (DH / 2) + dim / 2], cs1 = rope[t * (DH / 2) + dim / 2 + 1];
            v = make_float4(v.x * cs0.x - v.y * cs0.y, v.x * cs0.y + v.y * cs0.x, v.z * cs1.x - v.w * cs1.y,
                            v.z * cs1.y + v.w * cs1.x);
            if (g < QR) {
                *reinterpret_cast<float4*>(q + r * QR + g) = v;
                continue;
            }
        }
        const bool is_k = g < QR + KR;
        const int h = (g - QR - (is_k ? 0 : KR)) / DH;
        __nv_bfloat16* row = (is_k ? kc : vc) + layer_off + (((size_t)b * NKV + h) * max_seq + pos) * DH;
        __nv_bfloat16 o4[4] = {__float2bfloat16_rn(v.x), __float2bfloat16_rn(v.y), __float2bfloat16_rn(v.z),
                               __float2bfloat16_rn(v.w)};
        *reinterpret_cast<uint2*>(row + swz(dim, pos)) = *reinterpret_cast<const uint2*>(o4);
    }
}

// Causal attention on the tensor cores (mma.sync m16n8k16 bf16, f32
// accumulate), FlashAttention-2 style.  One block (4 warps) per (query tile,
// kv head, batch row) holds kPairs = 64 (prompt position, q head) rows of one
// GQA group -- kPairs / QPG consecutive positions x the group's QPG heads,
// all reading the same K/V -- warp w owning rows [16 w, 16 w + 16).  Keys
// [0, last position of the tile] stream through shared memory in tiles of
// kKeys (cp.async, double-buffered, un-swizzled from the cache's chunk order,
// rows padded so ldmatrix is conflict free).  Precision follows the decode
// kernel's tensor-core attention (decode_kernel.cuh attn_warp_pass): q enters
// as bf16 hi + lo (two MMAs), scores in f32 (log2 units, exp2), P as bf16
// hi + lo (two MMAs) against the bf16 V, O in f32; online softmax per row.
constexpr int kPairs = 64, kKeys = 64, kAttnThreads = 128;

template <int DH>
struct AttnSmem {
    static constexpr int RB = DH * 2 + 16;  // bytes per staged K / V row (padded)
    static constexpr int TILE = kKeys * RB;
    static constexpr int BYTES = 4 * TILE;  // K, V x 2 buffers
};

__device__ __forceinline__ uint32_t bf2(float lo_elem, float hi_elem) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}

template <int DH>
__global__ void __launch_bounds__(kAttnThreads) k_attention(const float* __restrict__ q,
                                                            const __nv_bfloat16* __restrict__ kc,
                                                            const __nv_bfloat16* __restrict__ vc,
                                                            __nv_bfloat16* __restrict__ y3, size_t oplane, int B,
                                                            int NQ, int NKV, int n, int64_t pos0, int64_t layer_off,
                                                            int64_t max_seq) {
    using SM = AttnSmem<DH>;
    constexpr int KS = DH / 16, CH = DH / 8;  // k-steps over d_head, 16-byte chunks per row
    extern __shared__ __align__(128) uint8_t sm[];
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q4 = lane & 3;
    const int qpg = NQ / NKV, tq = kPairs / qpg;
    const int t0 = blockIdx.x * tq, kvh = blockIdx.y, b = blockIdx.z;
    const int tlast = min(t0 + tq, n) - 1;
    const int64_t kend = pos0 + tlast + 1;  // keys of the whole tile
    const __nv_bfloat16* kb = kc + layer_off + ((size_t)b * NKV + kvh) * max_seq * DH;
    const __nv_bfloat16* vb = vc + layer_off + ((size_t)b * NKV + kvh) * max_seq * DH;

    auto load_tile = [&](int64_t k0, int buf) {
        const uint32_t kd = sbase + (2 * buf) * SM::TILE, vd = kd + SM::TILE;
        for (int i = threadIdx.x; i < kKeys * CH; i += kAttnThreads) {
            const int j = i / CH, c = i % CH;
            const int64_t pos = k0 + j;
            const bool ok = pos < kend;
            const int64_t ps = ok ? pos : 0;
            const int cs = c ^ (int)(ps & 7);  // the cache's chunk swizzle (kv_swz)
            cp_async16(kd + j * SM::RB + c * 16, kb + ps * DH + cs * 8, ok);
            cp_async16(vd + j * SM::RB + c * 16, vb + ps * DH + cs * 8, ok);
        }
        asm volatile("cp.async.commit_group;");
    };
    load_tile(0, 0);

    // this warp's rows g and g + 8: pair 16 w + r -> (position, head)
    const int pr0 = 16 * warp + g, pr1 = pr0 + 8;
    const int64_t qp0 = pos0 + min(t0 + pr0 / qpg, tlast), qp1 = pos0 + min(t0 + pr1 / qpg, tlast);
    const int64_t wend = pos0 + min(t0 + (16 * warp + 15) / qpg, tlast) + 1;
    // q (pre-scaled by log2(e) / sqrt(d_head)) as A fragments, bf16 hi and lo
    uint32_t qh[KS][4], ql[KS][4];
    {
        const float alpha = 1.4426950408889634f / sqrtf(static_cast<float>(DH));
        const int ta = t0 + pr0 / qpg, tb = t0 + pr1 / qpg;
        const float* r0 = q + ((size_t)ta * B + b) * NQ * DH + (size_t)(kvh * qpg + pr0 % qpg) * DH;
        const float* r1 = q + ((size_t)tb * B + b) * NQ * DH + (size_t)(kvh * qpg + pr1 % qpg) * DH;
        const bool v0 = ta < n, v1 = tb < n;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const bool second = r & 1;
                const int d = kk * 16 + 2 * q4 + 8 * (r >> 1);
                const float* src = second ? r1 : r0;
                const bool ok = second ? v1 : v0;
                const float x0 = ok ? alpha * src[d] : 0.f, x1 = ok ? alpha * src[d + 1] : 0.f;
                qh[kk][r] = bf2(x0, x1);
                ql[kk][r] = bf2(x0 - bf_round(x0), x1 - bf_round(x1));
            }
    }
    float o[DH / 8][4];
#pragma unroll
    for (int c = 0; c < DH / 8; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[c][e] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    const int ntile = (int)((kend + kKeys - 1) / kKeys);
    for (int it = 0; it < ntile; ++it) {
        const int64_t k0 = (int64_t)it * kKeys;
        if (it + 1 < ntile) {
            load_tile(k0 + kKeys, (it + 1) & 1);
            asm volatile("cp.async.wait_group 1;");
        } else {
            asm volatile("cp.async.wait_group 0;");
        }
        __syncthreads();
        if (k0 < wend) {
            const uint32_t kt = sbase + (2 * (it & 1)) * SM::TILE, vt = kt + SM::TILE;
            // S = q K^T over the 64 keys: 8 n8 tiles
            float s[8][4];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
#pragma unroll
                for (int np = 0; np < 4; ++np) {  // pairs of n8 tiles: keys 16 np .. 16 np + 15
                    uint32_t b0, b1, b2, b3;
                    const int row = 16 * np + (lane & 7) + 8 * (lane >> 4), ch = 2 * kk + ((lane >> 3) & 1);
                    ldsm4(kt + row * SM::RB + ch * 16, b0, b1, b2, b3);
                    mma16816(s[2 * np], qh[kk], b0, b1);
                    mma16816(s[2 * np], ql[kk], b0, b1);
                    mma16816(s[2 * np + 1], qh[kk], b2, b3);
                    mma16816(s[2 * np + 1], ql[kk], b2, b3);
                }
            // causal mask, row max
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t kp = k0 + nt * 8 + 2 * q4 + e;
                    if (kp > qp0) s[nt][e] = -INFINITY;
                    if (kp > qp1) s[nt][e + 2] = -INFINITY;
                    mx0 = fmaxf(mx0, s[nt][e]);
                    mx1 = fmaxf(mx1, s[nt][e + 2]);
                }
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
            const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);  // finite: key 0 precedes every row
            const float sc0 = exp2f(m0 - mn0), sc1 = exp2f(m1 - mn1);
            m0 = mn0;
            m1 = mn1;
            float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                s[nt][0] = exp2f(s[nt][0] - mn0);
                s[nt][1] = exp2f(s[nt][1] - mn0);
                s[nt][2] = exp2f(s[nt][2] - mn1);
                s[nt][3] = exp2f(s[nt][3] - mn1);
                ps0 += s[nt][0] + s[nt][1];
                ps1 += s[nt][2] + s[nt][3];
            }
            ps0 += __shfl_xor_sync(0xffffffffu, ps0, 1);
            ps0 += __shfl_xor_sync(0xffffffffu, ps0, 2);
            ps1 += __shfl_xor_sync(0xffffffffu, ps1, 1);
            ps1 += __shfl_xor_sync(0xffffffffu, ps1, 2);
            l0 = l0 * sc0 + ps0;
            l1 = l1 * sc1 + ps1;
#pragma unroll
            for (int c = 0; c < DH / 8; ++c) {
                o[c][0] *= sc0;
                o[c][1] *= sc0;
                o[c][2] *= sc1;
                o[c][3] *= sc1;
            }
            // O += P V, P as bf16 hi + lo A fragments, V via ldmatrix.trans
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t ph[4], pl[4];
                const float* a = s[2 * j];
                const float* c2 = s[2 * j + 1];
                ph[0] = bf2(a[0], a[1]);
                ph[1] = bf2(a[2], a[3]);
                ph[2] = bf2(c2[0], c2[1]);
                ph[3] = bf2(c2[2], c2[3]);
                pl[0] = bf2(a[0] - bf_round(a[0]), a[1] - bf_round(a[1]));
                pl[1] = bf2(a[2] - bf_round(a[2]), a[3] - bf_round(a[3]));
                pl[2] = bf2(c2[0] - bf_round(c2[0]), c2[1] - bf_round(c2[1]));
                pl[3] = bf2(c2[2] - bf_round(c2[2]), c2[3] - bf_round(c2[3]));
                const int row = 16 * j + (lane & 7) + 8 * ((lane >> 3) & 1);
#pragma unroll
                for (int c = 0; c < DH / 16; ++c) {
                    uint32_t b00, b01, b10, b11;
                    ldsm4t(vt + row * SM::RB + (2 * c + (lane >> 4)) * 16, b00, b01, b10, b11);
                    mma16816(o[2 * c], ph, b00, b01);
                    mma16816(o[2 * c], pl, b00, b01);
                    mma16816(o[2 * c + 1], ph, b10, b11);
                    mma16816(o[2 * c + 1], pl, b10, b11);
                }
            }
        }
        __syncthreads();  // buffer (it & 1) is refilled by the next iteration's prefetch
    }
    // normalise, split straight into the Waout GEMM's input planes
    const int ta = t0 + pr0 / qpg, tb = t0 + pr1 / qpg;
    const float i0 = 1.0f / l0, i1 = 1.0f / l1;
    const size_t at0 = ((size_t)ta * B + b) * NQ * DH + (size_t)(kvh * qpg + pr0 % qpg) * DH;
    const size_t at1 = ((size_t)tb * B + b) * NQ * DH + (size_t)(kvh * qpg + pr1 % qpg) * DH;
#pragma unroll
    for (int c = 0; c < DH / 8; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int d = c * 8 + 2 * q4 + e;
            __nv_bfloat16 hi, mi, lo;
            if (ta < n) {
                split3(o[c][e] * i0, hi, mi, lo);
                y3[at0 + d] = hi;
                y3[oplane + at0 + d] = mi;
                y3[2 * oplane + at0 + d] = lo;
            }
            if (tb < n) {
                split3(o[c][e + 2] * i1, hi, mi, lo);
                y3[at1 + d] = hi;
                y3[oplane + at1 + d] = mi;
                y3[2 * oplane + at1 + d] = lo;
            }
        }
}

// LM head: the three planes summed in place into plane 0 (the logits) and
// a (max, lowest index) candidate per block of each row (numerics.hpp:169-175)
constexpr int kArgBlocks = 64;
constexpr int kQChunk = 16384;  // quantized weights: output rows dequantised per GEMM
__global__ void k_logits_part(float* __restrict__ c3, size_t plane, int V, float2* __restrict__ part, int nt) {
    const int b = blockIdx.y;
    float* row = c3 + (size_t)b * V;
    const int per = (V + kArgBlocks - 1) / kArgBlocks, i0 = blockIdx.x * per, i1 = min(V, i0 + per);
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const float v = ld3(row, plane, i, nt);
        row[i] = v;
        if (v > bv) {
            bv = v;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
        }
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = bv;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) {
                bv = sv[w];
                bi = si[w];
            }
        part[b * kArgBlocks + blockIdx.x] = make_float2(bv, __int_as_float(bi));
    }
}

__global__ void k_argmax_final(const float2* __restrict__ part, int64_t* __restrict__ out) {
    const int b = blockIdx.x;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int k = 0; k < kArgBlocks; ++k) {
        const float2 c = part[b * kArgBlocks + k];
        const int ci = __float_as_int(c.y);
        if (c.x > bv || (c.x == bv && ci < bi)) {
            bv = c.x;
            bi = ci;
        }
    }
    out[b] = bi;
}

// ---- quantized weights (int4 / int8): exact bf16 planes -------------------
// A packed row (decode_kernel.cuh row format: codes | f32 scales | u8 zeros)
// holds w = (code - zero) * scale, the reference's snapped f32 weight bit for
// bit (the packer accepts a group only if that product reproduces every
// value, runtime.cu quant_try); w is split into three bf16 planes (24 bits:
// exact) so the tensor cores see the weight itself.
// rows [r0, r0 + nr) of a packed matrix with K columns -> planes
// w3[p][row - r0][k] (plane stride nr * K).  One thread per 8 consecutive
// columns (consecutive lanes: consecutive 16-byte stores per plane).  In the
// tensor-core code order (runtime.cu tc_nibble_index / tc_byte_index)
// columns 32 st + 4q + j (j < 4) are the low nibbles / first 4 bytes of lane
// quad q's word / 8 bytes of k32-step st, columns 32 st + 16 + 4q + j the
// high nibbles / last 4 bytes; in the plain order codes follow the columns.
__global__ void k_dequant3(const uint8_t* __restrict__ w, size_t row_bytes, int r0, int nr, int K, int qb, int tc,
                           __nv_bfloat16* __restrict__ w3) {
    const int ng = K / kQuantGroup, code_bytes = qb == 4 ? K / 2 : K;
    const size_t plane = (size_t)nr * K, n8 = plane / 8;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n8; e += (size_t)gridDim.x * blockDim.x) {
        const int rr = (int)(e / (K / 8)), k0 = (int)(e % (K / 8)) * 8;
        const int g = k0 / kQuantGroup, i0 = k0 % kQuantGroup, st = i0 / 32, hh = (i0 % 32) / 16, q0 = (i0 % 16) / 4;
        const uint8_t* row = w + (size_t)(r0 + rr) * row_bytes;
        const float sc = *reinterpret_cast<const float*>(row + code_bytes + 4 * g);
        const float z = static_cast<float>(row[code_bytes + 4 * ng + g]);
        int code[8];
        if (qb == 4) {
            const uint8_t* grp = row + g * 64;
            if (tc) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {  // lane quads q0, q0 + 1
                    const uint32_t wd = *reinterpret_cast<const uint32_t*>(grp + (q0 + u) * 16 + st * 4);
#pragma unroll
                    for (int j = 0; j < 4; ++j) code[4 * u + j] = (wd >> (8 * j + 4 * hh)) & 0xF;
                }
            } else {
                const uint32_t wd = *reinterpret_cast<const uint32_t*>(grp + i0 / 2);
#pragma unroll
                for (int i = 0; i < 8; ++i) code[i] = (wd >> (4 * i)) & 0xF;
            }
        } else {
            const uint8_t* grp = row + g * 128;
            if (tc) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint32_t wd = *reinterpret_cast<const uint32_t*>(grp + (q0 + u) * 32 + st * 8 + 4 * hh);
#pragma unroll
                    for (int j = 0; j < 4; ++j) code[4 * u + j] = (wd >> (8 * j)) & 0xFF;
                }
            } else {
                const uint2 v = *reinterpret_cast<const uint2*>(grp + i0);
#pragma unroll
                for (int i = 0; i < 8; ++i) code[i] = ((i < 4 ? v.x : v.y) >> (8 * (i % 4))) & 0xFF;
            }
        }
        __nv_bfloat16 hi[8], mi[8], lo[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) split3(__fmul_rn(static_cast<float>(code[i]) - z, sc), hi[i], mi[i], lo[i]);
        __nv_bfloat16* dst = w3 + (size_t)rr * K + k0;
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(hi);
        *reinterpret_cast<uint4*>(dst + plane) = *reinterpret_cast<const uint4*>(mi);
        *reinterpret_cast<uint4*>(dst + 2 * plane) = *reinterpret_cast<const uint4*>(lo);
    }
}

// batch >= 8 weights (fp16 values of the bf16 weights, K-chunked and
// swizzled for the decode kernel's tensor-core GEMV, runtime.cu upload):
// rows [r0, r0 + nr) -> one bf16 plane w1[row - r0][k] = bf16(fp16 value).
// That recovers the original bf16 weight wherever the fp16 value is within
// half a bf16 ulp of it -- every value in the fp16 normal range and all but
// the smallest subnormals (below ~2^-17 the fp16 storage itself rounded;
// ffb_info.fp16_inexact counts those).  layout 2: [K / KC][rows][KC], 8-column
// units of a row segment XOR-swizzled by row & 7; layout 3 (tcgen05 build):
// [K / KC][rows / 8][KC / 64][8 rows][64], the same swizzle inside each
// 128-byte piece.
__global__ void k_unpack_kc(const __half* __restrict__ w, int rows, int r0, int nr, int K, int KC, int layout,
                            __nv_bfloat16* __restrict__ w1) {
    const size_t plane = (size_t)nr * K, n8 = plane / 8;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n8; e += (size_t)gridDim.x * blockDim.x) {
        const int rr = (int)(e / (K / 8)), k0 = (int)(e % (K / 8)) * 8, r = r0 + rr;
        const int c = k0 / KC, kk = k0 % KC;
        size_t pos;
        if (layout == 3) {
            const int ka = kk / 64, u = (kk % 64) / 8;
            pos = ((((size_t)c * (rows / 8) + r / 8) * (KC / 64) + ka) * 8 + (r & 7)) * 64 + ((u ^ (r & 7)) * 8);
        } else {
            pos = ((size_t)c * rows + r) * KC + (((kk / 8) ^ (r & 7)) * 8);
        }
        const uint4 v = *reinterpret_cast<const uint4*>(w + pos);
        const __half* hv = reinterpret_cast<const __half*>(&v);
        __nv_bfloat16 hi[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) hi[i] = __float2bfloat16_rn(__half2float(hv[i]));
        *reinterpret_cast<uint4*>(w1 + (size_t)rr * K + k0) = *reinterpret_cast<const uint4*>(hi);
    }
}

// C3[3][rows][N] (f32, row-major) = Y3[3][rows][K] . W^T: ONE GEMM over the
// 3 * rows stacked split-term rows, so W is read once; consumers add the
// three planes (ld3).  W bf16 row-major [N][K] (w_kn = false) or [K][N]
// (w_kn = true: Wffn2^T stored [DI][D])
ffb_status gemm3(cublasHandle_t h, const __nv_bfloat16* y3, int rows, int K, const void* W, int N, bool w_kn,
                 float* C3, int nt) {
    const float one = 1.f, zero = 0.f;
    // column-major view: C'[N][3 rows] = op(W') . Y'[K][3 rows]
    const int st = cublas()->gemm_ex(h, w_kn ? CUBLAS_OP_N : CUBLAS_OP_T, CUBLAS_OP_N, N, nt * rows, K, &one, W,
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
    if (c.kind != 0 || m->tp_size != 1) return fail(FFB_UNSUPPORTED, "prefill: decoder on one GPU");
    if (!cublas()) return fail(FFB_UNSUPPORTED, "prefill: cuBLAS not available (dlopen libcublas.so.12)");
    for (int64_t l = 0; l < c.layers; ++l)
        if (m->kv_len[l] != pos0)
            return fail(FFB_VALIDATION, "prefill: cache length does not match position");
    if (pos0 + n > m->max_seq) return fail(FFB_VALIDATION, "prefill: positions exceed the KV cache");
    const int64_t B = c.batch;
    int64_t rows = n * B;  // activation rows (the LM head runs on B of them)
    for (int64_t i = 0; i < rows; ++i)
        if (tokens[i] < 0 || tokens[i] >= m->gcfg.vocab_size)
            return fail(FFB_VALIDATION, "prefill: token id out of range");
    if (rows > 1024) return fail(FFB_USAGE, "prefill: at most 1024 activation rows per call (n * batch)");
    const int D = (int)c.d_model, DI = (int)c.d_inter, DH = (int)c.d_head, NQ = (int)c.n_q_heads,
              NKV = (int)c.n_kv_heads, V = (int)c.vocab_size;
    const int QR = NQ * DH, QKVR = (int)m->qkv_rows(), AD = QR;
    if ((DH != 64 && DH != 128) || kPairs % (NQ / NKV) != 0 || D > kRowThreads * 4 * kRowVec)
        return fail(FFB_UNSUPPORTED, "prefill: head shape (d_head 64 / 128, q heads per kv head dividing 64)");
    CUDA_TRY(cudaSetDevice(m->device));
    // steps enqueued asynchronously on any stream (ffb_decode_step_device,
    // ffb_decode_loop) write the cache this call extends: let them land
    CUDA_TRY(cudaDeviceSynchronize());
    cudaStream_t s = m->stream;
    // scratch (kept; sized for the largest call so far): residual X, rotated
    // q, the GEMM outputs C3 (three planes), the GEMM inputs Y3 (three bf16
    // planes), the RoPE table, token ids, argmax candidates
    const int Kmax = std::max({D, AD, DI});
    const size_t Cn = 3 * std::max<size_t>((size_t)rows * std::max({QKVR, 2 * DI, D}), (size_t)B * V);
    const bool quant = m->ops->QB != 0, kcp = m->ops->kc != 0;
    // quantized weights: a chunk of kQChunk rows dequantised into three bf16
    // planes (W3) per projection
    const size_t w3n = quant || kcp ? 3 * std::max<size_t>((size_t)std::min(kQChunk, std::max({QKVR, 2 * DI, D, V})) *
                                                        std::max(D, AD),
                                                    (size_t)DI * D)
                                    : 0;
    size_t need = 0;
    auto carve = [&](size_t bytes) {  // 256-byte aligned sub-buffers
        const size_t at = need;
        need += (bytes + 255) / 256 * 256;
        return at;
    };
    const size_t oX = carve((size_t)rows * D * 4), oQ = carve((size_t)rows * QR * 4), oC = carve(Cn * 4),
                 oR = carve((size_t)n * DH * 4), oP = carve((size_t)B * kArgBlocks * 8), oT = carve(rows * 8),
                 oY = carve((size_t)3 * rows * Kmax * 2), oW3 = carve(w3n * 2);
    if (m->pf_bytes < need) {
        if (m->pf_buf) cudaFree(m->pf_buf);
        m->pf_buf = nullptr;
        m->pf_bytes = 0;
        CUDA_TRY(cudaMalloc(&m->pf_buf, need));
        m->pf_bytes = need;
    }
    auto* base = static_cast<uint8_t*>(m->pf_buf);
    auto* X = reinterpret_cast<float*>(base + oX);
    auto* Q = reinterpret_cast<float*>(base + oQ);
    auto* C = reinterpret_cast<float*>(base + oC);
    auto* rope = reinterpret_cast<float2*>(base + oR);
    auto* part = reinterpret_cast<float2*>(base + oP);
    auto* tok = reinterpret_cast<int64_t*>(base + oT);
    auto* Y3 = reinterpret_cast<__nv_bfloat16*>(base + oY);
    auto* W3 = reinterpret_cast<__nv_bfloat16*>(base + oW3);
    static bool attn_attr = [] {
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
    const float eps = static_cast<float>(c.rmsnorm_eps);
    const int ew = 4 * m->grid;  // grid of the element-wise kernels
    const int at = m->prefill_terms;         // activation split terms: 3 (f32-exact products) or 2
    const int nt = at;                       // planes of a projection's output the consumers add
    // one projection: Y3 (rows x K activations, split) . W^T -> C
    auto proj = [&](int K, const uint8_t* W, size_t row_bytes, int N, bool kn, int tc) -> ffb_status {
        if (!quant && !kcp) return gemm3(h, Y3, (int)rows, K, W, N, kn, C, at);
        const float one = 1.f, zero = 0.f;
        const int wpl = quant ? 3 : 1;  // bf16 planes of the stored weight
        for (int n0 = 0; n0 < N; n0 += kn ? N : kQChunk) {
            const int nc = kn ? N : std::min(kQChunk, N - n0);
            // kn (Wffn2^T): the packed rows are the GEMM's K, their columns N
            if (kcp)
                k_unpack_kc<<<4 * m->grid, 256, 0, s>>>(reinterpret_cast<const __half*>(W), N, n0, nc, K, RB->kc,
                                                        RB->kc_layout, W3);
            else if (kn)
                k_dequant3<<<4 * m->grid, 256, 0, s>>>(W, row_bytes, 0, K, N, RB->QB, tc, W3);
            else
                k_dequant3<<<4 * m->grid, 256, 0, s>>>(W, row_bytes, n0, nc, K, RB->QB, tc, W3);
            // weight plane pw against activation terms a < at - pw, summed
            // into the activation-term planes of C (beta = 1 after plane 0):
            // C[a] = W_hi y_a + W_mid y_a + W_lo y_a over the significant pairs
            for (int pw = 0; pw < wpl && pw < at; ++pw) {
                const int na = at - pw;
                const __nv_bfloat16* A = W3 + (size_t)pw * nc * K;
                // C planes [a][rows][N] are the rows a * rows + r of one
                // [at * rows][N] matrix: one GEMM over the na stacked terms
                const int st = cublas()->gemm_ex(h, kn ? CUBLAS_OP_N : CUBLAS_OP_T, CUBLAS_OP_N, nc, na * (int)rows, K,
                                                 &one, A, kCUDA_R_16BF, kn ? N : K, Y3, kCUDA_R_16BF, K,
                                                 pw == 0 ? &zero : &one, C + n0, kCUDA_R_32F, N, kCUBLAS_COMPUTE_32F,
                                                 kCUBLAS_GEMM_DEFAULT);
                if (st != 0) return fail(FFB_DEVICE, "prefill: cublasGemmEx failed (status %d)", st);
            }
        }
        return FFB_OK;
    };
    k_rope_table<<<(int)((n * DH / 2 + 255) / 256), 256, 0, s>>>(rope, (int)n, pos0, DH, c.rope_theta);
    k_embed<<<(int)rows, 256, 0, s>>>(X, m->embedding, tok, (int)rows, D);
    k_residual_norm_split<<<(int)rows, kRowThreads, 0, s>>>(X, nullptr, 0, m->norm_attn, eps, Y3, (int)rows, D, nt);
    const size_t pD = (size_t)rows * D;
    for (int64_t l = 0; l < c.layers; ++l) {
        const int64_t layer_off = l * B * NKV * m->max_seq * DH;
        ffb_status st = proj(D, m->wqkv + (size_t)l * QKVR * RB->row_bytes, RB->row_bytes, QKVR, false, RB->tc_d);
        if (st) return st;
        k_qkv_epilogue<<<ew, 256, 0, s>>>(C, (size_t)rows * QKVR, rope, Q, m->kcache, m->vcache, (int)rows, (int)B,
                                          NQ, NKV, DH, pos0, layer_off, m->max_seq, nt);
        const int tq = kPairs / (NQ / NKV);
        const dim3 ag((unsigned)((n + tq - 1) / tq), (unsigned)NKV, (unsigned)B);
        const size_t ap = (size_t)rows * AD;
        if (DH == 64)
            k_attention<64><<<ag, kAttnThreads, AttnSmem<64>::BYTES, s>>>(Q, m->kcache, m->vcache, Y3, ap, (int)B, NQ, NKV,
                                                                 (int)n, pos0, layer_off, m->max_seq);
        else if (DH == 128)
            k_attention<128><<<ag, kAttnThreads, AttnSmem<128>::BYTES, s>>>(Q, m->kcache, m->vcache, Y3, ap, (int)B, NQ,
                                                                   NKV, (int)n, pos0, layer_off, m->max_seq);
        st = proj(AD, m->waout + (size_t)l * D * RB->row_bytes_a, RB->row_bytes_a, D, false, RB->tc_a);
        if (st) return st;
        k_residual_norm_split<<<(int)rows, kRowThreads, 0, s>>>(X, C, pD, m->norm_ffn + l * D, eps, Y3, (int)rows,
                                                               D, nt);
        st = proj(D, m->wffn1 + (size_t)l * 2 * DI * RB->row_bytes, RB->row_bytes, 2 * DI, false, RB->tc_d);
        if (st) return st;
        k_silu_split<<<ew, 256, 0, s>>>(C, (size_t)rows * 2 * DI, Y3, (int)rows, DI, nt);
        // W2: [D][DI] rows (two-phase FFN shapes) or Wffn2^T [DI][D]
        st = quant ? proj(DI, m->wffn2t + (size_t)l * DI * RB->row_bytes, RB->row_bytes, D, true, 0)
                   : proj(DI, m->wffn2t + (size_t)l * D * DI * 2, 0, D, !RB->ffn2_rows, 0);
        if (st) return st;
        if (l + 1 < c.layers) {
            k_residual_norm_split<<<(int)rows, kRowThreads, 0, s>>>(X, C, pD, m->norm_attn + (l + 1) * D, eps, Y3,
                                                                   (int)rows, D, nt);
        } else {  // only the last position of each batch row feeds the LM head
            const size_t o = (size_t)(n - 1) * B * D;
            k_residual_norm_split<<<(int)B, kRowThreads, 0, s>>>(X + o, C + o, pD, m->final_norm, eps, Y3, (int)B,
                                                                D, nt);
        }
    }
    if (c.layers == 0) {
        const size_t o = (size_t)(n - 1) * B * D;
        k_residual_norm_split<<<(int)B, kRowThreads, 0, s>>>(X + o, nullptr, 0, m->final_norm, eps, Y3, (int)B, D, nt);
    }
    // LM head on the last position of every batch row
    ffb_status st;
    {
        const int64_t rows_all = rows;
        rows = B;  // the LM head's rows: the last position of each batch row
        st = proj(D, m->lm_head, RB->row_bytes, V, false, RB->tc_d);
        rows = rows_all;
    }
    if (st) return st;
    k_logits_part<<<dim3(kArgBlocks, (unsigned)B), 256, 0, s>>>(C, (size_t)B * V, V, part, nt);
    k_argmax_final<<<(int)B, 1, 0, s>>>(part, tok);
    CUDA_TRY(cudaGetLastError());
    if (logits) CUDA_TRY(cudaMemcpyAsync(logits, C, sizeof(float) * B * V, cudaMemcpyDeviceToHost, s));
    if (greedy) CUDA_TRY(cudaMemcpyAsync(greedy, tok, sizeof(int64_t) * B, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t l = 0; l < c.layers; ++l) m->kv_len[l] = pos0 + n;
    return FFB_OK;
}
