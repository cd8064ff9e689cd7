// Legacy tensor-core issue rate on this GPU: mma.sync f16 m16n8k16 vs
// s8 m16n8k32, independent chains per warp, W warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdint>
__global__ void k_f16(float* out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0; for (int j = 0; j < 4; ++j) for (int e = 0; e < 4; ++e) s += c[j][e];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_s8(float* out, int iters) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    int c[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0; for (int j = 0; j < 4; ++j) for (int e = 0; e < 4; ++e) s += c[j][e];
    if (s == 12345) out[0] = s;
}
int main() {
    float* d; cudaMalloc(&d, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        for (int kind = 0; kind < 2; ++kind) {
            for (int r = 0; r < 2; ++r) {
                cudaEventRecord(e0);
                if (kind == 0) k_f16<<<148, warps * 32>>>(d, iters); else k_s8<<<148, warps * 32>>>(d, iters);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                double mmas = 148.0 * warps * iters * 4;
                double macs = mmas * (kind == 0 ? 16 * 8 * 16 : 16 * 8 * 32);
                if (r) printf("%s warps/SM %2d: %.3f ms, %.2f mma/clk/SM (1.9 GHz), %.0f TOPS\n", kind ? "s8  k32" : "f16 k16",
                              warps, ms, mmas / 148 / (ms * 1e-3 * 1.9e9), 2 * macs / (ms * 1e-3) / 1e12);
            }
        }
    }
    return 0;
}
