// tma_bw.cu -- microbenchmark: per-SM ingest rate of 1-D TMA bulk copies
// (cp.async.bulk global->smem, mbarrier ring) and of plain 128-bit LDG, from
// an L2-resident region and from a DRAM-sized region.  Developer tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw tools/tma_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2505_22758_b200/csrc/ptx.cuh"

using namespace ffb200;

constexpr int NSLOTS = 6, SLOT = 32768;

__global__ void __launch_bounds__(288, 1) tma_kernel(const uint8_t* src, size_t region, size_t per_cta,
                                                     int slot_bytes, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + NSLOTS;
    uint8_t* ring = smem + 1024;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSLOTS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 8);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const size_t base = (size_t)blockIdx.x * per_cta;
    const int n = (int)(per_cta / slot_bytes);
    if (threadIdx.x == 256) {
        const uint64_t pol = policy_evict_first();
        for (int i = 0; i < n; ++i) {
            const uint32_t s = i % NSLOTS, ph = (i / NSLOTS) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], slot_bytes);
            tma_load_1d(ring + s * SLOT, src + (base + (size_t)i * slot_bytes) % region, slot_bytes,
                        &full[s], pol);
        }
    } else if (threadIdx.x < 256) {
        uint32_t acc = 0;
        for (int i = 0; i < n; ++i) {
            const uint32_t s = i % NSLOTS, ph = (i / NSLOTS) & 1;
            mbar_wait(&full[s], ph);
            acc += reinterpret_cast<const uint32_t*>(ring + s * SLOT)[threadIdx.x];
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 0x12345678u) atomicAdd(sink, 1ull);
    }
}

__global__ void __launch_bounds__(256, 1) ldg_kernel(const uint4* src, size_t region16, size_t per_cta16,
                                                     unsigned long long* sink) {
    const size_t base = (size_t)blockIdx.x * per_cta16;
    uint32_t acc = 0;
    for (size_t i = threadIdx.x; i < per_cta16; i += 256 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const size_t k = i + (size_t)u * 256;
            v[u] = k < per_cta16 ? __ldcs(src + (base + k) % region16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t big = 8ull << 30;
    uint8_t* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, big);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, big);
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         1024 + NSLOTS * SLOT);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Case { const char* name; size_t region; int grid; int slot; };
    Case cases[] = {{"tma dram 8GB  148cta 32KB", big, sms, 32768},
                    {"tma dram 8GB  148cta 16KB", big, sms, 16384},
                    {"tma l2   48MB 148cta 32KB", 48ull << 20, sms, 32768},
                    {"tma l2   48MB  74cta 32KB", 48ull << 20, sms / 2, 32768},
                    {"tma l2   48MB  16cta 32KB", 48ull << 20, 16, 32768},
                    {"tma dram 8GB   16cta 32KB", big, 16, 32768}};
    for (auto& c : cases) {
        const size_t per_cta = (64ull << 20) / (size_t)c.slot * (size_t)c.slot / 4;  // 16 MB per CTA
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            tma_kernel<<<c.grid, 288, 1024 + NSLOTS * SLOT>>>(buf, c.region, per_cta, c.slot, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)per_cta * c.grid;
        printf("%-28s %8.1f GB/s total  %6.1f GB/s per CTA\n", c.name, bytes / ms / 1e6,
               bytes / ms / 1e6 / c.grid);
    }
    struct LCase { const char* name; size_t region; int grid; };
    LCase lc[] = {{"ldg dram 8GB  148cta", big, sms}, {"ldg l2   48MB 148cta", 48ull << 20, sms},
                  {"ldg l2   48MB  16cta", 48ull << 20, 16}};
    for (auto& c : lc) {
        const size_t per_cta16 = (16ull << 20) / 16;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            ldg_kernel<<<c.grid, 256>>>(reinterpret_cast<const uint4*>(buf), c.region / 16,
                                        per_cta16, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)per_cta16 * 16 * c.grid;
        printf("%-28s %8.1f GB/s total  %6.1f GB/s per CTA\n", c.name, bytes / ms / 1e6,
               bytes / ms / 1e6 / c.grid);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
