// kernel_ops.cuh -- type-erased handle on one compile-time specialisation of
// the decode kernel.  Each kernels_*.cu translation unit instantiates a few
// shapes (compiled in parallel) and registers them here; the runtime picks
// the entry whose shape equals the model config (SURVEY.md §7 hard part 9:
// instantiate only the shapes that are used).
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "decode_kernel.cuh"

namespace ffb200 {

struct KernelOps {
    int D, DI, DH, NQ, NKV, B, QB;
    int threads, smem, nslots, slot_bytes, rg, tmax, kvc, rps, row_bytes, row_bytes_a;
    int tc_d, tc_a;  // d_model-column / Waout rows use the tensor-core code order
    int ffn2_rows;   // W2 stored [D][DI] (two-phase FFN, KTraits::F2R), else Wffn2^T
    int kc;          // batch >= 8: K-chunk width of the chunk-major matrix layout (0: row-major)
    int kc_layout;   // batch >= 8 weight / A-table layout: 2 = mma.sync, 3 = tcgen05 (FFB_KCP_TCGEN05)
    cudaError_t (*prepare)();
    cudaError_t (*launch)(const DecodeParams&, int grid, cudaStream_t, bool cooperative);
};

template <class S>
cudaError_t prepare_impl() {
    using T = KTraits<S>;
    return cudaFuncSetAttribute(decode_step_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                T::SMEM_BYTES);
}

template <class S>
cudaError_t launch_impl(const DecodeParams& p, int grid, cudaStream_t stream, bool cooperative) {
    using T = KTraits<S>;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(T::NTHREADS);
    cfg.dynamicSmemBytes = T::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = cooperative ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, decode_step_kernel<S>, p);
}

template <class S>
KernelOps make_ops() {
    using T = KTraits<S>;
    return KernelOps{S::D,        S::DI,         S::DH,     S::NQ,         S::NKV, S::B,
                     S::QB,       T::NTHREADS,   T::SMEM_BYTES, T::NSLOTS, T::SLOT_BYTES,
                     T::RG,       T::TMAX,       T::KVC,    T::RPS,        T::ROW_BYTES,
                     T::MA::ROW_BYTES, T::MD::TC ? 1 : 0, T::MA::TC ? 1 : 0, T::F2R ? 1 : 0, S::KCP ? S::KC : 0,
                     S::KCP ? kKcLayout : 0,
                     &prepare_impl<S>, &launch_impl<S>};
}

// registration hooks, one per kernels_*.cu
void register_kernels_small(std::vector<KernelOps>& v);
void register_kernels_1b(std::vector<KernelOps>& v);
void register_kernels_8b(std::vector<KernelOps>& v);
void register_kernels_quant(std::vector<KernelOps>& v);
void register_kernels_70b(std::vector<KernelOps>& v);
void register_kernels_kc(std::vector<KernelOps>& v);
void register_kernels_tp(std::vector<KernelOps>& v);

}  // namespace ffb200
