// Tensor-parallel shards of Llama-3.1-8B (config E sharded over 2 / 4 / 8
// B200s: kv heads, q heads, d_inter and vocabulary divided by TP, d_model
// replicated) and of the tiny config T at TP 2 (single-GPU
// TP parity tests).  The 70B shards live in kernels_70b.cu.
#include "kernel_ops.cuh"

namespace ffb200 {
void register_kernels_tp(std::vector<KernelOps>& v) {
    v.push_back(make_ops<Shape<4096, 7168, 128, 16, 4, 1>>());  // 8B, TP 2
    v.push_back(make_ops<Shape<4096, 3584, 128, 8, 2, 1>>());   // 8B, TP 4
    v.push_back(make_ops<Shape<4096, 1792, 128, 4, 1, 1>>());   // 8B, TP 8
    v.push_back(make_ops<Shape<512, 896, 64, 4, 1, 1>>());      // tiny, TP 2
}
}  // namespace ffb200
