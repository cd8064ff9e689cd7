// Llama-3-70B shape H (d_model 8192, 64 q / 8 kv heads, d_inter 28672,
// SURVEY.md §8) as the whole model (TP 1: 141 GB of bf16 weights fit one
// B200) and as the tensor-parallel shards of TP 2 / 4 / 8 (kv heads, q heads
// and d_inter divided by TP; d_model replicated).  8B / tiny shards:
// kernels_tp.cu.
#include "kernel_ops.cuh"

namespace ffb200 {
void register_kernels_70b(std::vector<KernelOps>& v) {
    v.push_back(make_ops<Shape<8192, 28672, 128, 64, 8, 1>>());
    v.push_back(make_ops<Shape<8192, 14336, 128, 32, 4, 1>>());
    v.push_back(make_ops<Shape<8192, 7168, 128, 16, 2, 1>>());
    v.push_back(make_ops<Shape<8192, 3584, 128, 8, 1, 1>>());
}
}  // namespace ffb200
