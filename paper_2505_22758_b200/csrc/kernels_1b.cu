// Specialisations for the Llama-3.2-1B shape S.
#include "kernel_ops.cuh"

namespace ffb200 {
void register_kernels_1b(std::vector<KernelOps>& v) {
    v.push_back(make_ops<Shape<2048, 8192, 64, 32, 8, 1>>());
    v.push_back(make_ops<Shape<2048, 8192, 64, 32, 8, 4>>());
}
}  // namespace ffb200
