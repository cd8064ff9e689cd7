// Specialisations for the Llama-3.1-8B shape E (presets.hpp:21-29), the
// headline roofline config.
#include "kernel_ops.cuh"

namespace ffb200 {
void register_kernels_8b(std::vector<KernelOps>& v) {
    v.push_back(make_ops<Shape<4096, 14336, 128, 32, 8, 1>>());
    v.push_back(make_ops<Shape<4096, 14336, 128, 32, 8, 2>>());
    v.push_back(make_ops<Shape<4096, 14336, 128, 32, 8, 4>>());
}
}  // namespace ffb200
