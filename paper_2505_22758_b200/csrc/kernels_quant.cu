// Weight-only quantized specialisations (BASELINE config Q: Llama-3.1-8B
// shape, int4 / int8, group 128, batch 1) and the toy / tiny parity shapes.
// int4 is the reference's scheme (quant.hpp:17-60); int8 its 255-level
// extension.
#include "kernel_ops.cuh"

namespace ffb200 {
void register_kernels_quant(std::vector<KernelOps>& v) {
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 1, 4>>());
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 4, 4>>());
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 1, 8>>());
    v.push_back(make_ops<Shape<512, 1792, 64, 8, 2, 1, 4>>());
    v.push_back(make_ops<Shape<4096, 14336, 128, 32, 8, 1, 4>>());
    v.push_back(make_ops<Shape<4096, 14336, 128, 32, 8, 1, 8>>());
}
}  // namespace ffb200
