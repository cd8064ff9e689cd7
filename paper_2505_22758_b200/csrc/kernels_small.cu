// Specialisations for the parity shapes: fusesim's llama31_8b-toy preset
// (presets.hpp:39-47) and the BASELINE "tiny" config T.
#include "kernel_ops.cuh"

namespace ffb200 {
void register_kernels_small(std::vector<KernelOps>& v) {
    // llama31_8b-toy: d 256, d_inter 896, d_head 64, 4 q / 2 kv heads
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 1>>());
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 2>>());
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 4>>());
    // tiny T: d 512, d_inter 1792, d_head 64, 8 q / 2 kv heads
    v.push_back(make_ops<Shape<512, 1792, 64, 8, 2, 1>>());
    v.push_back(make_ops<Shape<512, 1792, 64, 8, 2, 4>>());
}
}  // namespace ffb200
