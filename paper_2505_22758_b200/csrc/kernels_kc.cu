// Batch >= 8 specialisations (Shape::KCP: K-chunked tensor-core GEMVs):
// the toy parity shape, the tiny config T, and Llama-3.1-8B (config E lists
// batch 16).
#include "kernel_ops.cuh"

namespace ffb200 {
void register_kernels_kc(std::vector<KernelOps>& v) {
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 16>>());
    v.push_back(make_ops<Shape<256, 896, 64, 4, 2, 8>>());
    v.push_back(make_ops<Shape<512, 1792, 64, 8, 2, 16>>());
    // parity shapes with the 8B geometry (512-column K chunks) at small width;
    // the second also runs one attention CTA per (row, kv head)
    v.push_back(make_ops<Shape<512, 2048, 64, 8, 2, 16>>());
    v.push_back(make_ops<Shape<2048, 2048, 64, 32, 8, 16>>());
    v.push_back(make_ops<Shape<4096, 14336, 128, 32, 8, 16>>());
    v.push_back(make_ops<Shape<4096, 14336, 128, 32, 8, 8>>());
}
}  // namespace ffb200
