// bridge_parity.cpp -- the reference's own C++ objects driving the B200 kernel.
//
// Built by __graft_entry__.build() against the UNMODIFIED reference headers
// (/root/reference/proj/include) and include/ffb200/fusesim_bridge.hpp, linked
// to the in-tree libffb200.so.  Runs on the GPU box (no reference sources are
// read at run time).  Mirrors proj/tests/test_interpreter.cpp:51-70: a
// fusesim::init_weights store of llama31_8b-toy, synthetic prefill, then
// fusesim::reference_forward vs fusesim::b200::Decoder::forward, rel_err
// < 1e-4 (plain) or, when a bf16 K/V rounding flip occurred, < 5e-4.
// Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <random>

#include "fusesim/presets.hpp"
#include "fusesim/reference.hpp"
#include "ffb200/fusesim_bridge.hpp"

using namespace fusesim;

static void synthetic_prefill(TensorStore& st, int64_t prefill, uint64_t seed) {
    const ModelConfig& m = st.model;  // test_interpreter.cpp:16-30
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> dist(0.0f, 0.3f);
    std::vector<float> k(m.d_head), v(m.d_head);
    for (int64_t b = 0; b < m.batch; ++b)
        for (int64_t l = 0; l < m.layers; ++l)
            for (int64_t h = 0; h < m.n_kv_heads; ++h)
                for (int64_t p = 0; p < prefill; ++p) {
                    for (auto& x : k) x = dist(rng);
                    for (auto& x : v) x = dist(rng);
                    st.kv.set_position(b, l, h, p, k.data(), v.data());
                }
    for (int64_t l = 0; l < m.layers; ++l) st.kv.set_length(l, prefill);
}

int main() {
    ModelConfig m = model_preset("llama31_8b-toy");
    int failures = 0;
    for (int64_t prefill : {0, 1, 255, 256, 300}) {
        TensorStore ref = init_weights(m, 42, prefill + 4);
        synthetic_prefill(ref, prefill, 7);
        auto want = reference_forward(ref, {17}, prefill);

        TensorStore st = init_weights(m, 42, prefill + 4);
        synthetic_prefill(st, prefill, 7);
        b200::Decoder dec(st, prefill + 4, RunMode::FusedOverlap);
        auto got = dec.forward(st, {17}, prefill);

        double scale = 0, err = 0;
        for (double w : want[0]) scale = std::max(scale, std::abs(w));
        for (size_t i = 0; i < got[0].size(); ++i)
            err = std::max(err, std::abs(got[0][i] - want[0][i]) / scale);
        int flips = 0;
        for (int64_t l = 0; l < m.layers; ++l)
            for (int64_t h = 0; h < m.n_kv_heads; ++h)
                for (int64_t d = 0; d < m.d_head; ++d) {
                    flips += st.kv.k_at(0, l, h, prefill)[d] != ref.kv.k_at(0, l, h, prefill)[d];
                    flips += st.kv.v_at(0, l, h, prefill)[d] != ref.kv.v_at(0, l, h, prefill)[d];
                }
        const bool ok = (flips == 0 ? err < 1e-4 : err < 5e-4) && st.kv.length(0) == prefill + 1;
        std::printf("prefill %4lld: rel_err %.3e, bf16 K/V flips %d, store length %lld  %s\n",
                    (long long)prefill, err, flips, (long long)st.kv.length(0), ok ? "ok" : "FAIL");
        failures += !ok;
    }
    // validation errors surface as the reference's exception type
    TensorStore st = init_weights(m, 1, 4);
    b200::Decoder dec(st, 4);
    try {
        dec.forward(st, {m.vocab_size}, 0);
        std::printf("missing ValidationError  FAIL\n");
        ++failures;
    } catch (const ValidationError& e) {
        std::printf("ValidationError: %s  ok\n", e.what());
    }
    return failures == 0 ? 0 : 1;
}
