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
#include <algorithm>
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
    // prompt ingestion: Decoder::prefill (GEMMs) vs the reference's
    // decode-as-prefill (reference_forward per position).  Gate: the last
    // position from IDENTICAL history -- the store mirrors the device's K/V
    // rows, its cache is rewound one position and reference_forward redoes
    // the last token -- within 1e-4 (5e-4 if that step's K/V rows flipped a
    // bf16 rounding), as the single-step cases above; and the same greedy
    // token as the reference's own whole-prompt run.  The whole-prompt drift
    // (bf16 K/V flips compound over positions, for the kernel's own
    // decode-as-prefill just the same) is printed for context.
    {
        const int64_t n = 24;
        std::mt19937 gen(5);
        std::vector<std::vector<int64_t>> prompt(n);
        for (auto& row : prompt) row = {static_cast<int64_t>(gen() % m.vocab_size)};
        TensorStore ref = init_weights(m, 42, n + 4);
        std::vector<std::vector<double>> want;
        for (int64_t t = 0; t < n; ++t) want = reference_forward(ref, prompt[t], t);
        auto rel = [](const std::vector<float>& got, const std::vector<double>& w) {
            double scale = 0, e = 0;
            for (double x : w) scale = std::max(scale, std::abs(x));
            for (size_t i = 0; i < got.size(); ++i) e = std::max(e, std::abs(got[i] - w[i]) / scale);
            return e;
        };
        auto amax = [](const auto& v) { return std::max_element(v.begin(), v.end()) - v.begin(); };
        TensorStore st = init_weights(m, 42, n + 4);
        b200::Decoder dec(st, n + 4);
        auto got = dec.prefill(st, prompt, 0);
        const bool len_ok = st.kv.length(0) == n;
        // same history: rewind the mirrored store one position, redo the last token
        std::vector<float> kd(m.d_head), vd(m.d_head);
        int flips = 0;
        for (int64_t l = 0; l < m.layers; ++l) st.kv.set_length(l, n - 1);
        std::vector<std::vector<float>> dev_k, dev_v;  // the device's rows at n - 1
        for (int64_t l = 0; l < m.layers; ++l)
            for (int64_t h = 0; h < m.n_kv_heads; ++h) {
                dev_k.emplace_back(st.kv.k_at(0, l, h, n - 1), st.kv.k_at(0, l, h, n - 1) + m.d_head);
                dev_v.emplace_back(st.kv.v_at(0, l, h, n - 1), st.kv.v_at(0, l, h, n - 1) + m.d_head);
            }
        auto same = reference_forward(st, prompt[n - 1], n - 1);
        for (int64_t l = 0, i = 0; l < m.layers; ++l)
            for (int64_t h = 0; h < m.n_kv_heads; ++h, ++i)
                for (int64_t d = 0; d < m.d_head; ++d) {
                    flips += st.kv.k_at(0, l, h, n - 1)[d] != dev_k[i][d];
                    flips += st.kv.v_at(0, l, h, n - 1)[d] != dev_v[i][d];
                }
        const double e_same = rel(got[0], same[0]), e_drift = rel(got[0], want[0]);
        TensorStore st2 = init_weights(m, 42, n + 4);
        b200::Decoder dec2(st2, n + 4);
        std::vector<std::vector<float>> loop;
        for (int64_t t = 0; t < n; ++t) loop = dec2.forward(st2, prompt[t], t);
        const bool ok = len_ok && (flips == 0 ? e_same < 1e-4 : e_same < 5e-4) && amax(got[0]) == amax(want[0]);
        std::printf("prefill of %lld tokens: same-history rel_err %.3e (last-row flips %d), greedy %lld / %lld; "
                    "whole-prompt drift %.3e (kernel decode-as-prefill %.3e)  %s\n",
                    (long long)n, e_same, flips, (long long)amax(got[0]), (long long)amax(want[0]), e_drift,
                    rel(loop[0], want[0]), ok ? "ok" : "FAIL");
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
