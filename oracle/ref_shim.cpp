// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile against
// /root/reference/proj/include (the reference sources where they lie; nothing
// is copied) into oracle/_ref/libfusesim_ref.so.  Used to (1) pin the C
// restatement in oracle/fusesim_oracle.c bit-for-bit, (2) generate the golden
// fixtures in tests/golden/, and (3) serve as the timed CPU baseline
// (cpu_baseline.kind = "reference") in bench.py.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "fusesim/interpreter.hpp"
#include "fusesim/presets.hpp"
#include "fusesim/reference.hpp"
#include "fusesim/simulate.hpp"
#include "fusesim/verify.hpp"

using namespace fusesim;

namespace {
thread_local std::string g_err;

struct RefConfig {  // layout-identical to fo_config (oracle/fusesim_oracle.h)
    int64_t layers, d_model, d_inter, d_head, n_q_heads, n_kv_heads, vocab_size;
    double rope_theta, rmsnorm_eps;
    int32_t dtype, quant_bits, quant_group;
    int64_t batch;
};

ModelConfig to_model(const RefConfig* c) {
    ModelConfig m;
    m.kind = ModelKind::LlamaDecoder;
    m.layers = c->layers;
    m.d_model = c->d_model;
    m.d_inter = c->d_inter;
    m.d_head = c->d_head;
    m.n_q_heads = c->n_q_heads;
    m.n_kv_heads = c->n_kv_heads;
    m.vocab_size = c->vocab_size;
    m.rope_theta = c->rope_theta;
    m.rmsnorm_eps = c->rmsnorm_eps;
    m.dtype = c->dtype == 0 ? DType::BF16 : DType::F32;
    if (c->quant_bits) {
        QuantConfig q;
        q.bits = c->quant_bits;
        q.group_size = c->quant_group;
        m.quant = q;
    }
    m.batch = c->batch;
    return m;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 2;
    } catch (const VerifyError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_init_weights(const RefConfig* c, uint64_t seed, int64_t max_seq_len) {
    TensorStore* st = nullptr;
    int rc = guarded([&] { st = new TensorStore(init_weights(to_model(c), seed, max_seq_len)); });
    return rc == 0 ? st : nullptr;
}

// Store with correct shapes but cheap deterministic values (no <random>
// normal draws): for timing reference_forward where values do not matter.
void* ref_init_fast(const RefConfig* c, int64_t max_seq_len) {
    TensorStore* st = nullptr;
    int rc = guarded([&] {
        ModelConfig m = to_model(c);
        m.validate();
        auto* s = new TensorStore();
        s->model = m;
        s->residual.assign(m.batch, std::vector<float>(m.d_model, 0.0f));
        uint64_t state = 0x9e3779b97f4a7c15ull;
        auto fill = [&](Matrix& mx, MatrixKind kind, int32_t layer) {
            MatrixMeta meta = weight_meta(m, kind, layer);
            mx.rows = meta.rows;
            mx.cols = meta.cols;
            mx.dtype = meta.dtype;
            mx.quantized = meta.quantized;
            mx.quant_group = meta.quant_group;
            mx.values.resize(static_cast<size_t>(mx.rows) * mx.cols);
            for (auto& v : mx.values) {
                state = state * 6364136223846793005ull + 1442695040888963407ull;
                v = bf16_round(static_cast<float>(static_cast<int32_t>(state >> 40) - (1 << 23)) *
                               (1.0f / (1 << 23)) * 0.02f);
            }
        };
        s->layers.resize(m.layers);
        for (int32_t l = 0; l < m.layers; ++l) {
            auto& lw = s->layers[l];
            fill(lw.wqkv, MatrixKind::Wqkv, l);
            fill(lw.waout, MatrixKind::Waout, l);
            fill(lw.wffn1, MatrixKind::Wffn1, l);
            fill(lw.wffn2t, MatrixKind::Wffn2, l);
            lw.norm_attn.assign(m.d_model, 1.0f);
            lw.norm_ffn.assign(m.d_model, 1.0f);
        }
        s->final_norm.assign(m.d_model, 1.0f);
        fill(s->lm_head, MatrixKind::LmHead, -1);
        s->embedding = s->lm_head;
        s->kv = KVCache(m, max_seq_len);
        st = s;
    });
    return rc == 0 ? st : nullptr;
}

void ref_free(void* h) { delete static_cast<TensorStore*>(h); }

// name: "layer.<l>.wqkv|waout|wffn1|wffn2t|norm_attn|norm_ffn", "final_norm",
// "embedding", "lm_head".  Copies f32 values; returns the element count.
int64_t ref_get_tensor(void* h, const char* name, float* out) {
    auto* st = static_cast<TensorStore*>(h);
    std::string n(name);
    const std::vector<float>* v = nullptr;
    if (n.rfind("linear.", 0) == 0) v = &st->linear_layers.at(std::stoi(n.substr(7))).values;
    else if (n == "final_norm") v = &st->final_norm;
    else if (n == "embedding") v = &st->embedding.values;
    else if (n == "lm_head") v = &st->lm_head.values;
    else if (n.rfind("layer.", 0) == 0) {
        size_t dot = n.find('.', 6);
        int l = std::stoi(n.substr(6, dot - 6));
        std::string t = n.substr(dot + 1);
        auto& lw = st->layers.at(l);
        if (t == "wqkv") v = &lw.wqkv.values;
        else if (t == "waout") v = &lw.waout.values;
        else if (t == "wffn1") v = &lw.wffn1.values;
        else if (t == "wffn2t") v = &lw.wffn2t.values;
        else if (t == "norm_attn") v = &lw.norm_attn;
        else if (t == "norm_ffn") v = &lw.norm_ffn;
    }
    if (!v) return -1;
    if (out) std::memcpy(out, v->data(), v->size() * sizeof(float));
    return static_cast<int64_t>(v->size());
}

// tests/test_interpreter.cpp:16-30, verbatim semantics.
void ref_synthetic_prefill(void* h, int64_t prefill, uint64_t seed) {
    auto* st = static_cast<TensorStore*>(h);
    const ModelConfig& m = st->model;
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> dist(0.0f, 0.3f);
    std::vector<float> k(m.d_head), v(m.d_head);
    for (int64_t b = 0; b < m.batch; ++b)
        for (int64_t l = 0; l < m.layers; ++l)
            for (int64_t hh = 0; hh < m.n_kv_heads; ++hh)
                for (int64_t p = 0; p < prefill; ++p) {
                    for (auto& x : k) x = dist(rng);
                    for (auto& x : v) x = dist(rng);
                    st->kv.set_position(b, l, hh, p, k.data(), v.data());
                }
    for (int64_t l = 0; l < m.layers; ++l) st->kv.set_length(l, prefill);
}

void ref_kv_set_length(void* h, int64_t layer, int64_t n) {
    static_cast<TensorStore*>(h)->kv.set_length(layer, n);
}

int64_t ref_kv_length(void* h, int64_t layer) {
    return static_cast<TensorStore*>(h)->kv.length(layer);
}

void ref_kv_get(void* h, int64_t b, int64_t l, int64_t head, int64_t pos, float* k, float* v) {
    auto* st = static_cast<TensorStore*>(h);
    int64_t dh = st->model.d_head;
    std::memcpy(k, st->kv.k_at(b, l, head, pos), dh * sizeof(float));
    std::memcpy(v, st->kv.v_at(b, l, head, pos), dh * sizeof(float));
}

void ref_kv_set(void* h, int64_t b, int64_t l, int64_t head, int64_t pos, const float* k,
                const float* v) {
    static_cast<TensorStore*>(h)->kv.set_position(b, l, head, pos, k, v);
}

// reference_forward (reference.hpp:37-139); logits: batch x vocab doubles.
int ref_forward(void* h, const int64_t* tokens, int64_t pos, double* logits) {
    auto* st = static_cast<TensorStore*>(h);
    return guarded([&] {
        std::vector<int64_t> tok(tokens, tokens + st->model.batch);
        auto out = reference_forward(*st, tok, pos);
        for (size_t b = 0; b < out.size(); ++b)
            std::memcpy(logits + b * st->model.vocab_size, out[b].data(),
                        out[b].size() * sizeof(double));
    });
}

// execute_program (interpreter.hpp:502-506) with a plan for `num_sms` blocks.
// mode: 0 baseline, 1 fused, 2 fused_overlap.  logits: batch x vocab floats.
int ref_execute(void* h, const int64_t* tokens, int64_t pos, int mode, uint64_t stage_size,
                int64_t num_sms, float* logits) {
    auto* st = static_cast<TensorStore*>(h);
    return guarded([&] {
        HardwareConfig hw = hardware_preset("h100_sxm");
        hw.num_sms = num_sms;
        PipelineConfig pipe;
        pipe.stage_size = stage_size;
        WorkloadPlan plan = build_plan(st->model, hw, pipe, pos);
        auto programs = emit_programs(plan, static_cast<RunMode>(mode));
        auto diags = verify_programs(programs);
        if (!diags.empty()) throw VerifyError("verify_programs reported diagnostics");
        std::vector<int64_t> tok(tokens, tokens + st->model.batch);
        auto res = execute_program(programs, plan, *st, tok, pos);
        for (size_t b = 0; b < res.logits.size(); ++b)
            std::memcpy(logits + b * st->model.vocab_size, res.logits[b].data(),
                        res.logits[b].size() * sizeof(float));
    });
}

// StoreLayout byte accounting (tensor_store.hpp:170-192).
uint64_t ref_streamed_weight_bytes(const RefConfig* c) {
    return store_layout(to_model(c)).streamed_weight_bytes();
}
uint64_t ref_total_weight_bytes(const RefConfig* c) {
    return store_layout(to_model(c)).total_weight_bytes();
}

// Timed dense-oracle step for bench.py's CPU baseline: runs reference_forward
// at a fixed context (the cache length is reset after every step so the
// bytes per step stay exact).  Returns seconds per step (median of `steps`).
double ref_time_forward(void* h, const int64_t* tokens, int64_t pos, int steps) {
    auto* st = static_cast<TensorStore*>(h);
    std::vector<int64_t> tok(tokens, tokens + st->model.batch);
    std::vector<double> ts;
    for (int i = 0; i < steps; ++i) {
        for (int64_t l = 0; l < st->model.layers; ++l) st->kv.set_length(l, pos);
        auto t0 = std::chrono::steady_clock::now();
        auto out = reference_forward(*st, tok, pos);
        auto t1 = std::chrono::steady_clock::now();
        ts.push_back(std::chrono::duration<double>(t1 - t0).count());
        (void)out;
    }
    std::sort(ts.begin(), ts.end());
    return ts.empty() ? 0.0 : ts[ts.size() / 2];
}

// Stacked-linear kind (presets.hpp:48-55, reference.hpp:141-152).
void* ref_linear_init(int64_t layers, int64_t d_model, int64_t batch, uint64_t seed) {
    TensorStore* st = nullptr;
    int rc = guarded([&] {
        ModelConfig m;
        m.kind = ModelKind::StackedLinear;
        m.layers = layers;
        m.d_model = d_model;
        m.batch = batch;
        st = new TensorStore(init_weights(m, seed, 1));
    });
    return rc == 0 ? st : nullptr;
}

int ref_linear_forward(void* h, const float* x0, double* out) {
    auto* st = static_cast<TensorStore*>(h);
    return guarded([&] {
        const ModelConfig& m = st->model;
        for (int64_t b = 0; b < m.batch; ++b)
            std::memcpy(st->residual[b].data(), x0 + b * m.d_model, sizeof(float) * m.d_model);
        auto y = reference_linear_forward(*st);
        for (int64_t b = 0; b < m.batch; ++b)
            std::memcpy(out + b * m.d_model, y[b].data(), sizeof(double) * m.d_model);
    });
}

// fusesim::save_store / load_store (tensor_store.hpp:410-482), unchanged.
int ref_save_store(void* h, const char* path) {
    return guarded([&] { save_store(*static_cast<TensorStore*>(h), path); });
}

void* ref_load_store(const char* path, int64_t max_seq_len) {
    TensorStore* st = nullptr;
    int rc = guarded([&] { st = new TensorStore(load_store(path, max_seq_len)); });
    return rc == 0 ? st : nullptr;
}

// The reference's event-driven simulator (simulate.hpp:423, cost model
// cost_model.hpp:29-57) on the reference's own static schedule
// (partition.hpp:266 build_plan, emit.hpp:313 emit_programs) for a
// hardware / pipeline description -- the cost-model side of SURVEY.md
// §8(f) row 3.  hw: {num_sms, shared_mem_per_sm, peak_bandwidth,
// kernel_launch_overhead, barrier_latency, compute_throughput_per_sm};
// eff: {weight_matvec, kv_attention, glu, load_issue_cost} (< 0: default).
// Writes the total latency (s) and bytes moved, and "name=seconds;..." of the
// per-sublayer latencies into `subs`.
int ref_simulate(const RefConfig* c, const double* hw, const double* eff, int64_t stage_size,
                 int64_t depth, int64_t warps, int64_t seq_len, int32_t mode, int64_t attn_group,
                 double* total, double* bytes, char* subs, int64_t subs_len) {
    return guarded([&] {
        ModelConfig m = to_model(c);
        HardwareConfig h;
        h.num_sms = static_cast<int64_t>(hw[0]);
        h.shared_mem_per_sm = static_cast<uint64_t>(hw[1]);
        h.peak_bandwidth = hw[2];
        h.kernel_launch_overhead = hw[3];
        h.barrier_latency = hw[4];
        h.compute_throughput_per_sm = hw[5];
        PipelineConfig pc;
        pc.stage_size = static_cast<uint64_t>(stage_size);
        pc.depth = depth;
        pc.consumer_warps = warps;
        WorkloadPlan plan = build_plan(m, h, pc, seq_len, attn_group);
        CostModel cm = CostModel::from_hardware(h);
        if (eff[0] > 0) cm.eff_weight_matvec = eff[0];
        if (eff[1] > 0) cm.eff_kv_attention = eff[1];
        if (eff[2] > 0) cm.eff_glu = eff[2];
        if (eff[3] >= 0) cm.load_issue_cost = eff[3];
        const RunMode rm = mode == 0 ? RunMode::Baseline : mode == 1 ? RunMode::Fused
                                                                     : RunMode::FusedOverlap;
        SimResult r = simulate(emit_programs(plan, rm), cm);
        *total = r.total_latency;
        *bytes = static_cast<double>(r.bytes_moved);
        std::string out;
        for (const auto& [name, t] : r.sublayer_latency) out += name + "=" + std::to_string(t) + ";";
        std::snprintf(subs, static_cast<size_t>(subs_len), "%s", out.c_str());
    });
}

}  // extern "C"
