// fusesim_bridge.hpp -- the reference-side binding a fusesim maintainer adds.
//
// Header-only C++ over the C-ABI (include/flashformer_b200.h).  It keeps the
// reference's own types and contracts (/root/reference/proj/include/fusesim):
//
//   fusesim::reference_forward(store, tokens, pos)      reference.hpp:37-139
//   fusesim::execute_program(progs, plan, store, ...)   interpreter.hpp:502-506
//      -> fusesim::b200::Decoder::forward(store, tokens, pos)
//
// Same argument meaning (one token per batch row, pos == cache length), same
// side effect (one K/V position appended per layer -- on the device AND in
// store.kv, so the TensorStore stays usable by the CPU paths), same errors
// (fusesim::ValidationError for bad tokens / positions / capacity).  Device
// failures raise fusesim::b200::DeviceError.
//
// Include order: the maintainer's fusesim headers first, e.g.
//   #include "fusesim/tensor_store.hpp"
//   #include "ffb200/fusesim_bridge.hpp"
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../flashformer_b200.h"

namespace fusesim {
namespace b200 {

struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(ffb_status s) {
    switch (s) {
        case FFB_OK: return;
        case FFB_VALIDATION: throw ValidationError(ffb_last_error());
        case FFB_USAGE: throw ParseError(ffb_last_error());
        default: throw DeviceError(ffb_last_error());
    }
}

inline ffb_model_config to_c(const ModelConfig& m) {
    ffb_model_config c{};
    c.layers = m.layers;
    c.d_model = m.d_model;
    c.d_inter = m.d_inter;
    c.d_head = m.d_head;
    c.n_q_heads = m.n_q_heads;
    c.n_kv_heads = m.n_kv_heads;
    c.vocab_size = m.vocab_size;
    c.rope_theta = m.rope_theta;
    c.rmsnorm_eps = m.rmsnorm_eps;
    c.dtype = m.dtype == DType::BF16 ? 0 : 1;
    c.quant_bits = m.quant ? m.quant->bits : 0;
    c.quant_group = m.quant ? m.quant->group_size : 0;
    c.batch = m.batch;
    c.kind = m.kind == ModelKind::StackedLinear ? 1 : 0;
    return c;
}

inline ffb_mode to_c(RunMode r) {
    switch (r) {
        case RunMode::Baseline: return FFB_MODE_BASELINE;
        case RunMode::Fused: return FFB_MODE_FUSED;
        default: return FFB_MODE_FUSED_OVERLAP;
    }
}

// A TensorStore's weights and KV cache resident on one B200, plus the decode
// kernel specialised for its ModelConfig.
class Decoder {
public:
    Decoder(const TensorStore& st, int64_t max_seq_len, RunMode mode = RunMode::FusedOverlap,
            int device = 0)
        : model_(st.model) {
        const ffb_model_config c = to_c(st.model);
        check(ffb_create(&c, max_seq_len, device, 0, 1, &h_));
        try {
            upload(st);
            check(ffb_set_mode(h_, to_c(mode)));
        } catch (...) {
            ffb_destroy(h_);
            throw;
        }
    }
    ~Decoder() { ffb_destroy(h_); }
    Decoder(const Decoder&) = delete;
    Decoder& operator=(const Decoder&) = delete;

    // Weights (tensor_store.hpp:344-363 names) and the cached positions.
    void upload(const TensorStore& st) {
        auto put = [&](const std::string& name, const std::vector<float>& v) {
            check(ffb_upload_tensor(h_, name.c_str(), v.data(), static_cast<int64_t>(v.size())));
        };
        for (int64_t l = 0; l < model_.layers; ++l) {
            const std::string p = "layer." + std::to_string(l) + ".";
            const LayerWeights& lw = st.layers[l];
            put(p + "wqkv", lw.wqkv.values);
            put(p + "waout", lw.waout.values);
            put(p + "wffn1", lw.wffn1.values);
            put(p + "wffn2t", lw.wffn2t.values);
            put(p + "norm_attn", lw.norm_attn);
            put(p + "norm_ffn", lw.norm_ffn);
        }
        put("final_norm", st.final_norm);
        put("embedding", st.embedding.values);
        put("lm_head", st.lm_head.values);
        // KVCache keeps one contiguous [B][L][Hkv][S][dh] block per K / V
        // (tensor_store.hpp:139-148): one bulk import of the longest prefix
        int64_t n = 0;
        for (int64_t l = 0; l < model_.layers; ++l) n = std::max(n, st.kv.length(l));
        if (model_.layers > 0)
            check(ffb_kv_import(h_, st.kv.k_at(0, 0, 0, 0), st.kv.v_at(0, 0, 0, 0),
                                st.kv.max_seq_len(), n));
        for (int64_t l = 0; l < model_.layers; ++l) check(ffb_kv_set_length(h_, l, st.kv.length(l)));
    }

    // reference_forward contract: logits[batch][vocab]; store.kv gains the
    // same appended position (read back from the device cache).
    std::vector<std::vector<float>> forward(TensorStore& st, const std::vector<int64_t>& tokens,
                                            int64_t pos) {
        if (static_cast<int64_t>(tokens.size()) != model_.batch)
            throw ValidationError("reference_forward: one token per batch row required");
        std::vector<float> flat(static_cast<size_t>(model_.batch * model_.vocab_size));
        check(ffb_decode_step(h_, tokens.data(), pos, flat.data(), nullptr, nullptr));
        // the appended rows of every (batch row, layer, kv head): one bulk
        // export [B][L][Hkv][1][dh], then KVCache::append_token per layer
        const int64_t dh = model_.d_head, nkv = model_.n_kv_heads, L = model_.layers;
        std::vector<float> ka(static_cast<size_t>(model_.batch * L * nkv * dh)), va(ka.size());
        check(ffb_kv_export(h_, pos, 1, ka.data(), va.data()));
        for (int64_t l = 0; l < L; ++l) {
            std::vector<std::vector<float>> k(model_.batch), v(model_.batch);
            for (int64_t b = 0; b < model_.batch; ++b) {
                const size_t o = static_cast<size_t>((b * L + l) * nkv * dh);
                k[b].assign(ka.begin() + o, ka.begin() + o + nkv * dh);
                v[b].assign(va.begin() + o, va.begin() + o + nkv * dh);
            }
            if (st.kv.length(l) == pos) st.kv.append_token(l, k, v);
        }
        std::vector<std::vector<float>> out(model_.batch);
        for (int64_t b = 0; b < model_.batch; ++b)
            out[b].assign(flat.begin() + b * model_.vocab_size,
                          flat.begin() + (b + 1) * model_.vocab_size);
        return out;
    }

    // Prompt ingestion (ffb_prefill): prompt[t][b] at positions pos0 + t,
    // the replacement of the decode-as-prefill loop (reference_forward per
    // position, reference.hpp:60-61).  Returns the last position's logits;
    // store.kv gains every appended position (one bulk export).
    std::vector<std::vector<float>> prefill(TensorStore& st, const std::vector<std::vector<int64_t>>& prompt,
                                            int64_t pos0) {
        const int64_t n = static_cast<int64_t>(prompt.size()), B = model_.batch;
        std::vector<int64_t> flat_tok;
        for (const auto& row : prompt) {
            if (static_cast<int64_t>(row.size()) != B)
                throw ValidationError("prefill: one token per batch row required");
            flat_tok.insert(flat_tok.end(), row.begin(), row.end());
        }
        std::vector<float> flat(static_cast<size_t>(B * model_.vocab_size));
        check(ffb_prefill(h_, flat_tok.data(), n, pos0, flat.data(), nullptr));
        const int64_t dh = model_.d_head, nkv = model_.n_kv_heads, L = model_.layers;
        std::vector<float> ka(static_cast<size_t>(B * L * nkv * n * dh)), va(ka.size());  // [B][L][Hkv][n][dh]
        check(ffb_kv_export(h_, pos0, n, ka.data(), va.data()));
        for (int64_t t = 0; t < n; ++t)
            for (int64_t l = 0; l < L; ++l) {
                if (st.kv.length(l) != pos0 + t) continue;
                std::vector<std::vector<float>> k(B), v(B);
                for (int64_t b = 0; b < B; ++b)
                    for (int64_t h = 0; h < nkv; ++h) {
                        const size_t o = static_cast<size_t>((((b * L + l) * nkv + h) * n + t) * dh);
                        k[b].insert(k[b].end(), ka.begin() + o, ka.begin() + o + dh);
                        v[b].insert(v[b].end(), va.begin() + o, va.begin() + o + dh);
                    }
                st.kv.append_token(l, k, v);
            }
        std::vector<std::vector<float>> out(B);
        for (int64_t b = 0; b < B; ++b)
            out[b].assign(flat.begin() + b * model_.vocab_size, flat.begin() + (b + 1) * model_.vocab_size);
        return out;
    }

    ffb_model* handle() { return h_; }

private:
    ModelConfig model_;
    ffb_model* h_ = nullptr;
};

}  // namespace b200
}  // namespace fusesim
