// store_io.cu -- store files, device images and bulk KV export (C-ABI).
//
//   ffb_load_store   reads the reference's weight fixture container "FSTW" v1
//                    (save_store / load_store, tensor_store.hpp:367-482) and
//                    packs every record through ffb_upload_tensor: a store
//                    written by the reference (or its restatement) feeds the
//                    kernel without building a TensorStore in memory.
//   ffb_save_image / ffb_load_image
//                    the packed DEVICE image of a handle (bf16 / chunk-major /
//                    int4 / int8 rows, norms, embedding) as raw bytes plus a
//                    header naming the kernel specialisation and the TP shard
//                    it belongs to: reloading skips the packer (the quant grid
//                    re-derivation, the chunk-major swizzle, TP slicing).
//   ffb_kv_export    every KV row of positions [pos0, pos0 + n) in the
//                    reference layout [B][L][Hkv][n][dh] f32 (KVCache::k_at /
//                    v_at, tensor_store.hpp:109-125) in one gather kernel and
//                    one device-to-host copy.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "model.cuh"

namespace {

// ---------------------------------------------------------------- KV export
__global__ void kv_gather_kernel(const __nv_bfloat16* __restrict__ kc,
                                 const __nv_bfloat16* __restrict__ vc, float* __restrict__ out,
                                 int64_t B, int64_t L, int64_t H, int64_t S, int64_t dh,
                                 int64_t pos0, int64_t n_pos) {
    // out = [2][B][L][H][n_pos][dh]; cache = [L][B][H][S][dh], 16-byte units
    // of each position XOR-swizzled by pos & 7 (runtime.cu: kv_swz)
    const int64_t per = B * L * H * n_pos * dh;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * per;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kv = i / per, j = i % per;
        const int64_t d = j % dh, p = (j / dh) % n_pos, h = (j / (dh * n_pos)) % H,
                      l = (j / (dh * n_pos * H)) % L, b = j / (dh * n_pos * H * L);
        const int64_t pos = pos0 + p;
        const int64_t sd = (((d >> 3) ^ (pos & 7)) << 3) | (d & 7);
        const int64_t src = (((l * B + b) * H + h) * S + pos) * dh + sd;
        out[i] = __bfloat162float((kv ? vc : kc)[src]);
    }
}

// ---------------------------------------------------------------- FSTW reader
struct Reader {
    FILE* f = nullptr;
    std::string path;
    ~Reader() {
        if (f) std::fclose(f);
    }
    bool u64(uint64_t* v) { return std::fread(v, 8, 1, f) == 1; }
    bool str(std::string* s, uint64_t cap) {
        uint64_t n;
        if (!u64(&n) || n > cap) return false;
        s->resize(n);
        return n == 0 || std::fread(&(*s)[0], 1, n, f) == n;
    }
    bool floats(std::vector<float>* v, uint64_t cap) {
        uint64_t n;
        if (!u64(&n) || n > cap) return false;
        v->resize(n);
        return n == 0 || std::fread(v->data(), 4, n, f) == n;
    }
};

std::string trim(const std::string& s) {
    size_t a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    size_t b = s.find_last_not_of(" \t\r\n");
    return s.substr(a, b - a + 1);
}

// [model] section of serialize(RunConfig) (config.hpp:245-329)
ffb_status parse_model(const std::string& text, ffb_model_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->rope_theta = 500000.0;
    c->rmsnorm_eps = 1e-5;
    c->batch = 1;
    c->quant_group = 128;
    bool in_model = false, seen = false;
    size_t p = 0;
    while (p <= text.size()) {
        size_t e = text.find('\n', p);
        if (e == std::string::npos) e = text.size();
        std::string line = text.substr(p, e - p);
        p = e + 1;
        size_t h = line.find('#');
        if (h != std::string::npos) line.resize(h);
        line = trim(line);
        if (line.empty()) continue;
        if (line[0] == '[') {
            in_model = line == "[model]";
            seen |= in_model;
            continue;
        }
        if (!in_model) continue;
        size_t eq = line.find('=');
        if (eq == std::string::npos) return fail(FFB_VALIDATION, "load_store: expected key = value");
        const std::string k = trim(line.substr(0, eq)), v = trim(line.substr(eq + 1));
        if (k == "kind") {
            if (v == "llama_decoder") c->kind = 0;
            else if (v == "stacked_linear") c->kind = 1;
            else return fail(FFB_VALIDATION, "unknown model kind: %s", v.c_str());
        } else if (k == "layers") c->layers = std::atoll(v.c_str());
        else if (k == "d_model") c->d_model = std::atoll(v.c_str());
        else if (k == "d_inter") c->d_inter = std::atoll(v.c_str());
        else if (k == "d_head") c->d_head = std::atoll(v.c_str());
        else if (k == "n_q_heads") c->n_q_heads = std::atoll(v.c_str());
        else if (k == "n_kv_heads") c->n_kv_heads = std::atoll(v.c_str());
        else if (k == "vocab_size") c->vocab_size = std::atoll(v.c_str());
        else if (k == "rope_theta") c->rope_theta = std::strtod(v.c_str(), nullptr);
        else if (k == "rmsnorm_eps") c->rmsnorm_eps = std::strtod(v.c_str(), nullptr);
        else if (k == "dtype") c->dtype = v == "bf16" ? 0 : 1;
        else if (k == "batch") c->batch = std::atoll(v.c_str());
        else if (k == "quant_bits") c->quant_bits = std::atoi(v.c_str());
        else if (k == "quant_group_size") c->quant_group = std::atoi(v.c_str());
        else if (k == "quant_scheme") continue;
        else return fail(FFB_VALIDATION, "config: unknown [model] field '%s'", k.c_str());
    }
    if (!seen) return fail(FFB_VALIDATION, "config: missing [model] section");
    return FFB_OK;
}

// ---------------------------------------------------------------- device image
constexpr uint64_t kImageMagic = 0x33474d4942464646ull;  // "FFFBIMG3" (quant tensor-core code order v2)

struct ImageHeader {
    uint64_t magic;
    ffb_model_config gcfg;  // whole model
    int32_t tp_rank, tp_size;
    // identity of the kernel specialisation (device row formats)
    int32_t D, DI, DH, NQ, NKV, B, QB, row_bytes, row_bytes_a, tc_d, tc_a, ffn2_rows, kc, kc_layout;
    int32_t n_regions;
    uint64_t quant_inexact_groups;
    uint64_t fp16_inexact;
};

struct Region {
    void* ptr;
    uint64_t bytes;
};

std::vector<Region> regions(const ffb_model* m) {
    const auto& c = m->cfg;
    const uint64_t Lc = std::max<int64_t>(1, c.layers), D = c.d_model;
    const uint64_t RB = m->ops->row_bytes;
    if (c.kind == 1) return {{m->wlin, Lc * D * RB}};
    return {{m->wqkv, Lc * m->qkv_rows() * RB},
            {m->waout, Lc * D * (uint64_t)m->ops->row_bytes_a},
            {m->wffn1, Lc * 2 * c.d_inter * RB},
            {m->wffn2t, Lc * c.d_inter * RB},
            {m->norm_attn, Lc * D * 4},
            {m->norm_ffn, Lc * D * 4},
            {m->final_norm, D * 4},
            {m->embedding, (uint64_t)m->gcfg.vocab_size * D * 2},
            {m->lm_head, (uint64_t)c.vocab_size * RB}};
}

ImageHeader make_header(const ffb_model* m) {
    ImageHeader h;
    std::memset(&h, 0, sizeof(h));
    h.magic = kImageMagic;
    h.gcfg = m->gcfg;
    h.gcfg.batch = m->cfg.batch;
    h.tp_rank = m->tp_rank;
    h.tp_size = m->tp_size;
    const KernelOps* o = m->ops;
    h.D = o->D; h.DI = o->DI; h.DH = o->DH; h.NQ = o->NQ; h.NKV = o->NKV; h.B = o->B; h.QB = o->QB;
    h.row_bytes = o->row_bytes; h.row_bytes_a = o->row_bytes_a; h.tc_d = o->tc_d; h.tc_a = o->tc_a;
    h.ffn2_rows = o->ffn2_rows; h.kc = o->kc; h.kc_layout = o->kc_layout;
    h.n_regions = static_cast<int32_t>(regions(m).size());
    h.quant_inexact_groups = m->quant_inexact_groups;
    h.fp16_inexact = m->fp16_inexact;
    return h;
}

// host bounce buffer for chunked copies (pinned: full-speed DMA)
struct Bounce {
    void* p = nullptr;
    size_t n = 0;
    explicit Bounce(size_t bytes) {
        if (cudaMallocHost(&p, bytes) == cudaSuccess) n = bytes;
        else cudaGetLastError();
    }
    ~Bounce() {
        if (p) cudaFreeHost(p);
    }
};

}  // namespace

extern "C" {

ffb_status ffb_kv_export(ffb_model* m, int64_t pos0, int64_t n_pos, float* k_out, float* v_out) {
    if (!m || !k_out || !v_out) return fail(FFB_USAGE, "NULL argument");
    const auto& c = m->cfg;
    if (c.kind != 0) return fail(FFB_VALIDATION, "kv_export: llama_decoder models only");
    if (pos0 < 0 || n_pos < 0 || pos0 + n_pos > m->max_seq)
        return fail(FFB_VALIDATION, "kv_export: positions out of range");
    if (n_pos == 0) return FFB_OK;
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaStreamSynchronize(m->stream));
    const int64_t B = c.batch, L = c.layers, H = c.n_kv_heads, dh = c.d_head;
    const int64_t per = B * L * H * n_pos * dh;
    // one gather + one copy when both halves fit the staging buffer, else per
    // (batch row, layer) with position chunks
    if (2 * per <= ffb_model::kStagingElems) {
        kv_gather_kernel<<<592, 256, 0, m->stream>>>(m->kcache, m->vcache, m->staging, B, L, H,
                                                     m->max_seq, dh, pos0, n_pos);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(k_out, m->staging, sizeof(float) * per, cudaMemcpyDeviceToHost,
                                 m->stream));
        CUDA_TRY(cudaMemcpyAsync(v_out, m->staging + per, sizeof(float) * per,
                                 cudaMemcpyDeviceToHost, m->stream));
        CUDA_TRY(cudaStreamSynchronize(m->stream));
        return FFB_OK;
    }
    const int64_t pc = std::max<int64_t>(1, std::min<int64_t>(n_pos, ffb_model::kStagingElems /
                                                                         (2 * H * dh)));
    for (int64_t b = 0; b < B; ++b)
        for (int64_t l = 0; l < L; ++l)
            for (int64_t p0 = 0; p0 < n_pos; p0 += pc) {
                const int64_t np = std::min(pc, n_pos - p0);
                // gather [2][1][1][H][np][dh] of (b, l) through a shifted base
                const __nv_bfloat16* kb = m->kcache + ((l * B + b) * H) * m->max_seq * dh;
                const __nv_bfloat16* vb = m->vcache + ((l * B + b) * H) * m->max_seq * dh;
                kv_gather_kernel<<<592, 256, 0, m->stream>>>(kb, vb, m->staging, 1, 1, H,
                                                             m->max_seq, dh, pos0 + p0, np);
                CUDA_TRY(cudaGetLastError());
                const int64_t half = H * np * dh;
                for (int kv = 0; kv < 2; ++kv) {
                    float* dst = (kv ? v_out : k_out) + ((b * L + l) * H * n_pos + p0) * dh;
                    CUDA_TRY(cudaMemcpy2DAsync(dst, sizeof(float) * n_pos * dh,
                                               m->staging + kv * half, sizeof(float) * np * dh,
                                               sizeof(float) * np * dh, H,
                                               cudaMemcpyDeviceToHost, m->stream));
                }
                CUDA_TRY(cudaStreamSynchronize(m->stream));  // staging reused
            }
    return FFB_OK;
}

ffb_status ffb_load_store(ffb_model* m, const char* path) {
    if (!m || !path) return fail(FFB_USAGE, "NULL argument");
    Reader r;
    r.f = std::fopen(path, "rb");
    if (!r.f) return fail(FFB_USAGE, "load_store: cannot open %s", path);
    uint64_t magic = 0, ver = 0;
    if (!r.u64(&magic) || magic != 0x46535457u) return fail(FFB_USAGE, "load_store: bad magic");
    if (!r.u64(&ver) || ver != 1) return fail(FFB_USAGE, "load_store: bad version");
    std::string text;
    if (!r.str(&text, 1 << 20)) return fail(FFB_USAGE, "load_store: truncated file");
    ffb_model_config fc;
    ffb_status st = parse_model(text, &fc);
    if (st) return st;
    const auto& g = m->gcfg;
    const bool same = fc.kind == g.kind && fc.layers == g.layers && fc.d_model == g.d_model &&
                      (g.kind == 1 || (fc.d_inter == g.d_inter && fc.d_head == g.d_head &&
                                       fc.n_q_heads == g.n_q_heads &&
                                       fc.n_kv_heads == g.n_kv_heads &&
                                       fc.vocab_size == g.vocab_size));
    if (!same)
        return fail(FFB_VALIDATION,
                    "load_store: the file holds a different model shape (layers=%lld d_model=%lld "
                    "d_inter=%lld vocab=%lld)",
                    (long long)fc.layers, (long long)fc.d_model, (long long)fc.d_inter,
                    (long long)fc.vocab_size);
    const uint64_t cap = (uint64_t)1 << 40;
    std::vector<float> buf;
    std::string name;
    auto matrix = [&](const std::string& want) -> ffb_status {
        uint64_t dt, rows, cols;
        if (!r.str(&name, 256) || !r.u64(&dt) || !r.u64(&rows) || !r.u64(&cols) ||
            !r.floats(&buf, cap))
            return fail(FFB_USAGE, "load_store: truncated file (%s)", want.c_str());
        if (name != want)
            return fail(FFB_USAGE, "load_store: record '%s' where '%s' was expected", name.c_str(),
                        want.c_str());
        if (buf.size() != rows * cols)
            return fail(FFB_USAGE, "load_store: record '%s' is not rows x cols", want.c_str());
        return ffb_upload_tensor(m, want.c_str(), buf.data(), static_cast<int64_t>(buf.size()));
    };
    auto vector = [&](const std::string& want) -> ffb_status {
        if (!r.floats(&buf, cap)) return fail(FFB_USAGE, "load_store: truncated file (%s)", want.c_str());
        return ffb_upload_tensor(m, want.c_str(), buf.data(), static_cast<int64_t>(buf.size()));
    };
    uint64_t nl = 0;
    if (!r.u64(&nl) || (int64_t)nl != g.layers)
        return fail(FFB_USAGE, "load_store: layer count does not match the config record");
    for (uint64_t l = 0; l < nl; ++l) {
        const std::string p = (g.kind == 1 ? "linear." : "layer.") + std::to_string(l);
        if (g.kind == 1) {
            if ((st = matrix(p))) return st;
            continue;
        }
        if ((st = matrix(p + ".wqkv")) || (st = matrix(p + ".waout")) ||
            (st = matrix(p + ".wffn1")) || (st = matrix(p + ".wffn2t")) ||
            (st = vector(p + ".norm_attn")) || (st = vector(p + ".norm_ffn")))
            return st;
    }
    if (g.kind == 0 &&
        ((st = vector("final_norm")) || (st = matrix("embedding")) || (st = matrix("lm_head"))))
        return st;
    return FFB_OK;
}

ffb_status ffb_save_image(ffb_model* m, const char* path) {
    if (!m || !path) return fail(FFB_USAGE, "NULL argument");
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaDeviceSynchronize());
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(FFB_USAGE, "save_image: cannot open %s", path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    const ImageHeader h = make_header(m);
    if (std::fwrite(&h, sizeof(h), 1, f) != 1) return fail(FFB_USAGE, "save_image: write failed");
    Bounce bb(64ull << 20);
    if (!bb.n) return fail(FFB_DEVICE, "save_image: cudaMallocHost failed");
    for (const Region& rg : regions(m)) {
        if (std::fwrite(&rg.bytes, 8, 1, f) != 1) return fail(FFB_USAGE, "save_image: write failed");
        for (uint64_t off = 0; off < rg.bytes; off += bb.n) {
            const size_t n = std::min<uint64_t>(bb.n, rg.bytes - off);
            CUDA_TRY(cudaMemcpy(bb.p, static_cast<const uint8_t*>(rg.ptr) + off, n,
                                cudaMemcpyDeviceToHost));
            if (std::fwrite(bb.p, 1, n, f) != n) return fail(FFB_USAGE, "save_image: write failed");
        }
    }
    if (std::fclose(guard.release()) != 0) return fail(FFB_USAGE, "save_image: close failed");
    return FFB_OK;
}

ffb_status ffb_load_image(ffb_model* m, const char* path) {
    if (!m || !path) return fail(FFB_USAGE, "NULL argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(FFB_USAGE, "load_image: cannot open %s", path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    ImageHeader h;
    if (std::fread(&h, sizeof(h), 1, f) != 1 || h.magic != kImageMagic)
        return fail(FFB_USAGE, "load_image: not a device image");
    ImageHeader want = make_header(m);
    want.quant_inexact_groups = h.quant_inexact_groups;
    want.fp16_inexact = h.fp16_inexact;
    if (std::memcmp(&h, &want, sizeof(h)) != 0)
        return fail(FFB_VALIDATION,
                    "load_image: the image was packed for another model, shard or kernel "
                    "specialisation");
    CUDA_TRY(cudaSetDevice(m->device));
    CUDA_TRY(cudaDeviceSynchronize());
    Bounce bb(64ull << 20);
    if (!bb.n) return fail(FFB_DEVICE, "load_image: cudaMallocHost failed");
    for (const Region& rg : regions(m)) {
        uint64_t bytes = 0;
        if (std::fread(&bytes, 8, 1, f) != 1 || bytes != rg.bytes)
            return fail(FFB_USAGE, "load_image: truncated or mismatched region");
        for (uint64_t off = 0; off < rg.bytes; off += bb.n) {
            const size_t n = std::min<uint64_t>(bb.n, rg.bytes - off);
            if (std::fread(bb.p, 1, n, f) != n) return fail(FFB_USAGE, "load_image: truncated file");
            CUDA_TRY(cudaMemcpy(static_cast<uint8_t*>(rg.ptr) + off, bb.p, n,
                                cudaMemcpyHostToDevice));
        }
    }
    m->quant_inexact_groups = h.quant_inexact_groups;
    m->fp16_inexact = h.fp16_inexact;
    return FFB_OK;
}

}  // extern "C"
