"""CPU checker for the decode path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2505_22758_b200``) never does.

Two backends, same ctypes surface:
  * ``liboracle.so``  -- plain-C restatement (oracle/fusesim_oracle.c) of the
    reference's weight generation and dense f64 decode step.
  * ``_ref/libfusesim_ref.so`` -- the reference headers
    (/root/reference/proj/include/fusesim) compiled unchanged, used to pin the
    restatement and to generate tests/golden/.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfusesim_ref.so")


class FoConfig(C.Structure):
    _fields_ = [
        ("layers", C.c_int64), ("d_model", C.c_int64), ("d_inter", C.c_int64),
        ("d_head", C.c_int64), ("n_q_heads", C.c_int64), ("n_kv_heads", C.c_int64),
        ("vocab_size", C.c_int64), ("rope_theta", C.c_double), ("rmsnorm_eps", C.c_double),
        ("dtype", C.c_int32), ("quant_bits", C.c_int32), ("quant_group", C.c_int32),
        ("batch", C.c_int64),
    ]


class FoLayer(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_float)) for n in
                ("wqkv", "waout", "wffn1", "wffn2t", "norm_attn", "norm_ffn")]


class FoStore(C.Structure):
    _fields_ = [
        ("cfg", FoConfig), ("max_seq_len", C.c_int64), ("layers", C.POINTER(FoLayer)),
        ("final_norm", C.POINTER(C.c_float)), ("embedding", C.POINTER(C.c_float)),
        ("lm_head", C.POINTER(C.c_float)), ("k", C.POINTER(C.c_float)),
        ("v", C.POINTER(C.c_float)), ("kv_len", C.POINTER(C.c_int64)),
    ]


@dataclass(frozen=True)
class ModelCfg:
    """Mirror of fusesim::ModelConfig (config.hpp:45-86), decoder kind."""
    layers: int
    d_model: int
    d_inter: int
    d_head: int
    n_q_heads: int
    n_kv_heads: int
    vocab_size: int
    rope_theta: float = 500000.0
    rmsnorm_eps: float = 1e-5
    dtype: int = 0          # 0 bf16, 1 f32
    quant_bits: int = 0     # 0 none, 4 reference int4, 8 int8 extension
    quant_group: int = 128
    batch: int = 1

    def c(self) -> FoConfig:
        return FoConfig(self.layers, self.d_model, self.d_inter, self.d_head, self.n_q_heads,
                        self.n_kv_heads, self.vocab_size, self.rope_theta, self.rmsnorm_eps,
                        self.dtype, self.quant_bits, self.quant_group, self.batch)

    def replace(self, **kw) -> "ModelCfg":
        d = dict(self.__dict__)
        d.update(kw)
        return ModelCfg(**d)

    @property
    def qkv_rows(self) -> int:
        return self.n_q_heads * self.d_head + 2 * self.n_kv_heads * self.d_head


def _p(a, ct=C.c_float):
    return a.ctypes.data_as(C.POINTER(ct))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle not built: {ORACLE_SO} (run make -C oracle)")
        L = C.CDLL(ORACLE_SO)
        L.fo_last_error.restype = C.c_char_p
        L.fo_init_weights.restype = C.POINTER(FoStore)
        L.fo_init_weights.argtypes = [C.POINTER(FoConfig), C.c_uint64, C.c_int64, C.c_int]
        L.fo_free.argtypes = [C.POINTER(FoStore)]
        L.fo_synthetic_prefill.argtypes = [C.POINTER(FoStore), C.c_int64, C.c_uint64]
        L.fo_reference_forward.argtypes = [C.POINTER(FoStore), C.POINTER(C.c_int64), C.c_int64,
                                           C.POINTER(C.c_double)]
        L.fo_reference_forward_ex.argtypes = [C.POINTER(FoStore), C.POINTER(C.c_int64), C.c_int64,
                                              C.POINTER(C.c_double), C.POINTER(C.c_float),
                                              C.POINTER(C.c_float)]
        L.fo_kv_set_length.argtypes = [C.POINTER(FoStore), C.c_int64, C.c_int64]
        L.fo_kv_length.argtypes = [C.POINTER(FoStore), C.c_int64]
        L.fo_kv_length.restype = C.c_int64
        L.fo_bf16_round.argtypes = [C.c_float]
        L.fo_bf16_round.restype = C.c_float
        L.fo_mt64_next.restype = C.c_uint64
        L.fo_mt32_next.restype = C.c_uint32
        L.fo_fnv1a.restype = C.c_uint64
        L.fo_fnv1a.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.fo_streamed_weight_bytes.restype = C.c_uint64
        L.fo_streamed_weight_bytes.argtypes = [C.POINTER(FoConfig)]
        L.fo_total_weight_bytes.restype = C.c_uint64
        L.fo_total_weight_bytes.argtypes = [C.POINTER(FoConfig)]
        L.fo_quantize_group.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int32,
                                        C.POINTER(C.c_uint8), C.POINTER(C.c_float),
                                        C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.fo_dequantize_code.argtypes = [C.c_uint8, C.c_float, C.c_float]
        L.fo_dequantize_code.restype = C.c_float
        L.fo_quantize_value.argtypes = [C.c_float, C.c_float, C.c_float, C.c_int32]
        L.fo_quantize_value.restype = C.c_uint8
        L.fo_rmsnorm_f64.argtypes = [C.POINTER(C.c_double)] * 2 + [C.c_int64, C.c_double,
                                                                   C.POINTER(C.c_double)]
        L.fo_rope_f64.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_double]
        L.fo_silu.argtypes = [C.c_double]
        L.fo_silu.restype = C.c_double
        L.fo_argmax_f64.argtypes = [C.POINTER(C.c_double), C.c_int64]
        L.fo_argmax_f64.restype = C.c_int64
        L.fo_attn_partial_update.argtypes = [C.POINTER(C.c_double)] * 3 + [
            C.c_int64] + [C.POINTER(C.c_double)] * 3 + [C.c_int64, C.c_double]
        L.fo_attn_reduce.argtypes = [C.POINTER(C.c_double)] * 3 + [C.c_int64, C.c_int64,
                                                                   C.POINTER(C.c_double)]
        L.fo_normal_f64.argtypes = [C.c_uint64, C.c_double, C.c_double, C.POINTER(C.c_double),
                                    C.c_int64]
        L.fo_save_store.argtypes = [C.POINTER(FoStore), C.c_char_p]
        L.fo_store_set_batch.argtypes = [C.POINTER(FoStore), C.c_int64, C.c_int64]
        L.fo_load_store.restype = C.POINTER(FoStore)
        L.fo_load_store.argtypes = [C.c_char_p, C.c_int64]
        L.fo_serialize_config.restype = C.c_int64
        L.fo_serialize_config.argtypes = [C.POINTER(FoConfig), C.c_char_p, C.c_int64]
        _lib = L
    return _lib


class OracleStore:
    """A seeded fusesim TensorStore restated in C (tensor_store.hpp:304-366)."""

    def __init__(self, cfg: ModelCfg, seed: int, max_seq_len: int, nthreads: int | None = None):
        L = lib()
        self.cfg = cfg
        self._c = cfg.c()
        n = nthreads or min(32, os.cpu_count() or 1)
        self._s = L.fo_init_weights(C.byref(self._c), seed, max_seq_len, n)
        if not self._s:
            raise ValueError(L.fo_last_error().decode())
        self.max_seq_len = max_seq_len

    @classmethod
    def load(cls, path: str, max_seq_len: int) -> "OracleStore":
        """load_store (tensor_store.hpp:446-482): an FSTW v1 file -> store."""
        L = lib()
        s = L.fo_load_store(os.fsencode(path), max_seq_len)
        if not s:
            raise ValueError(L.fo_last_error().decode())
        self = cls.__new__(cls)
        self._s = s
        c = s.contents.cfg
        self.cfg = ModelCfg(c.layers, c.d_model, c.d_inter, c.d_head, c.n_q_heads, c.n_kv_heads,
                            c.vocab_size, c.rope_theta, c.rmsnorm_eps, c.dtype, c.quant_bits,
                            c.quant_group, c.batch)
        self._c = self.cfg.c()
        self.max_seq_len = max_seq_len
        return self

    def set_batch(self, batch: int, max_seq_len: int | None = None):
        """Keep the weights, start an empty KV cache for `batch` rows."""
        n = max_seq_len or self.max_seq_len
        if lib().fo_store_set_batch(self._s, batch, n) != 0:
            raise ValueError(lib().fo_last_error().decode())
        self.cfg = self.cfg.replace(batch=batch)
        self._c = self.cfg.c()
        self.max_seq_len = n

    def save(self, path: str):
        """save_store (tensor_store.hpp:410-444), FSTW v1."""
        if lib().fo_save_store(self._s, os.fsencode(path)) != 0:
            raise ValueError(lib().fo_last_error().decode())

    def close(self):
        if getattr(self, "_s", None):
            lib().fo_free(self._s)
            self._s = None

    def __del__(self):
        self.close()

    # -- views (no copies) over the C arrays --
    def _view(self, ptr, shape):
        return np.ctypeslib.as_array(ptr, shape=shape)

    def layer(self, l: int) -> dict:
        c = self.cfg
        L = self._s.contents.layers[l]
        d = c.d_model
        return {
            "wqkv": self._view(L.wqkv, (c.qkv_rows, d)),
            "waout": self._view(L.waout, (d, d)),
            "wffn1": self._view(L.wffn1, (2 * c.d_inter, d)),
            "wffn2t": self._view(L.wffn2t, (c.d_inter, d)),
            "norm_attn": self._view(L.norm_attn, (d,)),
            "norm_ffn": self._view(L.norm_ffn, (d,)),
        }

    @property
    def embedding(self):
        return self._view(self._s.contents.embedding, (self.cfg.vocab_size, self.cfg.d_model))

    @property
    def lm_head(self):
        return self._view(self._s.contents.lm_head, (self.cfg.vocab_size, self.cfg.d_model))

    @property
    def final_norm(self):
        return self._view(self._s.contents.final_norm, (self.cfg.d_model,))

    def kv(self):
        """(K, V) views shaped [B][L][Hkv][S][dh] (tensor_store.hpp:139-148)."""
        c = self.cfg
        shp = (c.batch, c.layers, c.n_kv_heads, self.max_seq_len, c.d_head)
        return self._view(self._s.contents.k, shp), self._view(self._s.contents.v, shp)

    def tensor(self, name: str):
        if name == "embedding":
            return self.embedding
        if name == "lm_head":
            return self.lm_head
        if name == "final_norm":
            return self.final_norm
        _, l, t = name.split(".")
        return self.layer(int(l))[t]

    def synthetic_prefill(self, prefill: int, seed: int):
        lib().fo_synthetic_prefill(self._s, prefill, seed)

    def set_length(self, layer: int, n: int):
        lib().fo_kv_set_length(self._s, layer, n)

    def length(self, layer: int) -> int:
        return lib().fo_kv_length(self._s, layer)

    def forward(self, tokens, pos: int, k_app=None, v_app=None) -> np.ndarray:
        """reference_forward restated; returns float64 logits [B][V].
        k_app/v_app ([B][L][Hkv][dh]): optional externally rounded K/V rows to
        append at `pos` (see fo_reference_forward_ex)."""
        c = self.cfg
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
        out = np.zeros((c.batch, c.vocab_size), dtype=np.float64)
        if k_app is not None:
            ka = np.ascontiguousarray(k_app, dtype=np.float32)
            va = np.ascontiguousarray(v_app, dtype=np.float32)
            rc = lib().fo_reference_forward_ex(self._s, _p(tok, C.c_int64), pos,
                                               _p(out, C.c_double), _p(ka), _p(va))
        else:
            rc = lib().fo_reference_forward(self._s, _p(tok, C.c_int64), pos,
                                            _p(out, C.c_double))
        if rc != 0:
            raise ValueError(lib().fo_last_error().decode())
        return out


# ---------------------------------------------------------------- reference
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference shim not built: {REF_SO}")
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_init_weights.restype = C.c_void_p
        R.ref_init_weights.argtypes = [C.POINTER(FoConfig), C.c_uint64, C.c_int64]
        R.ref_init_fast.restype = C.c_void_p
        R.ref_init_fast.argtypes = [C.POINTER(FoConfig), C.c_int64]
        R.ref_free.argtypes = [C.c_void_p]
        R.ref_get_tensor.restype = C.c_int64
        R.ref_get_tensor.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_float)]
        R.ref_synthetic_prefill.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        R.ref_kv_set_length.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        R.ref_kv_length.argtypes = [C.c_void_p, C.c_int64]
        R.ref_kv_length.restype = C.c_int64
        R.ref_kv_get.argtypes = [C.c_void_p] + [C.c_int64] * 4 + [C.POINTER(C.c_float)] * 2
        R.ref_kv_set.argtypes = [C.c_void_p] + [C.c_int64] * 4 + [C.POINTER(C.c_float)] * 2
        R.ref_forward.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int64,
                                  C.POINTER(C.c_double)]
        R.ref_execute.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int64, C.c_int,
                                  C.c_uint64, C.c_int64, C.POINTER(C.c_float)]
        R.ref_streamed_weight_bytes.restype = C.c_uint64
        R.ref_streamed_weight_bytes.argtypes = [C.POINTER(FoConfig)]
        R.ref_total_weight_bytes.restype = C.c_uint64
        R.ref_total_weight_bytes.argtypes = [C.POINTER(FoConfig)]
        R.ref_linear_init.restype = C.c_void_p
        R.ref_linear_init.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64]
        R.ref_linear_forward.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_double)]
        R.ref_save_store.argtypes = [C.c_void_p, C.c_char_p]
        R.ref_load_store.restype = C.c_void_p
        R.ref_load_store.argtypes = [C.c_char_p, C.c_int64]
        R.ref_time_forward.restype = C.c_double
        R.ref_time_forward.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int64, C.c_int]
        R.ref_simulate.argtypes = [C.POINTER(FoConfig), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int64,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p, C.c_int64]
        _ref = R
    return _ref


# B200 defaults for the reference simulator's HardwareConfig (config.hpp:88-96):
# 148 SMs, 228 KiB shared memory; peak bandwidth from MEASURED_PEAKS.json when
# the caller passes it.  Launch overhead / barrier latency / compute rate keep
# the reference's calibrated defaults unless overridden.
B200_HW = dict(num_sms=148, shared_mem_per_sm=228 * 1024, peak_bandwidth=8.0e12,
               kernel_launch_overhead=8e-6, barrier_latency=3e-7, compute_throughput_per_sm=8e10)


def ref_simulate(cfg: ModelCfg, seq_len: int, mode: int = 2, stage_size: int = 32768, depth: int = 6,
                 warps: int = 8, attn_group: int = 8, hw: dict | None = None,
                 eff: tuple = (-1.0, -1.0, -1.0, -1.0)) -> dict:
    """fusesim::simulate (simulate.hpp:423) of one decode step on the
    reference's own schedule (build_plan + emit_programs) -- the reference's
    cost model, here fed a B200 hardware description.  mode 0/1/2 =
    Baseline / Fused / FusedOverlap.  eff = (weight_matvec, kv_attention,
    glu, load_issue_cost); negative keeps the reference default.  Returns
    {"total": s, "bytes": B, "sublayers": {name: s}}."""
    h = dict(B200_HW)
    h.update(hw or {})
    hwv = (C.c_double * 6)(h["num_sms"], h["shared_mem_per_sm"], h["peak_bandwidth"],
                           h["kernel_launch_overhead"], h["barrier_latency"], h["compute_throughput_per_sm"])
    ev = (C.c_double * 4)(*eff)
    tot, nb = C.c_double(), C.c_double()
    buf = C.create_string_buffer(4096)
    R = ref_lib()
    fc = cfg.c()
    rc = R.ref_simulate(C.byref(fc), hwv, ev, stage_size, depth, warps, seq_len, mode, attn_group,
                        C.byref(tot), C.byref(nb), buf, 4096)
    if rc != 0:
        raise RuntimeError(R.ref_last_error().decode())
    subs = {}
    for kv in buf.value.decode().split(";"):
        if kv:
            k, v = kv.split("=")
            subs[k] = float(v)
    return {"total": tot.value, "bytes": nb.value, "sublayers": subs}


class RefStore:
    """fusesim::TensorStore built by the unmodified reference (oracle/_ref)."""

    def __init__(self, cfg: ModelCfg, seed: int | None, max_seq_len: int):
        R = ref_lib()
        self.cfg = cfg
        self._c = cfg.c()
        if seed is None:
            self._h = R.ref_init_fast(C.byref(self._c), max_seq_len)
        else:
            self._h = R.ref_init_weights(C.byref(self._c), seed, max_seq_len)
        if not self._h:
            raise ValueError(R.ref_last_error().decode())
        self.max_seq_len = max_seq_len

    @classmethod
    def load(cls, path: str, cfg: ModelCfg, max_seq_len: int) -> "RefStore":
        """fusesim::load_store, unchanged (it rebuilds shapes with
        init_weights(model, 0) first, so it is slow for large models)."""
        R = ref_lib()
        h = R.ref_load_store(os.fsencode(path), max_seq_len)
        if not h:
            raise ValueError(R.ref_last_error().decode())
        self = cls.__new__(cls)
        self._h, self.cfg, self._c, self.max_seq_len = h, cfg, cfg.c(), max_seq_len
        return self

    def save(self, path: str):
        if ref_lib().ref_save_store(self._h, os.fsencode(path)) != 0:
            raise ValueError(ref_lib().ref_last_error().decode())

    def close(self):
        if getattr(self, "_h", None):
            ref_lib().ref_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def tensor(self, name: str) -> np.ndarray:
        R = ref_lib()
        n = R.ref_get_tensor(self._h, name.encode(), None)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, dtype=np.float32)
        R.ref_get_tensor(self._h, name.encode(), _p(out))
        return out

    def synthetic_prefill(self, prefill: int, seed: int):
        ref_lib().ref_synthetic_prefill(self._h, prefill, seed)

    def set_length(self, layer: int, n: int):
        ref_lib().ref_kv_set_length(self._h, layer, n)

    def length(self, layer: int) -> int:
        return ref_lib().ref_kv_length(self._h, layer)

    def kv_get(self, b, l, h, pos):
        dh = self.cfg.d_head
        k = np.empty(dh, np.float32)
        v = np.empty(dh, np.float32)
        ref_lib().ref_kv_get(self._h, b, l, h, pos, _p(k), _p(v))
        return k, v

    def forward(self, tokens, pos: int) -> np.ndarray:
        c = self.cfg
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
        out = np.zeros((c.batch, c.vocab_size), dtype=np.float64)
        rc = ref_lib().ref_forward(self._h, _p(tok, C.c_int64), pos, _p(out, C.c_double))
        if rc != 0:
            raise ValueError(ref_lib().ref_last_error().decode())
        return out

    def execute(self, tokens, pos: int, mode: int = 2, stage_size: int = 32768,
                num_sms: int = 132) -> np.ndarray:
        c = self.cfg
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
        out = np.zeros((c.batch, c.vocab_size), dtype=np.float32)
        rc = ref_lib().ref_execute(self._h, _p(tok, C.c_int64), pos, mode, stage_size, num_sms,
                                   _p(out))
        if rc != 0:
            raise ValueError(ref_lib().ref_last_error().decode())
        return out

    def time_forward(self, tokens, pos: int, steps: int) -> float:
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
        return ref_lib().ref_time_forward(self._h, _p(tok, C.c_int64), pos, steps)


# ---------------------------------------------------------------- presets
# fusesim presets (presets.hpp:19-60) + BASELINE.json configs (SURVEY.md §8 tags)
PRESETS = {
    "llama31_8b-toy": ModelCfg(4, 256, 896, 64, 4, 2, 512),
    "tiny": ModelCfg(4, 512, 1792, 64, 8, 2, 32000),                 # T
    "llama32_1b": ModelCfg(16, 2048, 8192, 64, 32, 8, 128256),        # S
    "llama31_8b": ModelCfg(32, 4096, 14336, 128, 32, 8, 128256),      # E
    "llama31_70b": ModelCfg(80, 8192, 28672, 128, 64, 8, 128256),     # H
}


def preset(name: str) -> ModelCfg:
    return PRESETS[name]


def tiny_prompt(n: int = 128, vocab: int = 32000) -> list[int]:
    """T config prompt: n ids from std::mt19937(5)() % vocab."""
    L = lib()

    class MT32(C.Structure):
        _fields_ = [("mt", C.c_uint32 * 624), ("idx", C.c_int)]
    g = MT32()
    L.fo_mt32_seed(C.byref(g), C.c_uint32(5))
    return [int(L.fo_mt32_next(C.byref(g)) % vocab) for _ in range(n)]


class LinearOracle:
    """Stacked-linear kind (test infrastructure): the C restatement of
    init_weights' "linear.<l>" tensors and of reference_linear_forward
    (reference.hpp:141-152), f64."""

    def __init__(self, layers: int, d_model: int, batch: int = 1, seed: int = 1234, dtype: int = 0):
        self.layers, self.d_model, self.batch = layers, d_model, batch
        L = lib()
        L.fo_fill_linear.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_uint64, C.c_int32,
                                     C.POINTER(C.c_float)]
        L.fo_linear_forward.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_float), C.POINTER(C.c_double)]
        self.w = np.empty((layers, d_model, d_model), np.float32)
        for l in range(layers):
            L.fo_fill_linear(f"linear.{l}".encode(), d_model, d_model, seed, dtype,
                             _p(self.w[l]))

    def tensor(self, name: str) -> np.ndarray:
        return self.w[int(name.split(".")[1])]

    def forward(self, x0: np.ndarray) -> np.ndarray:
        x0 = np.ascontiguousarray(x0, np.float32).reshape(self.batch, self.d_model)
        out = np.empty((self.batch, self.d_model), np.float64)
        lib().fo_linear_forward(_p(self.w), self.layers, self.d_model, self.batch, _p(x0),
                                _p(out, C.c_double))
        return out


class RefLinear:
    """The same from the unmodified reference (oracle/_ref)."""

    def __init__(self, layers: int, d_model: int, batch: int = 1, seed: int = 1234):
        R = ref_lib()
        self.layers, self.d_model, self.batch = layers, d_model, batch
        self._h = R.ref_linear_init(layers, d_model, batch, seed)
        if not self._h:
            raise ValueError(R.ref_last_error().decode())

    def tensor(self, name: str) -> np.ndarray:
        R = ref_lib()
        out = np.empty((self.d_model, self.d_model), np.float32)
        if R.ref_get_tensor(self._h, name.encode(), _p(out)) < 0:
            raise KeyError(name)
        return out

    def forward(self, x0: np.ndarray) -> np.ndarray:
        x0 = np.ascontiguousarray(x0, np.float32).reshape(self.batch, self.d_model)
        out = np.empty((self.batch, self.d_model), np.float64)
        if ref_lib().ref_linear_forward(self._h, _p(x0), _p(out, C.c_double)):
            raise ValueError(ref_lib().ref_last_error().decode())
        return out

    def close(self):
        if getattr(self, "_h", None):
            ref_lib().ref_free(self._h)
            self._h = None

    def __del__(self):
        self.close()
