"""B200-native FlashFormer decode step (arxiv 2505.22758).

Host-side mirror of the reference's decode interface
(/root/reference/proj/include/fusesim/):

  fusesim::ModelConfig            config.hpp:45-86       -> ModelConfig
  fusesim::ValidationError, ...   types.hpp:17-31        -> ValidationError, ...
  fusesim::RunMode                types.hpp:64           -> RunMode
  fusesim::TensorStore + KVCache  tensor_store.hpp:63-366 -> DecodeModel (device store)
  fusesim::execute_program /      interpreter.hpp:502-506,
  fusesim::reference_forward      reference.hpp:37-139   -> DecodeModel.forward

Everything runs through the C-ABI in ``include/flashformer_b200.h`` implemented
by ``libffb200.so`` (hand-written sm_100a CUDA).  There is no CPU path: if the
library is missing or no B200 is visible, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, replace

import numpy as np

__all__ = [
    "ModelConfig", "RunMode", "DecodeModel", "ValidationError", "DeviceError",
    "UnsupportedConfigError", "UsageError", "PRESETS", "model_preset", "lib", "LIB_PATH",
    "tensor_names", "pack_quant_rows", "unpack_quant_rows", "tp_shard", "tp_unshard",
    "TPGroup", "all_gather_tp_blobs",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFB200_LIB") or os.path.join(HERE, "libffb200.so")


class FusesimError(RuntimeError):
    pass


class UsageError(FusesimError):          # CLI exit 1
    pass


class ValidationError(FusesimError):     # fusesim::ValidationError, exit 2
    pass


class DeviceError(FusesimError):         # CUDA failure, exit 3
    pass


class UnsupportedConfigError(FusesimError):
    pass


_STATUS = {1: UsageError, 2: ValidationError, 3: DeviceError, 4: UnsupportedConfigError}


class RunMode(enum.IntEnum):
    """fusesim::RunMode (types.hpp:64)."""
    BASELINE = 0        # one launch per sublayer stage (multi-kernel variant)
    FUSED = 1           # one persistent launch, producer waits at barriers
    FUSED_OVERLAP = 2   # one persistent launch, producer streams across barriers
    BASELINE_NCCL = 3   # TP only: BASELINE launches + host ncclAllReduce between them


class _Cfg(C.Structure):
    _fields_ = [
        ("layers", C.c_int64), ("d_model", C.c_int64), ("d_inter", C.c_int64),
        ("d_head", C.c_int64), ("n_q_heads", C.c_int64), ("n_kv_heads", C.c_int64),
        ("vocab_size", C.c_int64), ("rope_theta", C.c_double), ("rmsnorm_eps", C.c_double),
        ("dtype", C.c_int32), ("quant_bits", C.c_int32), ("quant_group", C.c_int32),
        ("batch", C.c_int64), ("kind", C.c_int32), ("reserved_", C.c_int32),
    ]


class _Info(C.Structure):
    _fields_ = [
        ("grid", C.c_int32), ("threads", C.c_int32), ("smem_bytes", C.c_int32),
        ("ring_slots", C.c_int32), ("slot_bytes", C.c_int32), ("attn_group", C.c_int32),
        ("launches_per_step", C.c_int32), ("mode", C.c_int32),
        ("weight_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
        ("quant_inexact_groups", C.c_uint64), ("row_bytes", C.c_int32), ("kc_layout", C.c_int32),
        ("fp16_inexact", C.c_uint64),
    ]


@dataclass(frozen=True)
class ModelConfig:
    """fusesim::ModelConfig (config.hpp:45-86), decoder kind."""
    layers: int
    d_model: int
    d_inter: int
    d_head: int
    n_q_heads: int
    n_kv_heads: int
    vocab_size: int
    rope_theta: float = 500000.0
    rmsnorm_eps: float = 1e-5
    dtype: int = 0
    quant_bits: int = 0
    quant_group: int = 128
    batch: int = 1
    kind: int = 0           # 0 llama_decoder, 1 stacked_linear (config.hpp:18)

    @property
    def qkv_rows(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.d_head

    @property
    def q_group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    def replace(self, **kw) -> "ModelConfig":
        return replace(self, **kw)

    def _c(self) -> _Cfg:
        return _Cfg(self.layers, self.d_model, self.d_inter, self.d_head, self.n_q_heads,
                    self.n_kv_heads, self.vocab_size, self.rope_theta, self.rmsnorm_eps,
                    self.dtype, self.quant_bits, self.quant_group, self.batch, self.kind, 0)

    def streamed_weight_bytes(self) -> int:
        """StoreLayout::streamed_weight_bytes (tensor_store.hpp:170-174)."""
        if self.kind == 1:  # linear layers are never quantized (tensor_store.hpp:199)
            return self.layers * self.d_model * self.d_model * 2
        if self.quant_bits == 4:
            row = self.d_model // 2 + (self.d_model // self.quant_group) * 4
        elif self.quant_bits == 8:
            row = self.d_model + (self.d_model // self.quant_group) * 4
        else:
            row = self.d_model * 2
        rows = self.layers * (self.qkv_rows + self.d_model + 3 * self.d_inter) + self.vocab_size
        return rows * row

    def kv_bytes_per_position(self) -> int:
        """StoreLayout::kv_bytes_per_position (tensor_store.hpp:188-192)."""
        return self.batch * self.layers * self.n_kv_heads * 2 * self.d_head * 2


PRESETS = {
    # fusesim presets (presets.hpp:19-47)
    "llama31_8b-toy": ModelConfig(4, 256, 896, 64, 4, 2, 512),
    "llama31_8b": ModelConfig(32, 4096, 14336, 128, 32, 8, 128256),
    "llama31_70b": ModelConfig(80, 8192, 28672, 128, 64, 8, 128256),
    # BASELINE.json configs (SURVEY.md §8 tags T, S)
    "tiny": ModelConfig(4, 512, 1792, 64, 8, 2, 32000),
    "llama32_1b": ModelConfig(16, 2048, 8192, 64, 32, 8, 128256),
    # stacked-linear presets (presets.hpp:48-55): 32 square layers
    "stacked_linear_2k": ModelConfig(32, 2048, 0, 0, 0, 0, 0, kind=1),
    "stacked_linear_4k": ModelConfig(32, 4096, 0, 0, 0, 0, 0, kind=1),
    "stacked_linear_8k": ModelConfig(32, 8192, 0, 0, 0, 0, 0, kind=1),
}


def model_preset(name: str) -> ModelConfig:
    """fusesim::model_preset (presets.hpp:19-60) for the decoder presets."""
    if name not in PRESETS:
        raise ValidationError(f"unknown model preset: {name}")
    return PRESETS[name]


def pack_quant_rows(values: np.ndarray, quant_bits: int, layout: int = 0) -> tuple[np.ndarray, int]:
    """Host weight packer (ffb_pack_quant_rows_ex): f32 [rows][cols] -> device
    row format bytes [rows][row_bytes], plus the count of groups that lie on
    no int4/int8 grid (packed lossily).  layout 1 = tensor-core code order."""
    v = np.ascontiguousarray(values, np.float32)
    rows, cols = v.shape
    rb = lib().ffb_quant_row_bytes(cols, quant_bits)
    if rb < 0:
        raise UsageError(f"unsupported quant row: cols={cols} bits={quant_bits}")
    out = np.zeros((rows, rb), np.uint8)
    n = lib().ffb_pack_quant_rows_ex(_fp(v), rows, cols, quant_bits, layout,
                                     out.ctypes.data_as(C.POINTER(C.c_uint8)))
    if n < 0:
        raise UsageError(lib().ffb_last_error().decode())
    return out, int(n)


def tc_code_positions(quant_bits: int) -> np.ndarray:
    """Column i of a 128-column group -> nibble (int4) / byte (int8)
    position in the tensor-core code order (runtime.cu: tc_nibble_index,
    tc_byte_index; decode_kernel.cuh: tc_slot, the mma.sync m16n8k32 u8 A
    fragments): lane quad q of k32-step s owns columns 32s + 4q + j (low
    nibbles / first 4 bytes) and 32s + 16 + 4q + j (high nibbles / last 4)."""
    i = np.arange(128)
    s, r = i // 32, i % 32
    half, q, j = r // 16, (r % 16) // 4, r % 4
    if quant_bits == 4:
        return q * 32 + s * 8 + 2 * j + half
    return q * 32 + s * 8 + half * 4 + j


def unpack_quant_rows(packed: np.ndarray, cols: int, quant_bits: int,
                      layout: int = 0) -> np.ndarray:
    """Inverse of pack_quant_rows: (code - zero) * scale in f32 (quant.hpp:23-25)."""
    ng = cols // 128
    cb = cols // 2 if quant_bits == 4 else cols
    codes = packed[:, :cb]
    if quant_bits == 4:
        c = np.empty((packed.shape[0], cols), np.uint8)
        c[:, 0::2] = codes & 0xF
        c[:, 1::2] = codes >> 4
    else:
        c = codes.copy()
    if layout == 1:  # stored position -> column
        pos = (np.arange(ng)[:, None] * 128 + tc_code_positions(quant_bits)[None, :]).ravel()
        c = c[:, pos]
    scale = packed[:, cb:cb + 4 * ng].copy().view(np.float32)
    zero = packed[:, cb + 4 * ng:cb + 5 * ng].astype(np.float32)
    g = np.arange(cols) // 128
    return ((c.astype(np.float32) - zero[:, g]) * scale[:, g]).astype(np.float32)


def tp_shard(cfg: ModelConfig, name: str, full: np.ndarray, rank: int, tp: int) -> np.ndarray:
    """Host restatement of the TP shard of one reference tensor (what
    ffb_upload_tensor keeps on rank `rank`, runtime.cu: resolve): Wqkv rows
    of the rank's q heads, then k heads, then v heads; Waout all rows x the
    rank's q-head columns; Wffn1 / Wffn2^T rows of d_inter slice r; lm_head
    vocab rows of slice r; everything else replicated."""
    if tp == 1:
        return full
    dh = cfg.d_head
    nq, nkv = cfg.n_q_heads // tp, cfg.n_kv_heads // tp
    ad, kv = nq * dh, nkv * dh
    gq, gk = cfg.n_q_heads * dh, cfg.n_kv_heads * dh
    di, v = cfg.d_inter // tp, cfg.vocab_size // tp
    t = name.split(".")[-1]
    if t == "wqkv":
        return np.concatenate([full[rank * ad:(rank + 1) * ad],
                               full[gq + rank * kv:gq + (rank + 1) * kv],
                               full[gq + gk + rank * kv:gq + gk + (rank + 1) * kv]])
    if t == "waout":
        return full[:, rank * ad:(rank + 1) * ad]
    if t == "wffn1":
        return full[2 * rank * di:2 * (rank + 1) * di]
    if t == "wffn2t":
        return full[rank * di:(rank + 1) * di]
    if name == "lm_head":
        return full[rank * v:(rank + 1) * v]
    return full


def tp_unshard(cfg: ModelConfig, name: str, shards: list[np.ndarray]) -> np.ndarray:
    """Inverse of tp_shard (replicated tensors: rank 0's copy)."""
    tp = len(shards)
    if tp == 1:
        return shards[0]
    t = name.split(".")[-1]
    if t == "wqkv":
        dh = cfg.d_head
        ad, kv = cfg.n_q_heads // tp * dh, cfg.n_kv_heads // tp * dh
        return np.concatenate([s[:ad] for s in shards] + [s[ad:ad + kv] for s in shards] +
                              [s[ad + kv:] for s in shards])
    if t == "waout":
        return np.concatenate(shards, axis=1)
    if t in ("wffn1", "wffn2t") or name == "lm_head":
        return np.concatenate(shards)
    return shards[0]


def all_gather_tp_blobs(blob: bytes, group=None) -> list[bytes]:
    """Multi-process TP wiring: all-gather every rank's ffb_tp_export blob
    over torch.distributed (any backend), ordered by rank."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    return out


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for ffb_tp_nccl_init (rank 0 makes
    it, the caller broadcasts it)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().ffb_nccl_unique_id(buf))
    return bytes(buf)


def broadcast_nccl_id(group=None) -> bytes:
    """Rank 0's ncclUniqueId on every rank (torch.distributed, any backend)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def tensor_names(cfg: ModelConfig) -> list[str]:
    """Reference tensor names (tensor_store.hpp:339-363) in upload order."""
    if cfg.kind == 1:
        return [f"linear.{l}" for l in range(cfg.layers)]
    names = []
    for l in range(cfg.layers):
        names += [f"layer.{l}.{t}" for t in
                  ("wqkv", "waout", "wffn1", "wffn2t", "norm_attn", "norm_ffn")]
    return names + ["final_norm", "embedding", "lm_head"]


_lib = None


def lib():
    """Load libffb200.so (fails loudly; there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(f"CUDA extension not built: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.ffb_last_error.restype = C.c_char_p
    L.ffb_version.restype = C.c_char_p
    L.ffb_config_supported.argtypes = [P(_Cfg)]
    L.ffb_create.argtypes = [P(_Cfg), C.c_int64, C.c_int, C.c_int, C.c_int, P(C.c_void_p)]
    L.ffb_create_ex.argtypes = [P(_Cfg), C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                P(C.c_void_p)]
    L.ffb_tp_blob_bytes.restype = C.c_int64
    L.ffb_tp_export.argtypes = [C.c_void_p, C.c_void_p]
    L.ffb_tp_connect.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
    L.ffb_nccl_unique_id.argtypes = [C.c_void_p]
    L.ffb_tp_nccl_init.argtypes = [C.c_void_p, C.c_void_p]
    L.ffb_destroy.argtypes = [C.c_void_p]
    L.ffb_destroy.restype = None
    L.ffb_upload_tensor.argtypes = [C.c_void_p, C.c_char_p, P(C.c_float), C.c_int64]
    L.ffb_init_synthetic.argtypes = [C.c_void_p, C.c_uint64]
    L.ffb_kv_set.argtypes = [C.c_void_p] + [C.c_int64] * 4 + [P(C.c_float)] * 2
    L.ffb_kv_get.argtypes = [C.c_void_p] + [C.c_int64] * 4 + [P(C.c_float)] * 2
    L.ffb_kv_import.argtypes = [C.c_void_p, P(C.c_float), P(C.c_float), C.c_int64, C.c_int64]
    L.ffb_sync.argtypes = [C.c_void_p]
    L.ffb_kv_export.argtypes = [C.c_void_p, C.c_int64, C.c_int64, P(C.c_float), P(C.c_float)]
    L.ffb_load_store.argtypes = [C.c_void_p, C.c_char_p]
    L.ffb_save_image.argtypes = [C.c_void_p, C.c_char_p]
    L.ffb_load_image.argtypes = [C.c_void_p, C.c_char_p]
    L.ffb_kv_set_length.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
    L.ffb_kv_length.argtypes = [C.c_void_p, C.c_int64]
    L.ffb_kv_length.restype = C.c_int64
    L.ffb_set_mode.argtypes = [C.c_void_p, C.c_int]
    L.ffb_set_debug.argtypes = [C.c_void_p, C.c_int32]
    L.ffb_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    L.ffb_set_trace.argtypes = [C.c_void_p, C.c_int]
    L.ffb_get_trace.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]
    L.ffb_get_trace.restype = C.c_int64
    # (raw addresses: the per-token host path avoids ctypes pointer objects)
    L.ffb_decode_step.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ffb_decode_step_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
    L.ffb_get_info.argtypes = [C.c_void_p, P(_Info)]
    L.ffb_decode_loop.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                  C.c_void_p, C.c_void_p]
    L.ffb_prefill.argtypes = [C.c_void_p, P(C.c_int64), C.c_int64, C.c_int64, P(C.c_float),
                              P(C.c_int64)]
    L.ffb_linear_forward.argtypes = [C.c_void_p, P(C.c_float), P(C.c_float), C.c_void_p]
    L.ffb_linear_forward_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ffb_logits_device.argtypes = [C.c_void_p]
    L.ffb_logits_device.restype = C.c_void_p
    L.ffb_quant_row_bytes.argtypes = [C.c_int64, C.c_int32]
    L.ffb_quant_row_bytes.restype = C.c_int64
    L.ffb_pack_quant_rows.argtypes = [P(C.c_float), C.c_int64, C.c_int64, C.c_int32,
                                      P(C.c_uint8)]
    L.ffb_pack_quant_rows.restype = C.c_int64
    L.ffb_calibrate.argtypes = [C.c_void_p, C.c_int32]
    L.ffb_get_plan_weights.argtypes = [C.c_void_p, P(C.c_double), C.c_int64]
    L.ffb_get_plan_weights.restype = C.c_int64
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = lib().ffb_last_error().decode()
        raise _STATUS.get(rc, FusesimError)(msg)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class DecodeModel:
    """Device-resident decoder: weights, KV cache and the decode kernel.

    Mirrors the mutable state the reference threads through
    ``TensorStore&`` (weights + ``KVCache``) and the two entry points that
    consume it.  ``forward(tokens, pos)`` has reference_forward's contract
    (reference.hpp:37-139): pos must equal every layer's cache length, one KV
    position per layer is appended, logits[batch][vocab] are returned.
    """

    def __init__(self, cfg: ModelConfig, max_seq_len: int, device: int = 0,
                 mode: RunMode = RunMode.FUSED_OVERLAP, tp_rank: int = 0, tp_size: int = 1,
                 grid: int = 0):
        """cfg is the WHOLE model; with tp_size > 1 this handle is shard
        tp_rank (ffb_create_ex) and must be connected to its
        peers (tp_connect) before stepping."""
        L = lib()
        self.cfg = cfg
        self.tp_rank, self.tp_size = tp_rank, tp_size
        self.device = device
        self.max_seq_len = max_seq_len
        self._c = cfg._c()
        h = C.c_void_p()
        _check(L.ffb_create_ex(C.byref(self._c), max_seq_len, device, tp_rank, tp_size, grid,
                               C.byref(h)))
        self._h = h
        self.set_mode(mode)

    # ------------------------------------------------------------ TP wiring
    def tp_blob(self) -> bytes:
        """This rank's exchange-buffer descriptor (ffb_tp_export)."""
        buf = C.create_string_buffer(lib().ffb_tp_blob_bytes())
        _check(lib().ffb_tp_export(self._h, buf))
        return buf.raw

    def tp_connect(self, blobs: list[bytes]):
        """Connect to every rank's blob, ordered by rank (ffb_tp_connect)."""
        raw = b"".join(blobs)
        _check(lib().ffb_tp_connect(self._h, C.create_string_buffer(raw, len(raw)), len(blobs)))

    def tp_nccl_init(self, nccl_id: bytes):
        """This rank's NCCL communicator for RunMode.BASELINE_NCCL
        (ffb_tp_nccl_init; collective over the TP ranks)."""
        _check(lib().ffb_tp_nccl_init(self._h, C.create_string_buffer(nccl_id, 128)))

    @staticmethod
    def supported(cfg: ModelConfig) -> bool:
        c = cfg._c()
        return bool(lib().ffb_config_supported(C.byref(c)))

    def close(self):
        if getattr(self, "_h", None):
            lib().ffb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------ weights
    def upload_tensor(self, name: str, values: np.ndarray):
        a = np.ascontiguousarray(values, dtype=np.float32).ravel()
        _check(lib().ffb_upload_tensor(self._h, name.encode(), _fp(a), a.size))

    def upload_store(self, store):
        """Pack every tensor of a TensorStore-like object (``store.tensor(name)``)."""
        for n in tensor_names(self.cfg):
            self.upload_tensor(n, store.tensor(n))

    def init_synthetic(self, seed: int = 1234):
        _check(lib().ffb_init_synthetic(self._h, seed))

    def load_store(self, path: str):
        """Pack a fusesim "FSTW" v1 store file (save_store, tensor_store.hpp:
        410-444) into the device weights (ffb_load_store)."""
        _check(lib().ffb_load_store(self._h, os.fsencode(path)))

    def save_image(self, path: str):
        """Write the packed device weights (ffb_save_image)."""
        _check(lib().ffb_save_image(self._h, os.fsencode(path)))

    def load_image(self, path: str):
        """Reload a packed device image of the same model / shard / kernel."""
        _check(lib().ffb_load_image(self._h, os.fsencode(path)))

    # ------------------------------------------------------------ KV cache
    def kv_set(self, b, layer, head, pos, k, v):
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        _check(lib().ffb_kv_set(self._h, b, layer, head, pos, _fp(k), _fp(v)))

    def kv_get(self, b, layer, head, pos):
        dh = self.cfg.d_head
        k = np.empty(dh, np.float32)
        v = np.empty(dh, np.float32)
        _check(lib().ffb_kv_get(self._h, b, layer, head, pos, _fp(k), _fp(v)))
        return k, v

    def kv_export(self, pos0: int, n_pos: int = 1):
        """Positions [pos0, pos0 + n_pos) as (K, V) f32 [B][L][Hkv][n_pos][dh]
        (ffb_kv_export; one gather + one copy)."""
        c = self.cfg
        shp = (c.batch, c.layers, c.n_kv_heads // self.tp_size, n_pos, c.d_head)
        k = np.empty(shp, np.float32)
        v = np.empty(shp, np.float32)
        _check(lib().ffb_kv_export(self._h, pos0, n_pos, _fp(k), _fp(v)))
        return k, v

    def kv_import(self, k: np.ndarray, v: np.ndarray, n_pos: int):
        """Import a reference-layout cache [B][L][Hkv][S][dh] (positions < n_pos)
        and set every layer's length to n_pos."""
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        _check(lib().ffb_kv_import(self._h, _fp(k), _fp(v), k.shape[3], n_pos))
        for l in range(self.cfg.layers):
            self.set_length(l, n_pos)

    def set_length(self, layer: int, n: int):
        _check(lib().ffb_kv_set_length(self._h, layer, n))

    def length(self, layer: int) -> int:
        return lib().ffb_kv_length(self._h, layer)

    # ------------------------------------------------------------ execution
    def set_mode(self, mode: RunMode):
        _check(lib().ffb_set_mode(self._h, int(mode)))
        self.mode = RunMode(mode)

    def set_option(self, key: str, value: int):
        """Tuning knobs (ffb_set_option), e.g. ("l2_prefetch_bytes", 262144)."""
        _check(lib().ffb_set_option(self._h, key.encode(), int(value)))

    def calibrate(self, iterations: int = 3):
        """Per-SM load balance from measured streaming rates (ffb_calibrate);
        0 restores the uniform plan."""
        _check(lib().ffb_calibrate(self._h, int(iterations)))

    def plan_weights(self) -> np.ndarray:
        n = lib().ffb_get_plan_weights(self._h, None, 0)
        out = np.zeros(n, np.float64)
        lib().ffb_get_plan_weights(self._h, out.ctypes.data_as(C.POINTER(C.c_double)), n)
        return out

    def set_debug(self, flags: int):
        """Diagnostics only (ffb_set_debug): 1 = streaming-only run."""
        _check(lib().ffb_set_debug(self._h, flags))

    def set_trace(self, enable: bool = True):
        """Per-CTA stage timestamps of the next steps (ffb_set_trace)."""
        _check(lib().ffb_set_trace(self._h, 1 if enable else 0))

    def trace(self) -> np.ndarray:
        """[grid][5L+1][8] u64: stage entry, dependency met, stage done, stage
        mark (ns timestamps), ns starved on ring data, spare."""
        n = lib().ffb_get_trace(self._h, None, 0)
        if n < 0:
            raise DeviceError("tracing not enabled")
        out = np.zeros(n, np.uint64)
        if lib().ffb_get_trace(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)), n) < 0:
            raise DeviceError(lib().ffb_last_error().decode())
        return out.reshape(self.info()["grid"], self.cfg.layers * 5 + 1, 8)

    def step(self, tokens, pos: int, logits: bool = True, out: np.ndarray | None = None,
             greedy: np.ndarray | None = None, stream: int = 0):
        """One decode step; returns (logits f32 [B][V] or None, greedy int64 [B]).

        ``out``/``greedy`` may be preallocated (ideally pinned) host buffers;
        ``stream`` is a cudaStream_t handle (0 = the model's own stream)."""
        c = self.cfg
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64).reshape(-1))
        if tok.size != c.batch:
            raise ValidationError("execute_program: one token per batch row required")
        if out is None and logits:  # a TP rank returns its vocabulary slice
            out = np.empty((c.batch, c.vocab_size // self.tp_size), np.float32)
        elif out is not None:
            if (out.dtype != np.float32 or not out.flags.c_contiguous
                    or out.size < c.batch * (c.vocab_size // self.tp_size)):
                raise UsageError("step: out must be C-contiguous f32 with room for [batch][vocab / tp]")
        if greedy is None:
            greedy = np.empty(c.batch, np.int64)
        elif greedy.dtype != np.int64 or not greedy.flags.c_contiguous or greedy.size < c.batch:
            raise UsageError("step: greedy must be C-contiguous int64 [batch]")
        addr = lambda a: a.__array_interface__["data"][0]  # noqa: E731
        _check(lib().ffb_decode_step(self._h, addr(tok), pos, addr(out) if out is not None else None,
                                     addr(greedy), stream or None))
        return out, greedy

    def forward(self, tokens, pos: int) -> np.ndarray:
        """reference_forward / execute_program contract: logits [batch][vocab]."""
        return self.step(tokens, pos, logits=True)[0]

    def step_device(self, d_tokens: int, pos: int, d_logits: int = 0, d_greedy: int = 0,
                    stream: int = 0):
        """Asynchronous step on raw device pointers (e.g. torch ``data_ptr()``)."""
        _check(lib().ffb_decode_step_device(self._h, C.c_void_p(d_tokens), pos,
                                            C.c_void_p(d_logits or None),
                                            C.c_void_p(d_greedy or None),
                                            C.c_void_p(stream or None)))

    def sync(self):
        """Wait for enqueued steps; raise ValidationError if a device-resident
        token id was out of range (ffb_sync)."""
        _check(lib().ffb_sync(self._h))

    def prefill(self, tokens, pos: int = 0, logits: bool = True):
        """Prompt ingestion as GEMMs (ffb_prefill): tokens [n][batch] at
        positions pos .. pos+n-1; returns (logits f32 [B][V] or None, greedy
        int64 [B]) of the last position.  The cache ends at pos + n, exactly
        where n decode steps would leave it; prompts longer than 1024 rows
        (n * batch) are fed in chunks."""
        c = self.cfg
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64))
        if tok.ndim == 1:
            tok = tok.reshape(-1, 1) if c.batch == 1 else tok.reshape(1, -1)
        if tok.ndim != 2 or tok.shape[1] != c.batch or tok.shape[0] == 0:
            raise ValidationError("prefill: tokens must be [n][batch]")
        out = np.empty((c.batch, c.vocab_size), np.float32) if logits else None
        greedy = np.empty(c.batch, np.int64)
        chunk = max(1, 1024 // c.batch)
        for t0 in range(0, tok.shape[0], chunk):
            part = np.ascontiguousarray(tok[t0:t0 + chunk])
            last = t0 + chunk >= tok.shape[0]
            _check(lib().ffb_prefill(self._h, part.ctypes.data_as(C.POINTER(C.c_int64)),
                                     part.shape[0], pos + t0,
                                     _fp(out) if (last and out is not None) else None,
                                     greedy.ctypes.data_as(C.POINTER(C.c_int64))))
        return out, greedy

    def decode_loop(self, d_tokens: int, pos: int, n_steps: int, d_out: int,
                    teacher_forced: bool = False, stream: int = 0):
        """Device-resident multi-token decode (ffb_decode_loop): raw device
        pointers, asynchronous on `stream`."""
        _check(lib().ffb_decode_loop(self._h, C.c_void_p(d_tokens), pos, n_steps,
                                     1 if teacher_forced else 0, C.c_void_p(d_out),
                                     C.c_void_p(stream or None)))

    def generate(self, tokens, pos: int, n_steps: int, prompt=None, use_prefill: bool = False) -> np.ndarray:
        """Greedy generation on the device (decode_loop): returns the n_steps
        produced tokens int64 [n_steps][batch].  With `prompt` ([n][batch],
        from `pos`), token 0 is the prediction after the prompt -- ingested
        teacher-forced through the decode loop (the reference's
        decode-as-prefill), or with `use_prefill` through ffb_prefill's GEMMs;
        otherwise `tokens` ([batch]) is consumed at `pos` first.  The cache
        ends holding every consumed token."""
        import torch
        dev = f"cuda:{self.device}"
        B = self.cfg.batch
        stream = torch.cuda.Stream(device=self.device)  # (0 would mean the handle's own stream)
        with torch.cuda.stream(stream):
            return self._generate(torch, dev, B, stream.cuda_stream, tokens, pos, n_steps, prompt,
                                  use_prefill)

    def _generate(self, torch, dev, B, st, tokens, pos, n_steps, prompt, use_prefill=False):
        out = torch.empty((n_steps, B), dtype=torch.int64, device=dev)
        if prompt is not None and use_prefill:
            pr = np.asarray(prompt, np.int64).reshape(-1, B)
            _, g = self.prefill(pr, pos, logits=False)
            out[0] = torch.as_tensor(g, device=dev)
            if n_steps > 1:
                torch.cuda.current_stream().synchronize()
                self.decode_loop(out[0].data_ptr(), pos + pr.shape[0], n_steps - 1,
                                 out[1:].data_ptr(), False, st)
        elif prompt is not None:
            pr = torch.as_tensor(np.asarray(prompt, np.int64).reshape(-1, B), device=dev)
            po = torch.empty_like(pr)
            self.decode_loop(pr.data_ptr(), pos, pr.shape[0], po.data_ptr(), True, st)
            out[0] = po[-1]
            if n_steps > 1:
                self.decode_loop(po[-1].data_ptr(), pos + pr.shape[0], n_steps - 1,
                                 out[1:].data_ptr(), False, st)
        else:
            start = torch.as_tensor(np.asarray(tokens, np.int64).reshape(B), device=dev)
            self.decode_loop(start.data_ptr(), pos, n_steps, out.data_ptr(), False, st)
        torch.cuda.synchronize(self.device)
        return out.cpu().numpy()

    def linear_forward(self, x=None) -> np.ndarray:
        """Stacked-linear kind (reference_linear_forward, reference.hpp:141-152):
        x [batch][d_model] (None: the uploaded "residual") -> W_{L-1}...W_0 x."""
        c = self.cfg
        out = np.empty((c.batch, c.d_model), np.float32)
        xi = None if x is None else np.ascontiguousarray(x, np.float32).reshape(c.batch, c.d_model)
        _check(lib().ffb_linear_forward(self._h, _fp(xi) if xi is not None else None, _fp(out),
                                        None))
        return out

    def linear_forward_device(self, d_x_in: int = 0, d_x_out: int = 0, stream: int = 0):
        _check(lib().ffb_linear_forward_device(self._h, C.c_void_p(d_x_in or None),
                                               C.c_void_p(d_x_out or None),
                                               C.c_void_p(stream or None)))

    def info(self) -> dict:
        i = _Info()
        _check(lib().ffb_get_info(self._h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in _Info._fields_}

    def logits_device_ptr(self) -> int:
        return lib().ffb_logits_device(self._h) or 0


class TPGroup:
    """The ranks of one tensor-parallel group driven from ONE process: on
    several GPUs, or co-located on one GPU with the SMs split between the
    ranks (grid = SMs / tp each) -- the single-GPU test harness of the TP
    path.  Steps launch every rank asynchronously on its own stream (the
    ranks wait for each other inside the kernel), then synchronise.  Logits
    are gathered across ranks (each rank holds a vocab slice)."""

    def __init__(self, cfg: ModelConfig, max_seq_len: int, tp: int, devices=None, grid: int = 0,
                 mode: RunMode = RunMode.FUSED_OVERLAP):
        import torch
        self.torch = torch
        self.cfg, self.tp = cfg, tp
        devices = devices or [0] * tp
        if grid == 0 and len(set(devices)) < tp:
            sms = torch.cuda.get_device_properties(devices[0]).multi_processor_count
            grid = sms // tp
        self.ranks = [DecodeModel(cfg, max_seq_len, device=d, mode=mode, tp_rank=r, tp_size=tp,
                                  grid=grid) for r, d in enumerate(devices)]
        blobs = [m.tp_blob() for m in self.ranks]
        for m in self.ranks:
            m.tp_connect(blobs)
        self.streams = [torch.cuda.Stream(device=d) for d in devices]
        self.devices = devices

    def close(self):
        for m in self.ranks:
            m.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def upload_store(self, store):
        for m in self.ranks:
            m.upload_store(store)

    def init_synthetic(self, seed: int = 1234):
        for m in self.ranks:
            m.init_synthetic(seed)

    def kv_import(self, k, v, n_pos):
        for m in self.ranks:
            m.kv_import(k, v, n_pos)

    def set_length(self, layer, n):
        for m in self.ranks:
            m.set_length(layer, n)

    def set_mode(self, mode):
        for m in self.ranks:
            m.set_mode(mode)

    def length(self, layer):
        return self.ranks[0].length(layer)

    def step(self, tokens, pos: int):
        """One decode step on every rank: (logits [B][V] gathered, greedy [B])."""
        torch = self.torch
        c = self.cfg
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64).reshape(-1))
        if tok.size != c.batch:
            raise ValidationError("execute_program: one token per batch row required")
        vl = c.vocab_size // self.tp
        dts = [torch.from_numpy(tok).to(f"cuda:{d}") for d in self.devices]
        lgs = [torch.empty((c.batch, vl), dtype=torch.float32, device=f"cuda:{d}")
               for d in self.devices]
        grs = [torch.empty(c.batch, dtype=torch.int64, device=f"cuda:{d}") for d in self.devices]
        for d, s in zip(self.devices, self.streams):
            s.wait_stream(torch.cuda.current_stream(d))
        for m, t, lg, gr, s in zip(self.ranks, dts, lgs, grs, self.streams):
            m.step_device(t.data_ptr(), pos, lg.data_ptr(), gr.data_ptr(), s.cuda_stream)
        for s in self.streams:
            s.synchronize()
        greedy = [g.cpu().numpy() for g in grs]
        for g in greedy[1:]:  # every rank agrees on the global argmax
            if not np.array_equal(g, greedy[0]):
                raise DeviceError(f"TP ranks disagree on the greedy token: {greedy}")
        return np.concatenate([lg.cpu().numpy() for lg in lgs], axis=1), greedy[0]

    def forward(self, tokens, pos: int) -> np.ndarray:
        return self.step(tokens, pos)[0]
