"""Shared helpers for the GPU parity tests: build a device model from the C
oracle's TensorStore restatement (bit-identical to the reference's
init_weights, pinned by tests/test_oracle.py) and compare against the dense
f64 oracle, with the reference's own error metric."""
import os

import numpy as np

import oracle as O
from paper_2505_22758_b200 import DecodeModel, ModelConfig, RunMode

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def to_model_cfg(c: O.ModelCfg) -> ModelConfig:
    return ModelConfig(c.layers, c.d_model, c.d_inter, c.d_head, c.n_q_heads, c.n_kv_heads,
                       c.vocab_size, c.rope_theta, c.rmsnorm_eps, c.dtype, c.quant_bits,
                       c.quant_group, c.batch)


def rel_err(got, want) -> float:
    """max-abs error / max|oracle| (proj/tests/test_interpreter.cpp:32-40)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = np.abs(want).max()
    if scale == 0:
        scale = 1.0
    return float(np.abs(got - want).max() / scale)


def device_from_store(store: "O.OracleStore", max_seq_len: int | None = None,
                      mode: RunMode = RunMode.FUSED_OVERLAP) -> DecodeModel:
    cfg = to_model_cfg(store.cfg)
    m = DecodeModel(cfg, max_seq_len or store.max_seq_len, mode=mode)
    m.upload_store(store)
    k, v = store.kv()
    n = store.length(0) if store.cfg.layers > 0 else 0
    m.kv_import(k, v, n)
    return m


def bf16_ulp_distance(a, b) -> np.ndarray:
    """Distance in bf16 grid steps between values already on the bf16 grid."""
    def ordinal(x):
        u = (np.ascontiguousarray(x, np.float32).view(np.uint32) >> 16).astype(np.int64)
        return np.where(u & 0x8000, -(u & 0x7fff), u)
    return np.abs(ordinal(a) - ordinal(b))


def kv_rows_match(dev, ora) -> bool:
    """Appended K/V rows (..., d_head) agree up to one bf16 rounding flip.

    The device rounds an f32 value, the oracle an f64 one; they differ by an
    f32 accumulation error, which scales with the row (sum of |terms|), not
    with the element.  So an element may differ by one bf16 ulp of itself,
    or -- for elements near zero, where the ulp is tiny -- by 2^-16 of the
    row's largest magnitude."""
    dev = np.asarray(dev, np.float32)
    ora = np.asarray(ora, np.float32)
    row = np.abs(ora).max(axis=-1, keepdims=True)
    tol = np.abs(ora) * 2.0 ** -7 + row * 2.0 ** -16
    return bool(np.all((bf16_ulp_distance(dev, ora) <= 1) | (np.abs(dev - ora) <= tol)))


def appended_kv(m: DecodeModel, pos: int):
    """K/V rows the device appended at `pos`, as [B][L][Hkv][dh] f32 (one
    bulk ffb_kv_export)."""
    k, v = m.kv_export(pos, 1)
    return k[:, :, :, 0], v[:, :, :, 0]


def check_step(store: "O.OracleStore", m: DecodeModel, tokens, pos: int,
               strict: float = 2e-5, plain: float = 1e-4):
    """One decode step on both sides from identical state.

    * every appended K/V element equals the oracle's or differs by one bf16
      ulp (a rounding flip: the oracle rounds f64 -> f32 -> bf16, the device
      rounds an f32 value one ~1e-7 relative error away);
    * with the device's K/V rows fed to the oracle (fo_reference_forward_ex)
      the logits agree to `strict` -- the arithmetic itself;
    * without that hook they agree to the reference's own 1e-4 bound
      (test_interpreter.cpp:66) whenever no flip occurred.
    Returns (plain rel_err, strict rel_err, flips)."""
    import copy  # noqa: F401
    got = m.forward(tokens, pos)
    k_dev, v_dev = appended_kv(m, pos)
    # oracle with its own rounding
    want = store.forward(tokens, pos)
    K, V = store.kv()
    k_or = K[:, :, :, pos].copy()
    v_or = V[:, :, :, pos].copy()
    # rows of layer l are comparable while no earlier layer's row flipped (a
    # flip changes the next layer's input, the oracle's rows then legitimately
    # drift by more than one rounding step); the hooked run below checks
    # the arithmetic of every layer regardless
    flips = 0
    for l in range(store.cfg.layers):
        if flips == 0:
            for dev, ora in ((k_dev, k_or), (v_dev, v_or)):
                assert kv_rows_match(dev[:, l], ora[:, l]), f"layer {l}"
        flips += int((k_dev[:, l] != k_or[:, l]).sum() + (v_dev[:, l] != v_or[:, l]).sum())
    # rewind the oracle cache and redo the step with the device's rows
    for l in range(store.cfg.layers):
        store.set_length(l, pos)
    want_hooked = store.forward(tokens, pos, k_app=k_dev, v_app=v_dev)
    e_plain = max(rel_err(got[b], want[b]) for b in range(store.cfg.batch))
    e_strict = max(rel_err(got[b], want_hooked[b]) for b in range(store.cfg.batch))
    assert e_strict < strict, (e_strict, flips)
    if flips == 0:
        assert e_plain < plain, e_plain
    return e_plain, e_strict, flips
