"""GPU parity of the GEMM prefill path (ffb_prefill, csrc/prefill.cu; SURVEY.md
§8(f) row 1) against the CPU oracle's decode-as-prefill (reference.hpp:60-61:
reference_forward once per prompt position).

The oracle ingests the prompt one position at a time; the device ingests all
positions of a chunk per layer at once.  Position by position they are
compared the way tests/gpu_helpers.check_step compares one decode step:
* the oracle, starting from the DEVICE's K/V history, computes its own K/V
  row for position t -- every element equals the device's row or differs by
  one bf16 rounding flip (kv_rows_match), layer by layer while no earlier
  layer flipped;
* the oracle cache is then rewound and position t appended with the device's
  rows, so the next position starts again from identical history;
* the last position's logits: rel_err < 2e-5 against the oracle run on the
  device's K/V (the arithmetic), < 1e-4 (the reference's own bound,
  test_interpreter.cpp:66) against the oracle's own rows when no flip
  occurred;
* decode then continues from the prefilled cache (check_step at pos0 + n).
"""
import numpy as np
import pytest

import oracle as O
from gpu_helpers import check_step, device_from_store, kv_rows_match, rel_err
from paper_2505_22758_b200 import (DecodeModel, ModelConfig, UnsupportedConfigError, UsageError,
                                   ValidationError)

pytestmark = pytest.mark.gpu


def _prompt(n, batch, vocab, seed):
    return np.random.default_rng(seed).integers(0, vocab, size=(n, batch), dtype=np.int64)


def _check_prefill(st, m, tokens, pos0, strict=2e-5, plain=1e-4):
    """Device prefill of tokens[n][B] at pos0 vs the oracle position by
    position (see module docstring).  Returns (plain, strict, flips)."""
    n = tokens.shape[0]
    L = st.cfg.layers
    got, greedy = m.prefill(tokens, pos0)
    for l in range(L):
        assert m.length(l) == pos0 + n
    k_dev, v_dev = m.kv_export(pos0, n)  # [B][L][Hkv][n][dh]
    flips = 0
    for t in range(n):
        pos = pos0 + t
        want = st.forward(tokens[t], pos)  # oracle's own rows, device history
        K, V = st.kv()
        kd, vd = k_dev[:, :, :, t], v_dev[:, :, :, t]
        fl = 0
        for l in range(L):
            if fl == 0:
                for dev, ora in ((kd, K[:, :, :, pos]), (vd, V[:, :, :, pos])):
                    assert kv_rows_match(dev[:, l], ora[:, l]), f"position {pos} layer {l}"
            fl += int((kd[:, l] != K[:, l, :, pos]).sum() + (vd[:, l] != V[:, l, :, pos]).sum())
        flips += fl
        for l in range(L):
            st.set_length(l, pos)
        want_hooked = st.forward(tokens[t], pos, k_app=kd, v_app=vd)
    e_strict = max(rel_err(got[b], want_hooked[b]) for b in range(st.cfg.batch))
    e_plain = max(rel_err(got[b], want[b]) for b in range(st.cfg.batch))
    assert e_strict < strict, (e_strict, flips)
    if fl == 0:
        assert e_plain < plain, e_plain
    for b in range(st.cfg.batch):
        assert int(greedy[b]) == int(np.argmax(got[b]))
    return e_plain, e_strict, flips


@pytest.mark.parametrize("batch,n", [(1, 1), (1, 37), (2, 33), (4, 9)])
def test_prefill_matches_oracle_then_decode_continues(batch, n):
    cfg = O.preset("llama31_8b-toy").replace(batch=batch)
    st = O.OracleStore(cfg, 42, n + 8)
    with device_from_store(st, n + 8) as m:
        toks = _prompt(n, batch, cfg.vocab_size, 5 + n)
        e_plain, e_strict, flips = _check_prefill(st, m, toks, 0)
        print(f"b{batch} n{n}: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")
        # the persistent decode kernel continues from the GEMM-built cache
        check_step(st, m, [3, 17, 99, 5][:batch], n)


def test_prefill_in_chunks_after_existing_context():
    """pos0 > 0: a prompt on top of an existing cache (synthetic context),
    fed as two calls -- the second chunk attends over everything before it."""
    cfg = O.preset("llama31_8b-toy").replace(batch=2)
    st = O.OracleStore(cfg, 7, 96)
    st.synthetic_prefill(40, 3)
    with device_from_store(st, 96) as m:
        toks = _prompt(30, 2, cfg.vocab_size, 11)
        _check_prefill(st, m, toks[:17], 40)
        _check_prefill(st, m, toks[17:], 57)
        check_step(st, m, [1, 2], 70)


@pytest.mark.parametrize("name,batch,ctx,n", [("llama32_1b", 1, 300, 64), ("llama31_8b", 1, 1000, 48),
                                              ("llama31_8b", 4, 0, 16)])
def test_prefill_full_width_matches_oracle(name, batch, ctx, n):
    """Real d_model / heads / d_inter (reduced depth and vocabulary so the f64
    oracle stays cheap); with and without prior context."""
    cfg = O.preset(name).replace(layers=2, vocab_size=4096, batch=batch)
    st = O.OracleStore(cfg, 1234, ctx + n + 2)
    if ctx:
        st.synthetic_prefill(ctx, 7)
    with device_from_store(st) as m:
        e_plain, e_strict, flips = _check_prefill(st, m, _prompt(n, batch, cfg.vocab_size, 9), ctx)
    print(f"{name} b{batch} ctx {ctx} n {n}: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")


@pytest.mark.parametrize("name,batch,ctx,n", [("llama31_8b-toy", 1, 0, 37), ("llama31_8b-toy", 2, 40, 20),
                                              ("llama31_8b", 1, 1000, 48)])
def test_prefill_two_term_split_within_reference_bound(name, batch, ctx, n):
    """Option prefill_terms = 2 (activations as bf16 hi + lo, ~2^-17
    relative): same checks, logits within the reference's own 1e-4 bound
    (test_interpreter.cpp:66) of the oracle run on the device's K/V."""
    cfg = O.preset(name).replace(batch=batch)
    if name == "llama31_8b":
        cfg = cfg.replace(layers=2, vocab_size=4096)
    st = O.OracleStore(cfg, 1234, ctx + n + 2)
    if ctx:
        st.synthetic_prefill(ctx, 7)
    with device_from_store(st) as m:
        m.set_option("prefill_terms", 2)
        e_plain, e_strict, flips = _check_prefill(st, m, _prompt(n, batch, cfg.vocab_size, 3), ctx,
                                                  strict=1e-4, plain=2e-4)
    print(f"2-term {name} b{batch} ctx {ctx} n {n}: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")


@pytest.mark.parametrize("qb,name,batch,ctx,n", [(4, "llama31_8b-toy", 1, 0, 29), (8, "llama31_8b-toy", 1, 30, 17), (4, "llama31_8b-toy", 4, 12, 9),
                                                 (4, "llama31_8b", 1, 500, 24), (8, "llama31_8b", 1, 0, 16)])
def test_prefill_quantized_weights_match_oracle(qb, name, batch, ctx, n):
    """int4 / int8 weights (quant.hpp:17-60): the packed rows are dequantised
    into three exact bf16 planes per projection (w = (code - zero) * scale,
    the reference's snapped weight bit for bit), so the same bounds hold as
    for bf16; the 8B width runs the tensor-core code order of the decode
    kernel's rows (Wqkv / Waout / Wffn1 / lm_head), the toy the plain one."""
    cfg = O.preset(name).replace(batch=batch, quant_bits=qb)
    if name == "llama31_8b":
        cfg = cfg.replace(layers=2, vocab_size=4096)
    st = O.OracleStore(cfg, 77, ctx + n + 2)
    if ctx:
        st.synthetic_prefill(ctx, 7)
    with device_from_store(st) as m:
        assert m.info()["quant_inexact_groups"] == 0
        e_plain, e_strict, flips = _check_prefill(st, m, _prompt(n, batch, cfg.vocab_size, 13), ctx)
        check_step(st, m, [5, 9, 11, 13][:batch], ctx + n)
    print(f"int{qb} {name} b{batch} ctx {ctx} n {n}: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")


@pytest.mark.parametrize("name,batch,ctx,n", [("llama31_8b-toy", 16, 0, 21), ("llama31_8b-toy", 16, 40, 9),
                                              ("llama31_8b", 8, 300, 12), ("llama31_8b", 16, 0, 8)])
def test_prefill_batch8_16_tensor_core_layout_matches_oracle(name, batch, ctx, n):
    """batch >= 8 models store the weights as fp16 in the K-chunked,
    swizzled tensor-core layout (layout 2, or 3 in the tcgen05 build): the
    prefill unpacks them per projection to bf16 (the original weights but
    for the smallest fp16 subnormals); the decode step that follows runs the
    batch-16 kernel (fp16 operands) on the prefilled cache, to the tcgen05
    suite's 3e-5 same-KV bound."""
    cfg = O.preset(name).replace(batch=batch)
    if name == "llama31_8b":
        cfg = cfg.replace(layers=2, vocab_size=4096)
    st = O.OracleStore(cfg, 5, ctx + n + 2)
    if ctx:
        st.synthetic_prefill(ctx, 7)
    with device_from_store(st) as m:
        e_plain, e_strict, flips = _check_prefill(st, m, _prompt(n, batch, cfg.vocab_size, 17), ctx, strict=3e-5,
                                                  plain=2e-4)
        check_step(st, m, list(range(3, 3 + batch)), ctx + n, strict=3e-5)
    print(f"b{batch} {name} ctx {ctx} n {n}: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")


def test_generate_with_prefill_matches_decode_loop_generation():
    """DecodeModel.generate(prompt=..., use_prefill=True): the prompt through
    ffb_prefill, then the device-resident decode loop -- the same tokens as
    the all-decode-loop generation on the tiny model."""
    cfg = O.preset("tiny").replace(layers=2)
    prompt = O.tiny_prompt(20, cfg.vocab_size)
    gens = []
    for use_prefill in (True, False):
        st = O.OracleStore(cfg, 42, 64)
        with device_from_store(st, 64) as m:
            gens.append([int(t) for t in m.generate(None, 0, 10, prompt=prompt, use_prefill=use_prefill)[:, 0]])
            assert m.length(0) == len(prompt) + 9
    assert gens[0] == gens[1], gens


def test_prefill_greedy_continuation_matches_decode_as_prefill():
    """Greedy generation after a GEMM prefill equals generation after the
    reference's decode-as-prefill (the persistent kernel stepping through the
    prompt), token for token, on the tiny model."""
    cfg = O.preset("tiny").replace(layers=2)
    prompt = O.tiny_prompt(24, cfg.vocab_size)
    out = []
    for use_prefill in (True, False):
        st = O.OracleStore(cfg, 42, 64)
        with device_from_store(st, 64) as m:
            if use_prefill:
                _, g = m.prefill(np.asarray(prompt).reshape(-1, 1), 0)
            else:
                for pos, t in enumerate(prompt):
                    _, g = m.step([t], pos, logits=False)
            gen = [int(g[0])]
            for i in range(12):
                _, g = m.step([gen[-1]], len(prompt) + i, logits=False)
                gen.append(int(g[0]))
        out.append(gen)
    assert out[0] == out[1], out


def test_prefill_full_size_8b_properties():
    """Full Llama-3.1-8B shape (32 layers, 128256 vocab), synthetic weights:
    a 512-token prompt in one call, then decoding continues; logits finite,
    greedy == argmax, the cache at 512, and a repeat is deterministic."""
    cfg = O.preset("llama31_8b")
    from gpu_helpers import to_model_cfg
    mc = to_model_cfg(cfg)
    m = DecodeModel(mc, 600)
    m.init_synthetic(7)
    toks = _prompt(512, 1, cfg.vocab_size, 1)
    lg1, g1 = m.prefill(toks, 0)
    assert np.isfinite(lg1).all() and int(g1[0]) == int(np.argmax(lg1[0]))
    assert m.length(0) == 512 and m.length(cfg.layers - 1) == 512
    lg2, g2 = m.step([int(g1[0])], 512)
    assert np.isfinite(lg2).all()
    for l in range(cfg.layers):
        m.set_length(l, 0)
    lg3, _ = m.prefill(toks, 0)
    np.testing.assert_array_equal(lg1, lg3)
    m.close()


def test_prefill_validation():
    cfg = O.preset("tiny").replace(layers=2)
    st = O.OracleStore(cfg, 42, 32)
    with device_from_store(st, 32) as m:
        with pytest.raises(ValidationError):  # position != cache length
            m.prefill([[1], [2]], 3)
        with pytest.raises(ValidationError):  # token id out of range
            m.prefill([[1], [cfg.vocab_size]], 0)
        with pytest.raises(ValidationError):  # beyond the KV capacity
            m.prefill(np.ones((40, 1), np.int64), 0)
        assert m.length(0) == 0  # nothing appended by a failed call
        m.prefill([[1], [2]], 0)
        assert m.length(0) == 2
        with pytest.raises(UsageError):
            m.set_option("prefill_terms", 1)
    lin = DecodeModel(ModelConfig(2, 2048, 0, 0, 0, 0, 0, kind=1), 8)  # stacked-linear kind: no prompt
    with pytest.raises(UnsupportedConfigError):
        lin.prefill([[1]], 0)
    lin.close()
