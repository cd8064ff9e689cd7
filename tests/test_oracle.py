"""CPU tests pinning the oracle (oracle/fusesim_oracle.c) to the reference.

* against the golden fixtures in tests/golden/ (produced from the unmodified
  reference by tests/golden/gen_golden.py) -- runs everywhere;
* against oracle/_ref (the reference headers compiled unchanged) when that
  library is present -- bit-exact weights, caches and logits;
* the reference's own unit cases, restated (proj/tests/test_numerics.cpp,
  proj/tests/test_store.cpp, test_partition.cpp:21-32 byte counts).
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(GOLDEN, "golden.json")))
TOY = O.preset("llama31_8b-toy")


def fnv(a):
    a = np.ascontiguousarray(a)
    return "%016x" % O.lib().fo_fnv1a(a.ctypes.data, a.nbytes, 0xcbf29ce484222325)


def dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ------------------------------------------------------------------ golden
def test_weights_match_reference_checksums():
    st = O.OracleStore(TOY, 42, 8)
    for name, want in META["toy_weight_fnv"].items():
        assert fnv(st.tensor(name)) == want, name
    T = O.preset("tiny")
    st = O.OracleStore(T, 1234, 8)
    for name, want in META["tiny_weight_fnv"].items():
        assert fnv(st.tensor(name)) == want, name


def test_int4_weights_match_reference_checksums():
    st = O.OracleStore(TOY.replace(quant_bits=4), 42, 40)
    for name, want in META["toy_int4_weight_fnv"].items():
        assert fnv(st.tensor(name)) == want, name


@pytest.mark.parametrize("prefill", [0, 1, 255, 256, 300])
def test_oracle_logits_bit_exact_vs_golden(prefill):
    g = np.load(os.path.join(GOLDEN, "toy_logits.npz"))
    st = O.OracleStore(TOY, 42, prefill + 4)
    st.synthetic_prefill(prefill, 7)
    got = st.forward([17], prefill)[0]
    np.testing.assert_array_equal(got, g[f"oracle_{prefill}"])
    # the reference's interpreter agrees with its oracle at the 1e-4 bound
    interp = g[f"interp_{prefill}"]
    assert np.abs(interp - got).max() / np.abs(got).max() < 1e-4
    K, V = st.kv()
    np.testing.assert_array_equal(np.concatenate([K[0, 0, 0, prefill], V[0, 0, 0, prefill]]),
                                  g[f"kv_{prefill}"])
    assert st.length(0) == prefill + 1


def test_int4_oracle_logits_bit_exact_vs_golden():
    st = O.OracleStore(TOY.replace(quant_bits=4), 42, 40)
    st.synthetic_prefill(33, 7)
    np.testing.assert_array_equal(st.forward([17], 33)[0],
                                  np.load(os.path.join(GOLDEN, "toy_int4_logits.npy")))


def test_tiny_prompt_and_first_steps_vs_golden():
    g = np.load(os.path.join(GOLDEN, "tiny_decode.npz"))
    assert O.tiny_prompt(8) == META["tiny_prompt_head"]
    T = O.preset("tiny")
    st = O.OracleStore(T, 1234, 8)
    for i in range(3):
        lg = st.forward([int(g["fed"][i])], i)[0]
        assert int(np.argmax(lg)) == int(g["argmax"][i])
        if i == 0:
            np.testing.assert_array_equal(lg, g["logits_0"])


def test_byte_accounting_matches_reference():
    """test_store.cpp:73-86 and tensor_store.hpp:170-192."""
    for name, want in META["streamed_weight_bytes"].items():
        cfg = O.preset("llama31_8b").replace(quant_bits=4) if name.endswith("int4") \
            else O.preset(name)
        assert O.lib().fo_streamed_weight_bytes(cfg.c()) == want
    assert META["streamed_weight_bytes"]["llama31_8b"] == 32 * 436207616 + 1050673152


# ------------------------------------------------------------------ vs _ref
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("quant", [0, 4])
def test_restatement_bit_exact_vs_reference(quant):
    cfg = TOY.replace(batch=2, quant_bits=quant)
    o = O.OracleStore(cfg, 3, 40)
    r = O.RefStore(cfg, 3, 40)
    for l in range(cfg.layers):
        for t in ("wqkv", "waout", "wffn1", "wffn2t", "norm_attn", "norm_ffn"):
            n = f"layer.{l}.{t}"
            np.testing.assert_array_equal(o.tensor(n).ravel(), r.tensor(n))
    for n in ("embedding", "lm_head", "final_norm"):
        np.testing.assert_array_equal(o.tensor(n).ravel(), r.tensor(n))
    o.synthetic_prefill(21, 11)
    r.synthetic_prefill(21, 11)
    for pos in (21, 22):
        np.testing.assert_array_equal(o.forward([5, 300], pos), r.forward([5, 300], pos))


@needs_ref
def test_reference_validation_errors_restated():
    o = O.OracleStore(TOY, 3, 4)
    with pytest.raises(ValueError, match="out of range"):
        o.forward([512], 0)
    with pytest.raises(ValueError, match="does not match"):
        o.forward([1], 2)
    r = O.RefStore(TOY, 3, 4)
    with pytest.raises(ValueError, match="out of range"):
        r.forward([512], 0)
    with pytest.raises(ValueError, match="does not match"):
        r.forward([1], 2)


# ------------------------------------------------------------------ numerics
L = O.lib()


def rmsnorm(x, w, eps):
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    y = np.empty_like(x)
    L.fo_rmsnorm_f64(dp(x), dp(w), x.size, eps, dp(y))
    return y


def test_rmsnorm_unit_cases():
    """test_numerics.cpp:49-57."""
    y = rmsnorm([1, 1, 1, 1], [1] * 4, 0.0)
    np.testing.assert_allclose(y, 1.0)
    y = rmsnorm([2, 0, 0, 0], [1] * 4, 0.0)
    assert y[0] == pytest.approx(2.0) and y[1] == 0.0


def test_rmsnorm_extended_precision():
    """test_numerics.cpp:59-75 (long double recomputation, 1e-12)."""
    rng = np.random.default_rng(5)
    x, w = rng.standard_normal(257), rng.standard_normal(257)
    y = rmsnorm(x, w, 1e-5)
    xl, wl = x.astype(np.longdouble), w.astype(np.longdouble)
    inv = 1 / np.sqrt((xl * xl).sum() / 257 + np.longdouble(1e-5))
    np.testing.assert_allclose(y, (wl * xl * inv).astype(np.float64), rtol=1e-12, atol=1e-12)


def test_rope_basics():
    """test_numerics.cpp:77-100: identity at pos 0, norm preserved, closed form."""
    v = np.array([0.3, -1.2, 0.7, 2.2])
    a = v.copy()
    L.fo_rope_f64(dp(a), 4, 0, 500000.0)
    np.testing.assert_array_equal(a, v)
    a = v.copy()
    L.fo_rope_f64(dp(a), 4, 37, 500000.0)
    assert np.linalg.norm(a) == pytest.approx(np.linalg.norm(v), rel=1e-12)
    a = np.array([1.0, 0.0])
    L.fo_rope_f64(dp(a), 2, 1, 500000.0)
    np.testing.assert_allclose(a, [np.cos(1.0), np.sin(1.0)], rtol=1e-12)


def partial(q, K, V, state=None, alpha=1.0):
    d = q.size
    m = C.c_double(-np.inf if state is None else state[0])
    l = C.c_double(0.0 if state is None else state[1])
    o = np.zeros(d) if state is None else state[2].copy()
    K = np.ascontiguousarray(K, np.float64)
    V = np.ascontiguousarray(V, np.float64)
    L.fo_attn_partial_update(C.byref(m), C.byref(l), dp(o), d, dp(np.ascontiguousarray(q)),
                             dp(K), dp(V), K.shape[0], alpha)
    return m.value, l.value, o


def reduce(parts):
    d = parts[0][2].size
    m = np.array([p[0] for p in parts])
    l = np.array([p[1] for p in parts])
    o = np.ascontiguousarray(np.stack([p[2] for p in parts]))
    out = np.empty(d)
    rc = L.fo_attn_reduce(dp(m), dp(l), dp(o), len(parts), d, dp(out))
    return rc, out


def test_reduction_known_answers():
    """test_numerics.cpp:143-175."""
    rc, out = reduce([(0.0, 1.0, np.array([2.0])), (0.0, 3.0, np.array([6.0]))])
    assert rc == 0 and out[0] == pytest.approx(2.0)
    rc, out = reduce([(np.log(2.0), 1.0, np.array([2.0])), (0.0, 2.0, np.array([2.0]))])
    assert out[0] == pytest.approx(1.5)
    rc, _ = reduce([(-np.inf, 0.0, np.array([0.0]))])
    assert rc == 2


def test_partitioned_attention_equals_monolithic():
    """test_numerics.cpp:177-208: 50 randomized trials, < 1e-12 vs long double."""
    rng = np.random.default_rng(123)
    for _ in range(50):
        n, d = int(rng.integers(1, 300)), int(rng.integers(1, 64))
        q = rng.standard_normal(d)
        K = rng.standard_normal((n, d))
        V = rng.standard_normal((n, d))
        alpha = 1 / np.sqrt(d)
        cuts = np.sort(rng.integers(0, n + 1, size=int(rng.integers(1, 8))))
        bounds = [0] + list(cuts) + [n]
        parts = [partial(q, K[a:b], V[a:b], alpha=alpha) for a, b in zip(bounds, bounds[1:])]
        rc, out = reduce(parts)
        s = (K.astype(np.longdouble) @ q.astype(np.longdouble)) * np.longdouble(alpha)
        w = np.exp(s - s.max())
        want = (w / w.sum()) @ V.astype(np.longdouble)
        scale = max(1.0, float(np.abs(want).max()))
        assert np.abs(out - want.astype(np.float64)).max() / scale < 1e-12


def test_swiglu_limits_and_argmax_ties():
    """test_numerics.cpp:239-249, 297-301."""
    assert L.fo_silu(0.0) == 0.0
    assert L.fo_silu(40.0) == pytest.approx(40.0)
    assert abs(L.fo_silu(-40.0)) < 1e-15
    v = np.array([1.0, 3.0, 3.0, 2.0])
    assert L.fo_argmax_f64(dp(v), 4) == 1


def test_quant_formula_grid_and_roundtrip():
    """test_store.cpp:10-48."""
    assert L.fo_dequantize_code(8, 0.5, 8.0) == 0.0
    assert L.fo_dequantize_code(3, 0.5, 8.0) == -2.5
    for scale in (0.03125, 0.5, 1.3):
        for zero in (0.0, 4.0, 8.0, 15.0):
            for c in range(16):
                v = np.float32((np.float32(c) - np.float32(zero)) * np.float32(scale))
                assert L.fo_quantize_value(float(v), scale, zero, 15) == c
    rng = np.random.default_rng(99)
    vals = rng.standard_normal(128).astype(np.float32)
    codes = np.zeros(128, np.uint8)
    s, z = C.c_float(), C.c_float()
    deq = np.zeros(128, np.float32)
    L.fo_quantize_group(vals.ctypes.data_as(C.POINTER(C.c_float)), 128, 15,
                        codes.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(s), C.byref(z),
                        deq.ctypes.data_as(C.POINTER(C.c_float)))
    again = [L.fo_quantize_value(float(v), s.value, z.value, 15) for v in deq]
    assert list(codes) == again


def test_same_seed_same_store():
    """test_store.cpp:62-71."""
    a = O.OracleStore(TOY, 7, 64)
    b = O.OracleStore(TOY, 7, 64)
    c = O.OracleStore(TOY, 8, 64)
    np.testing.assert_array_equal(a.layer(2)["wqkv"], b.layer(2)["wqkv"])
    np.testing.assert_array_equal(a.lm_head, b.lm_head)
    assert not np.array_equal(a.layer(0)["wqkv"], c.layer(0)["wqkv"])


def test_capacity_error():
    """test_store.cpp:109-118."""
    st = O.OracleStore(TOY, 3, 2)
    st.forward([1], 0)
    st.forward([1], 1)
    with pytest.raises(ValueError, match="capacity"):
        st.forward([1], 2)


def test_stacked_linear_oracle_bit_exact_vs_reference():
    """Stacked-linear kind: the restated linear.<l>
    tensors and reference_linear_forward equal the reference's bit for bit."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    lo = O.LinearOracle(3, 256, 2, 1234)
    rl = O.RefLinear(3, 256, 2, 1234)
    for l in range(3):
        np.testing.assert_array_equal(lo.tensor(f"linear.{l}"), rl.tensor(f"linear.{l}"))
    x = np.random.default_rng(0).standard_normal((2, 256)).astype(np.float32)
    np.testing.assert_array_equal(lo.forward(x), rl.forward(x))


# ------------------------------------------------------------------ store file
@needs_ref
@pytest.mark.parametrize("quant", [0, 4])
def test_store_file_byte_identical_to_reference(tmp_path, quant):
    """'store dump/load round-trips' (proj/tests/test_store.cpp:120-131): the
    restatement's FSTW v1 file is byte-identical to the reference's
    save_store output, and each side loads the other's file."""
    cfg = TOY.replace(quant_bits=quant)
    o = O.OracleStore(cfg, 11, 32)
    r = O.RefStore(cfg, 11, 32)
    po, pr = tmp_path / "oracle.fstw", tmp_path / "ref.fstw"
    o.save(str(po))
    r.save(str(pr))
    assert po.read_bytes() == pr.read_bytes()
    back = O.OracleStore.load(str(pr), 32)
    assert back.cfg == cfg
    for n in ("layer.1.wffn1", "layer.3.norm_ffn", "final_norm", "embedding", "lm_head"):
        np.testing.assert_array_equal(back.tensor(n).ravel(), r.tensor(n))
    rb = O.RefStore.load(str(po), cfg, 32)
    np.testing.assert_array_equal(rb.tensor("layer.2.wqkv"), o.tensor("layer.2.wqkv").ravel())
    back.synthetic_prefill(5, 3)
    rb.synthetic_prefill(5, 3)
    np.testing.assert_array_equal(back.forward([9], 5), rb.forward([9], 5))


def test_store_file_roundtrip_and_errors(tmp_path):
    cfg = O.ModelCfg(2, 256, 512, 64, 4, 2, 300, batch=2)
    o = O.OracleStore(cfg, 5, 8)
    p = tmp_path / "s.fstw"
    o.save(str(p))
    back = O.OracleStore.load(str(p), 8)
    assert back.cfg == cfg
    for n in ("layer.0.wqkv", "layer.1.wffn2t", "layer.1.norm_attn", "embedding", "lm_head"):
        np.testing.assert_array_equal(back.tensor(n), o.tensor(n))
    raw = bytearray(p.read_bytes())
    bad = tmp_path / "bad.fstw"
    bad.write_bytes(b"\0" * 8 + bytes(raw[8:]))
    with pytest.raises(ValueError, match="bad magic"):
        O.OracleStore.load(str(bad), 8)
    raw2 = bytearray(raw)
    raw2[8] = 2
    bad.write_bytes(bytes(raw2))
    with pytest.raises(ValueError, match="bad version"):
        O.OracleStore.load(str(bad), 8)
    bad.write_bytes(bytes(raw[:len(raw) // 2]))
    with pytest.raises(ValueError, match="truncated|bad tensor"):
        O.OracleStore.load(str(bad), 8)
    with pytest.raises(ValueError, match="cannot open"):
        O.OracleStore.load(str(tmp_path / "missing.fstw"), 8)


def test_parallel_forward_is_bit_identical_across_thread_counts():
    """The OpenMP forward keeps every element's operation order: the same
    logits for 1 and many threads (and the reference pins the former)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import numpy as np, oracle as O;"
            "c = O.ModelCfg(2, 512, 1792, 64, 8, 2, 2000, batch=2);"
            "s = O.OracleStore(c, 4, 80); s.synthetic_prefill(70, 2);"
            "sys.stdout.buffer.write(s.forward([3, 99], 70).tobytes())"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    outs = []
    for n in ("1", "7"):
        env = dict(os.environ, OMP_NUM_THREADS=n)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, check=True,
                                   capture_output=True).stdout)
    assert len(outs[0]) == 2 * 2000 * 8 and outs[0] == outs[1]
