"""GPU parity of the weight-only int4 / int8 decode kernels (BASELINE config
Q): fused in-kernel dequantization of every streamed
matrix against the CPU oracle on the same snapped weights.

The packer re-derives the reference's grid exactly (tests/test_quant.py), so
the device multiplies the very f32 weights the oracle uses: the same
tolerances as the bf16 kernel apply (check_step: 2e-5 with the device's K/V
rows, 1e-4 -- test_interpreter.cpp:66 -- without).  int4 is pinned to the
reference itself (tests/golden/toy_int4_logits.npy); int8 is the 255-level
extension restated by the oracle."""
import os

import numpy as np
import pytest

import oracle as O
from gpu_helpers import GOLDEN, check_step, device_from_store, rel_err, to_model_cfg
from paper_2505_22758_b200 import DecodeModel, RunMode

pytestmark = pytest.mark.gpu

MODES = [RunMode.BASELINE, RunMode.FUSED, RunMode.FUSED_OVERLAP]
TOY = O.preset("llama31_8b-toy")


@pytest.mark.parametrize("qb", [4, 8])
@pytest.mark.parametrize("prefill", [0, 1, 255, 300])
def test_quant_toy_matches_oracle(qb, prefill):
    for mode in MODES:
        st = O.OracleStore(TOY.replace(quant_bits=qb), 42, prefill + 4)
        st.synthetic_prefill(prefill, 7)
        with device_from_store(st, mode=mode) as m:
            assert m.info()["quant_inexact_groups"] == 0
            e_plain, e_strict, flips = check_step(st, m, [17], prefill)
            print(f"int{qb} prefill {prefill} {mode.name}: rel_err {e_plain:.2e} "
                  f"same-KV {e_strict:.2e} flips {flips}")


def test_int4_toy_vs_reference_golden():
    """The reference's own int4 logits (fusesim reference_forward on its
    snapped store, tests/golden/gen_golden.py) at prefill 33."""
    st = O.OracleStore(TOY.replace(quant_bits=4), 42, 40)
    st.synthetic_prefill(33, 7)
    golden = np.load(os.path.join(GOLDEN, "toy_int4_logits.npy"))
    with device_from_store(st) as m:
        got = m.forward([17], 33)[0]
    assert rel_err(got, golden) < 1e-4
    assert int(np.argmax(got)) == int(np.argmax(golden))


def test_quant_batched_rows_and_mode_identity():
    cfg = TOY.replace(quant_bits=4, batch=4)
    outs = []
    for mode in MODES:
        st = O.OracleStore(cfg, 9, 44)
        st.synthetic_prefill(40, 5)
        with device_from_store(st, mode=mode) as m:
            check_step(st, m, [11, 400, 7, 99], 40)
            for l in range(cfg.layers):
                m.set_length(l, 40)
            outs.append(m.forward([11, 400, 7, 99], 40))
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[1], outs[2])


@pytest.mark.parametrize("qb", [4, 8])
def test_quant_full_width_8b_single_step(qb):
    """E width (d_model 4096, 32/8 heads, d_inter 14336), one layer, reduced
    vocab, 4k context: the Q-config kernels against the f64 oracle."""
    cfg = O.preset("llama31_8b").replace(layers=1, vocab_size=4096, quant_bits=qb)
    st = O.OracleStore(cfg, 1234, 4098)
    st.synthetic_prefill(4096, 7)
    with device_from_store(st) as m:
        assert m.info()["quant_inexact_groups"] == 0
        e_plain, e_strict, flips = check_step(st, m, [17], 4096)
    print(f"8B int{qb}: rel_err {e_plain:.2e} same-KV {e_strict:.2e} flips {flips}")


@pytest.mark.parametrize("qb", [4, 8])
def test_quant_full_size_8b_greedy_and_determinism(qb):
    cfg = to_model_cfg(O.preset("llama31_8b")).replace(quant_bits=qb)
    m = DecodeModel(cfg, 4100)
    m.init_synthetic(7)
    outs = []
    for mode in MODES:
        m.set_mode(mode)
        for l in range(cfg.layers):
            m.set_length(l, 4096)
        lg, greedy = m.step([17], 4096)
        assert np.isfinite(lg).all()
        assert int(greedy[0]) == int(np.argmax(lg[0]))
        outs.append(lg)
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[1], outs[2])
    m.close()
