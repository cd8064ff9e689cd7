"""Batch 8 / 16 (config E lists batch 16): every projection on tensor cores,
streamed in K chunks (decode_kernel.cuh: Shape::KCP, gemv_kc), the FFN in two
phases, the weights as fp16 (the bf16 values; exact in the fp16 normal
range) and the activations as fp16 hi/lo MMA A-fragment tables.  Same bars as the
batch 1-4 parity suite (tests/test_gpu_parity.py): with the device's K/V rows
fed to the oracle rel_err < 2e-5, without that hook the reference's 1e-4
whenever no bf16 rounding flip occurred; all run modes bit-identical."""
import numpy as np
import pytest

import oracle as O
from gpu_helpers import check_step, device_from_store, to_model_cfg
from paper_2505_22758_b200 import DecodeModel, RunMode

pytestmark = pytest.mark.gpu

MODES = [RunMode.BASELINE, RunMode.FUSED, RunMode.FUSED_OVERLAP]
TOY = O.preset("llama31_8b-toy")
TOKENS = [17, 3, 99, 400, 11, 250, 7, 501, 42, 1, 333, 64, 128, 5, 77, 260]


@pytest.mark.parametrize("batch,prefill", [(16, 0), (16, 40), (16, 300), (8, 40)])
def test_toy_batch_rows_match_oracle(batch, prefill):
    st = O.OracleStore(TOY.replace(batch=batch), 21, prefill + 4)
    st.synthetic_prefill(prefill, 3)
    with device_from_store(st) as m:
        e_plain, e_strict, flips = check_step(st, m, TOKENS[:batch], prefill)
    print(f"toy b{batch} prefill {prefill}: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")


@pytest.mark.parametrize("dims", [(512, 2048, 64, 8, 2), (2048, 2048, 64, 32, 8)])
def test_small_512_column_chunks_match_oracle(dims):
    """The 8B geometry (512-column K chunks, 4 k parts per weight slot) at
    small width; (2048, .., 8 kv heads) also runs one CTA per (row, kv head)
    in the attention (128 units, split-K group 1)."""
    d, di, dh, nq, nkv = dims
    cfg = O.ModelCfg(2, d, di, dh, nq, nkv, 1024).replace(batch=16)
    st = O.OracleStore(cfg, 3, 70)
    st.synthetic_prefill(64, 1)
    with device_from_store(st) as m:
        e_plain, e_strict, flips = check_step(st, m, TOKENS, 64)
    print(f"{dims} b16: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")


def test_toy_batch16_modes_bit_identical_multi_step():
    outs = []
    for mode in MODES:
        st = O.OracleStore(TOY.replace(batch=16), 9, 110)
        st.synthetic_prefill(100, 5)
        with device_from_store(st, mode=mode) as m:
            steps = []
            for i in range(4):
                lg, greedy = m.step(TOKENS, 100 + i)
                assert np.array_equal(greedy, np.argmax(lg, axis=1))
                steps.append(lg)
            outs.append(np.stack(steps))
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[1], outs[2])


def test_8b_width_batch16_single_step_matches_oracle():
    """E width (d_model 4096, 32 / 8 heads, d_inter 14336), one layer,
    reduced vocabulary, 512-position context."""
    cfg = O.preset("llama31_8b").replace(layers=1, vocab_size=4096, batch=16)
    st = O.OracleStore(cfg, 1234, 514)
    st.synthetic_prefill(512, 7)
    with device_from_store(st) as m:
        e_plain, e_strict, flips = check_step(st, m, TOKENS, 512)
    print(f"8B width b16: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, flips {flips}")


def test_full_size_8b_batch16_greedy_and_modes():
    cfg = to_model_cfg(O.preset("llama31_8b")).replace(batch=16)
    m = DecodeModel(cfg, 1028)
    m.init_synthetic(7)
    for l in range(cfg.layers):
        m.set_length(l, 1024)
    m.calibrate(1)  # per-SM plan weights also drive the batch >= 8 row split
    outs = []
    for mode in MODES:
        m.set_mode(mode)
        for l in range(cfg.layers):
            m.set_length(l, 1024)
        lg, greedy = m.step(TOKENS, 1024)
        assert np.array_equal(greedy, np.argmax(lg, axis=1))
        assert np.isfinite(lg).all()
        outs.append(lg)
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[1], outs[2])
    m.close()


def test_toy_batch16_device_decode_loop_matches_stepwise():
    """ffb_decode_loop at batch 16: teacher-forced prompt rows then greedy
    generation on the device give the host-driven step loop's tokens."""
    cfg = TOY.replace(batch=16, layers=2)
    prompt = np.array([[(7 * i + 3 * b) % cfg.vocab_size for b in range(16)] for i in range(6)],
                      np.int64)
    n = 5
    st = O.OracleStore(cfg, 42, 20)
    with device_from_store(st, 20) as m:
        gen = m.generate(None, 0, n, prompt=prompt)
    st2 = O.OracleStore(cfg, 42, 20)
    with device_from_store(st2, 20) as m2:
        for pos in range(len(prompt)):
            _, g = m2.step(list(prompt[pos]), pos, logits=False)
        ref = [np.array(g)]
        for i in range(1, n):
            _, g = m2.step(list(ref[-1]), len(prompt) + i - 1, logits=False)
            ref.append(np.array(g))
    np.testing.assert_array_equal(gen, np.stack(ref))


def test_toy_batch16_zero_layers_is_lm_head_of_embedding():
    """layers = 0: the A table of the LM head comes straight from the kernel's
    embedding init (init counter, no decoder stage in between)."""
    cfg = TOY.replace(batch=16, layers=0)
    st = O.OracleStore(cfg, 5, 4)
    with device_from_store(st, 4) as m:
        e_plain, e_strict, flips = check_step(st, m, TOKENS, 0)
    assert flips == 0


def test_gemv_layout_is_the_loaded_librarys():
    """kc_layout reports which batch >= 8 GEMV this library runs: 2 =
    mma.sync (libffb200.so), 3 = tcgen05 with TMEM accumulators
    (libffb200_tc05.so, tests/test_gpu_tcgen05.py runs this file on it)."""
    import os
    cfg = to_model_cfg(TOY).replace(batch=16)
    m = DecodeModel(cfg, 8)
    want = int(os.environ.get("FFB_EXPECT_KC_LAYOUT", "2"))
    assert m.info()["kc_layout"] == want
    m.close()


def test_fp16_range_weights_rejected_and_counted():
    """Batch >= 8 stores the bf16 weights as fp16 (the tensor-core operand):
    values beyond ±65504 are rejected at upload (no silent inf), values
    below the fp16 normal range are stored rounded and counted
    (ffb_info.fp16_inexact)."""
    from paper_2505_22758_b200 import UnsupportedConfigError
    cfg = to_model_cfg(TOY).replace(batch=16)
    st = O.OracleStore(TOY.replace(batch=16), 3, 8)
    m = DecodeModel(cfg, 8)
    w = np.array(st.tensor("layer.0.wqkv"), np.float32)
    m.upload_tensor("layer.0.wqkv", w)
    base = m.info()["fp16_inexact"]
    w2 = w.copy().ravel()
    w2[:3] = [1e-6, -3e-7, 2.5e-6]   # below 2^-14 and not multiples of 2^-24 after bf16 rounding
    m.upload_tensor("layer.0.wqkv", w2)
    assert m.info()["fp16_inexact"] >= base + 3
    w2[5] = 1.0e5
    with pytest.raises(UnsupportedConfigError):
        m.upload_tensor("layer.0.wqkv", w2)
    m.close()


def test_fp16_range_activation_overflow_is_reported():
    """An activation beyond the fp16 range of the batch >= 8 A tables (here:
    a huge embedding row) latches the device error flag; the step reports
    it instead of returning inf / NaN logits silently."""
    from paper_2505_22758_b200 import FusesimError
    st = O.OracleStore(TOY.replace(batch=16), 21, 8)
    with device_from_store(st) as m:
        emb = np.array(st.tensor("embedding"), np.float32)
        emb[17] = 3.0e5
        m.upload_tensor("embedding", emb)
        with pytest.raises(FusesimError, match="fp16 range"):
            m.step(TOKENS, 0)
        for l in range(TOY.layers):  # (that step appended its K/V rows)
            m.set_length(l, 0)
        logits, _ = m.step([1] * 16, 0)  # the latch was cleared: a clean step runs
        assert np.isfinite(logits).all()
