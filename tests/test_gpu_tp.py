"""GPU parity of the tensor-parallel shards, run as a TP
group co-located on ONE B200 (each rank a persistent kernel on half of the
SMs, the cross-rank sums over the same device's memory -- the code path a
multi-GPU group runs over NVLink P2P): the gathered logits and the global
greedy token against the dense f64 oracle of the whole model."""
import numpy as np
import pytest

import oracle as O
from gpu_helpers import rel_err, to_model_cfg
from paper_2505_22758_b200 import RunMode, TPGroup

pytestmark = pytest.mark.gpu

MODES = [RunMode.BASELINE, RunMode.FUSED, RunMode.FUSED_OVERLAP]


def _group(st, tp, mode=RunMode.FUSED_OVERLAP):
    g = TPGroup(to_model_cfg(st.cfg), st.max_seq_len, tp, mode=mode)
    g.upload_store(st)
    k, v = st.kv()
    g.kv_import(k, v, st.length(0))
    return g


@pytest.mark.parametrize("prefill", [0, 1, 40, 300])
def test_tiny_tp2_matches_oracle(prefill):
    cfg = O.preset("tiny").replace(layers=2)
    for mode in MODES:
        st = O.OracleStore(cfg, 42, prefill + 4)
        st.synthetic_prefill(prefill, 7)
        with _group(st, 2, mode) as g:
            logits, greedy = g.step([17], prefill)
            assert g.length(0) == prefill + 1
        want = st.forward([17], prefill)[0]
        e = rel_err(logits[0], want)
        print(f"tiny TP2 prefill {prefill} {mode.name}: rel_err {e:.2e}")
        assert e < 1e-4
        assert int(greedy[0]) == int(np.argmax(want))


def test_tiny_tp2_greedy_decode_and_mode_identity():
    """A short greedy decode: every rank agrees on the token (checked inside
    TPGroup.step) and it equals the oracle's argmax at every step; the three
    run modes give bit-identical logits."""
    cfg = O.preset("tiny").replace(layers=2)
    st = O.OracleStore(cfg, 5, 64)
    st.synthetic_prefill(20, 3)
    with _group(st, 2) as g:
        tok = 17
        for pos in range(20, 28):
            logits, greedy = g.step([tok], pos)
            want = st.forward([tok], pos)[0]
            assert rel_err(logits[0], want) < 1e-3
            assert int(greedy[0]) == int(np.argmax(want))
            tok = int(greedy[0])
    outs = []
    for mode in MODES:
        st2 = O.OracleStore(cfg, 5, 64)
        st2.synthetic_prefill(20, 3)
        with _group(st2, 2, mode) as g:
            outs.append(g.step([17], 20)[0])
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[1], outs[2])


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_8b_width_tp_shards_single_step(tp):
    """Llama-3.1-8B width (32 q / 8 kv heads, d_inter 14336) as TP 2 / 4 / 8
    shards (kernels_tp.cu: the shapes bench.py --gpus N runs), two layers,
    reduced vocabulary, 1k context, co-located on one GPU."""
    cfg = O.preset("llama31_8b").replace(layers=2, vocab_size=4096)
    st = O.OracleStore(cfg, 1234, 1026)
    st.synthetic_prefill(1024, 7)
    with _group(st, tp) as g:
        logits, greedy = g.step([17], 1024)
    want = st.forward([17], 1024)[0]
    e = rel_err(logits[0], want)
    print(f"8B width TP{tp}: rel_err {e:.2e}")
    assert e < 1e-4
    assert int(greedy[0]) == int(np.argmax(want))


@pytest.mark.parametrize("tp", [1, 2, 4, 8])
def test_70b_width_shards_match_oracle(tp):
    """Llama-3-70B width (d_model 8192, 64 q / 8 kv heads, d_inter 28672):
    the TP 1/2/4/8 shard kernels (kernels_70b.cu) of one layer, reduced
    vocabulary, 256-position context, co-located on one GPU (148 / TP SMs
    per rank), against the f64 oracle of the whole layer."""
    cfg = O.preset("llama31_70b").replace(layers=1, vocab_size=4096)
    st = O.OracleStore(cfg, 1234, 258)
    st.synthetic_prefill(256, 7)
    want = None
    with _group(st, tp) as g:
        logits, greedy = g.step([17], 256)
    for l in range(cfg.layers):
        st.set_length(l, 256)
    want = st.forward([17], 256)[0]
    e = rel_err(logits[0], want)
    print(f"70B width TP{tp}: rel_err {e:.2e}")
    assert e < 1e-4
    assert int(greedy[0]) == int(np.argmax(want))
