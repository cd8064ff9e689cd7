"""GPU greedy tie rule: the kernel's argmax picks the LOWEST vocabulary index
among exactly equal logits, as the reference's argmax_token does
(/root/reference/proj/include/fusesim/numerics.hpp:168-175, strict `>` scan
from index 0) -- across the rows of one CTA, across CTAs of the LM-head
stage, and across the vocabulary slices of tensor-parallel ranks.

Exact device ties need logits whose value does not depend on the summation
order, so the tied LM-head rows are scaled one-hot rows C * e_k (C a power
of two): every row's dot product is one nonzero product plus exact zeros,
bit-identical wherever the row is computed.  k and the sign are picked so the
tied logit is the largest of every batch row by a wide margin (checked on the
f64 oracle)."""
import numpy as np
import pytest

import oracle as O
from gpu_helpers import device_from_store, rel_err
from test_gpu_tp import _group

pytestmark = pytest.mark.gpu

C_SCALE = 1024.0


def _tied_store(preset: str, batch: int, tie_rows, **over):
    cfg = O.preset(preset).replace(batch=batch, **over)
    tokens = [17 + 3 * b for b in range(batch)]

    def fresh():
        st = O.OracleStore(cfg, 42, 48)
        st.synthetic_prefill(33, 7)
        return st

    # probe: LM-head row j = e_j gives logit[b][j] = normed h_b[j] * final_norm[j]
    st = fresh()
    lm = st.lm_head
    d = cfg.d_model
    lm[:d] = np.eye(d, dtype=np.float32)
    probe = st.forward(tokens, 33)[:, :d]  # [B][d]
    st.close()
    same_sign = np.all(probe > 0, axis=0) | np.all(probe < 0, axis=0)
    score = np.where(same_sign, np.abs(probe).min(axis=0), 0.0)
    k = int(np.argmax(score))
    assert score[k] > 0, "no column with one sign over the batch"
    sign = 1.0 if probe[0, k] > 0 else -1.0

    st = fresh()
    lm = st.lm_head
    for r in tie_rows:
        lm[r] = 0.0
        lm[r, k] = sign * C_SCALE
    want = st.forward(tokens, 33)
    for b in range(batch):
        top = want[b, tie_rows[0]]
        assert all(want[b, r] == top for r in tie_rows)
        others = np.delete(want[b], tie_rows)
        assert top > others.max() + 1.0, "tied logit must be the clear maximum"
    st.close()
    st = fresh()
    lm = st.lm_head
    for r in tie_rows:
        lm[r] = 0.0
        lm[r, k] = sign * C_SCALE
    return st, tokens, want


@pytest.mark.parametrize("preset,batch", [("tiny", 1), ("llama31_8b-toy", 1), ("llama31_8b-toy", 4)])
def test_greedy_lowest_index_among_exact_ties(preset, batch):
    v = O.preset(preset).vocab_size
    ties = [5, v // 2 + 3, v - 1]  # different CTAs of the LM-head stage
    st, tokens, want = _tied_store(preset, batch, ties)
    with device_from_store(st) as m:
        logits, greedy = m.step(tokens, 33)
    for b in range(batch):
        vals = logits[b, ties]
        assert np.all(vals == vals[0]), f"row {b}: tied logits differ on the device: {vals}"
        assert int(greedy[b]) == 5 == int(np.argmax(want[b])), (b, int(greedy[b]))
        assert rel_err(logits[b], want[b]) < 1e-3


def test_greedy_tie_order_independent_of_cta_order():
    """The tie winner is the lowest index even when it is in the last CTA's
    rows and a higher-indexed copy sits in the first CTA's."""
    v = O.preset("llama31_8b-toy").vocab_size
    ties = [v - 2, v - 1]
    st, tokens, want = _tied_store("llama31_8b-toy", 1, ties)
    with device_from_store(st) as m:
        _, greedy = m.step(tokens, 33)
    assert int(greedy[0]) == v - 2 == int(np.argmax(want[0]))


@pytest.mark.parametrize("preset,over,tp", [("tiny", {"layers": 2}, 2),
                                            ("llama31_8b", {"layers": 1, "vocab_size": 4096}, 4)])
def test_tp_greedy_tie_across_rank_slices(preset, over, tp):
    """Exact ties straddling the vocabulary slices of TP ranks (the in-kernel
    argmax exchange), ranks co-located on one GPU: the lowest global index
    wins on every rank (TPGroup.step checks the ranks agree)."""
    v = over.get("vocab_size", O.preset(preset).vocab_size)
    vl = v // tp
    ties = [vl - 1, vl, v - 1]  # last row of rank 0, first of rank 1, last of the last rank
    st, tokens, want = _tied_store(preset, 1, ties, **over)
    with _group(st, tp) as g:
        logits, greedy = g.step(tokens, 33)
    vals = logits[0, ties]
    assert np.all(vals == vals[0]), vals
    assert int(greedy[0]) == vl - 1 == int(np.argmax(want[0]))
