"""Full-depth parity of every north-star configuration (BASELINE.json configs
S, E, Q, H; SURVEY.md §8 tags) against the dense f64 oracle -- the
restatement pinned bit-exact to the reference's reference_forward
(tests/test_oracle.py) -- on the reference's own seeded weights
(init_weights(cfg, 1234), tensor_store.hpp:304-366) and KV history:

  * S  Llama-3.2-1B, 16 layers, full 128256 vocabulary, 1k context
  * E  Llama-3.1-8B, 32 layers, full vocabulary, 4k context, batch 1
  * E  the same weights at batch 16 (every projection on the tensor-core path)
  * Q  8B int4 (reference grid) and int8 (extension), 32 layers, full vocab
  * H  Llama-3-70B width, 2 layers, full vocabulary, TP 2 / 4 / 8 shards
       co-located on one GPU

Each run is ONE decode step from identical state (check_step: appended K/V
within one bf16 flip, logits within the stated tolerance with the device's K/V
rows fed to the oracle and within the reference's own 1e-4,
test_interpreter.cpp:66, when no bf16 flip occurred), then a decode stream:
teacher-forced prompt tokens followed by greedy generation, both sides fed
the same tokens, the oracle appending the device's K/V rows
(fo_reference_forward_ex) so the two caches stay identical.  Every step must
give identical greedy ids (the north star's "greedy token IDs identical over
the tested decode steps") and logits within the tolerance.  The smallest
top-1 / top-2 logit gap of the oracle over the stream is printed next to the
errors.

Tolerances (max-abs / max|logit|, the reference's metric, test_interpreter.
cpp:32-40), stated per arithmetic path:
  * 2e-5 -- bf16 weights on the CUDA-core GEMV (f32 FMA chains): measured
    5.6e-6 (8B, 32 layers, ctx 4096), growing ~linearly with depth;
  * 1e-4 -- the reference's own bound for its f32 interpreter against the
    f64 oracle -- for the tensor-core paths (int4 / int8 weights at batch 1,
    every projection at batch 16): activations enter the MMA as a two-term
    16-bit split and the MMA's f32 accumulation truncates, measured
    1.7e-5 (int8) / 3.9e-5 (int4, batch 16) at 32 layers, ctx 256.
"""
import numpy as np
import pytest

import oracle as O
from gpu_helpers import check_step, device_from_store, rel_err, to_model_cfg
from paper_2505_22758_b200 import RunMode, TPGroup

pytestmark = pytest.mark.gpu

STRICT = 2e-5      # bf16 CUDA-core path
STRICT_TC = 1e-4   # tensor-core paths (quant weights, batch >= 8)


def prompt_ids(n: int, batch: int, vocab: int, seed: int = 5) -> np.ndarray:
    """[n][batch] prompt ids from std::mt19937(seed) % vocab (the T config's
    recipe); batch rows are offset so they differ."""
    base = np.asarray(O.tiny_prompt(n * batch, vocab), np.int64).reshape(n, batch)
    return base


def fast_prefill(store, n: int, seed: int):
    """KV history for large batches: N(0, 0.3) rows rounded to bf16 (the
    distribution of synthetic_prefill, test_interpreter.cpp:16-30, drawn with
    numpy instead of one sequential mt19937_64 stream)."""
    k, v = store.kv()
    rng = np.random.default_rng(seed)
    for arr in (k, v):
        for b in range(arr.shape[0]):
            x = (rng.standard_normal(arr[b, :, :, :n].shape, dtype=np.float32) * 0.3)
            u = x.view(np.uint32).astype(np.uint64)
            u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16  # bf16 RNE (finite values)
            arr[b, :, :, :n] = u.astype(np.uint32).view(np.float32)
    for l in range(store.cfg.layers):
        store.set_length(l, n)


class _Dev:
    """One device handle or a co-located TP group behind the same calls."""

    def __init__(self, store, tp: int = 1):
        self.tp = tp
        if tp == 1:
            self.m = device_from_store(store)
            self.ranks = [self.m]
        else:
            self.m = TPGroup(to_model_cfg(store.cfg), store.max_seq_len, tp)
            self.m.upload_store(store)
            k, v = store.kv()
            self.m.kv_import(k, v, store.length(0))
            self.ranks = self.m.ranks

    def step(self, tokens, pos):
        return self.m.step(tokens, pos)

    def appended(self, pos):
        parts = [r.kv_export(pos, 1) for r in self.ranks]
        k = np.concatenate([p[0] for p in parts], axis=2)[:, :, :, 0]
        v = np.concatenate([p[1] for p in parts], axis=2)[:, :, :, 0]
        return k, v

    def close(self):
        self.m.close()


def decode_stream(store, dev: _Dev, pos: int, prompt: np.ndarray, n_gen: int, label: str,
                  tol: float = STRICT):
    """Teacher-forced prompt rows, then n_gen greedy steps; returns the ids."""
    B = store.cfg.batch
    worst, min_gap, ids = 0.0, np.inf, []
    tok = prompt[0]
    n_tf = prompt.shape[0]
    for i in range(n_tf + n_gen):
        logits, greedy = dev.step(tok, pos)
        k_dev, v_dev = dev.appended(pos)
        want = store.forward(tok, pos, k_app=k_dev, v_app=v_dev)
        for b in range(B):
            e = rel_err(logits[b], want[b])
            worst = max(worst, e)
            top2 = np.partition(want[b], -2)[-2:]
            min_gap = min(min_gap, float(top2[1] - top2[0]))
            assert e < tol, (label, i, b, e)
            assert int(greedy[b]) == int(np.argmax(want[b])), (label, i, b, int(greedy[b]),
                                                              int(np.argmax(want[b])))
        ids.append(np.asarray(greedy).copy())
        pos += 1
        tok = prompt[i + 1] if i + 1 < n_tf else np.asarray(greedy)
    print(f"{label}: {n_tf} teacher-forced + {n_gen} generated steps, greedy ids identical, "
          f"max rel_err {worst:.2e}, min oracle top-1/top-2 gap {min_gap:.3e}")
    return np.stack(ids)


def _single_and_stream(store, pos, n_tf, n_gen, label, tp=1, single=True, tol=STRICT):
    dev = _Dev(store, tp)
    try:
        if single:
            e_plain, e_strict, flips = check_step(store, dev.m,
                                                  list(range(17, 17 + store.cfg.batch)), pos,
                                                  strict=tol)
            print(f"{label} single step @ {pos}: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, "
                  f"bf16 flips {flips}")
            pos += 1
        pr = prompt_ids(n_tf, store.cfg.batch, store.cfg.vocab_size)
        return decode_stream(store, dev, pos, pr, n_gen, label, tol)
    finally:
        dev.close()


# ------------------------------------------------------------------ E (bf16)
@pytest.fixture(scope="module")
def store_8b():
    st = O.OracleStore(O.preset("llama31_8b"), 1234, 4096 + 40)
    yield st
    st.close()


def test_E_llama31_8b_b1_full_depth(store_8b):
    """Headline config: 32 layers, full vocabulary, 4096-position history."""
    st = store_8b
    st.synthetic_prefill(4096, 7)
    _single_and_stream(st, 4096, 16, 16, "E 8B bf16 b1 ctx 4096")


def test_E_llama31_8b_b16_full_depth(store_8b):
    """Batch 16 (tensor-core K-chunked projections), 32 layers, full
    vocabulary, 512-position history per row."""
    st = store_8b
    st.set_batch(16, 512 + 40)
    fast_prefill(st, 512, 11)
    _single_and_stream(st, 512, 16, 16, "E 8B bf16 b16 ctx 512", tol=STRICT_TC)
    st.set_batch(1, 4096 + 40)


# ------------------------------------------------------------------ S
def test_S_llama32_1b_full_depth():
    st = O.OracleStore(O.preset("llama32_1b"), 1234, 1024 + 40)
    st.synthetic_prefill(1024, 7)
    _single_and_stream(st, 1024, 16, 16, "S 1B bf16 ctx 1024")
    st.close()


# ------------------------------------------------------------------ Q
@pytest.mark.parametrize("qb", [4, 8])
def test_Q_llama31_8b_quant_full_depth(qb):
    st = O.OracleStore(O.preset("llama31_8b").replace(quant_bits=qb), 1234, 1024 + 40)
    st.synthetic_prefill(1024, 7)
    dev = _Dev(st)
    try:
        assert dev.m.info()["quant_inexact_groups"] == 0  # the reference's grid, bit for bit
        e_plain, e_strict, flips = check_step(st, dev.m, [17], 1024, strict=STRICT_TC)
        print(f"Q int{qb} single step: rel_err {e_plain:.2e}, same-KV {e_strict:.2e}, "
              f"flips {flips}")
        decode_stream(st, dev, 1025, prompt_ids(16, 1, st.cfg.vocab_size), 16,
                      f"Q 8B int{qb} ctx 1024", STRICT_TC)
    finally:
        dev.close()
        st.close()


# ------------------------------------------------------------------ H
@pytest.fixture(scope="module")
def store_70b():
    st = O.OracleStore(O.preset("llama31_70b").replace(layers=2), 1234, 512 + 40)
    yield st
    st.close()


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_H_llama3_70b_width_tp_full_vocab(store_70b, tp):
    """70B width (d_model 8192, 64 q / 8 kv heads, d_inter 28672), 2 layers,
    full vocabulary, as TP 2 / 4 / 8 shards co-located on one GPU, the two
    per-layer residual exchanges and the argmax exchange inside the kernel."""
    st = store_70b
    st.synthetic_prefill(512, 7)
    dev = _Dev(st, tp)
    try:
        logits, greedy = dev.step([17], 512)
        k_dev, v_dev = dev.appended(512)
        want_plain = st.forward([17], 512)
        for l in range(st.cfg.layers):
            st.set_length(l, 512)
        want = st.forward([17], 512, k_app=k_dev, v_app=v_dev)
        e, ep = rel_err(logits[0], want[0]), rel_err(logits[0], want_plain[0])
        print(f"H 70B width TP{tp} single step: rel_err {ep:.2e}, same-KV {e:.2e}")
        assert e < STRICT
        assert int(greedy[0]) == int(np.argmax(want[0]))
        decode_stream(st, dev, 513, prompt_ids(16, 1, st.cfg.vocab_size), 16,
                      f"H 70B width 2L TP{tp}")
    finally:
        dev.close()
