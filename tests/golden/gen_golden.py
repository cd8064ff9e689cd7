"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

The reference ships no golden vectors (proj/tests/golden/toy_block0_fused.txt
is empty and SPEC.md:401's logits file was never produced), so these are
produced here by running the reference's own code: fusesim::init_weights,
the synthetic_prefill helper of proj/tests/test_interpreter.cpp:16-30,
reference_forward (reference.hpp:37-139) and execute_program
(interpreter.hpp:502-506), compiled unchanged from /root/reference by
oracle/Makefile.  Run from the repo root:

    make -C oracle && python tests/golden/gen_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def fnv(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % O.lib().fo_fnv1a(a.ctypes.data, a.nbytes, 0xcbf29ce484222325)


def top5(v):
    idx = np.argsort(-v, kind="stable")[:5]
    return [int(i) for i in idx], [float(v[i]) for i in idx]


def main():
    meta = {"generator": "tests/golden/gen_golden.py", "source": "oracle/_ref (reference headers)"}

    # 1. toy preset, the reference's own interpreter test (test_interpreter.cpp:51-70)
    toy = O.preset("llama31_8b-toy")
    toy_logits, toy_exec, toy_kv = {}, {}, {}
    for prefill in (0, 1, 255, 256, 300):
        r = O.RefStore(toy, 42, prefill + 4)
        r.synthetic_prefill(prefill, 7)
        toy_logits[str(prefill)] = r.forward([17], prefill)[0]
        k, v = r.kv_get(0, 0, 0, prefill)
        toy_kv[str(prefill)] = np.concatenate([k, v])
        r2 = O.RefStore(toy, 42, prefill + 4)
        r2.synthetic_prefill(prefill, 7)
        toy_exec[str(prefill)] = r2.execute([17], prefill, mode=2, stage_size=32768, num_sms=132)[0]
    np.savez_compressed(os.path.join(OUT, "toy_logits.npz"),
                        **{f"oracle_{k}": v for k, v in toy_logits.items()},
                        **{f"interp_{k}": v for k, v in toy_exec.items()},
                        **{f"kv_{k}": v for k, v in toy_kv.items()})
    r = O.RefStore(toy, 42, 8)
    meta["toy_weight_fnv"] = {n: fnv(r.tensor(n)) for n in
                              ["embedding", "lm_head", "final_norm", "layer.0.wqkv",
                               "layer.3.wffn2t", "layer.1.norm_attn"]}

    # 2. toy int4 (reference quant scheme, quant.hpp:42-54)
    tq = toy.replace(quant_bits=4, quant_group=128)
    rq = O.RefStore(tq, 42, 40)
    rq.synthetic_prefill(33, 7)
    q_logits = rq.forward([17], 33)[0]
    meta["toy_int4_weight_fnv"] = {n: fnv(rq.tensor(n)) for n in ["layer.0.wqkv", "lm_head"]}
    np.save(os.path.join(OUT, "toy_int4_logits.npy"), q_logits)

    # 3. tiny T: 128-token prompt + 64 greedy steps
    T = O.preset("tiny")
    prompt = O.tiny_prompt(128, T.vocab_size)
    steps = 128 + 64
    r = O.RefStore(T, 1234, steps + 1)
    fed, argmax, top_ids, top_vals, sums, gaps = [], [], [], [], [], []
    keep = {}
    tok = prompt[0]
    for i in range(steps):
        fed.append(int(tok))
        lg = r.forward([tok], i)[0]
        a = int(np.argmax(lg))
        argmax.append(a)
        ids, vals = top5(lg)
        top_ids.append(ids)
        top_vals.append(vals)
        sums.append([float(lg.sum()), float((lg * lg).sum())])
        gaps.append(float((vals[0] - vals[1]) / np.abs(lg).max()))
        if i in (0, 127, 191):
            keep[f"logits_{i}"] = lg.astype(np.float64)
        tok = prompt[i + 1] if i + 1 < 128 else a
    np.savez_compressed(os.path.join(OUT, "tiny_decode.npz"), fed=np.array(fed, np.int64),
                        argmax=np.array(argmax, np.int64), top_ids=np.array(top_ids, np.int64),
                        top_vals=np.array(top_vals), sums=np.array(sums), gaps=np.array(gaps),
                        **keep)
    r2 = O.RefStore(T, 1234, 8)
    meta["tiny_weight_fnv"] = {n: fnv(r2.tensor(n)) for n in
                               ["embedding", "lm_head", "layer.0.wqkv", "layer.3.wffn1"]}
    meta["tiny_prompt_head"] = prompt[:8]
    meta["tiny_min_top_gap"] = min(gaps)

    # 4. byte accounting (tensor_store.hpp:170-192) for the BASELINE shapes
    meta["streamed_weight_bytes"] = {
        name: int(O.ref_lib().ref_streamed_weight_bytes(O.preset(name).c()))
        for name in O.PRESETS}
    meta["total_weight_bytes"] = {
        name: int(O.ref_lib().ref_total_weight_bytes(O.preset(name).c()))
        for name in O.PRESETS}
    q8 = O.preset("llama31_8b").replace(quant_bits=4)
    meta["streamed_weight_bytes"]["llama31_8b_int4"] = int(
        O.ref_lib().ref_streamed_weight_bytes(q8.c()))

    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote fixtures to", OUT)


if __name__ == "__main__":
    main()
