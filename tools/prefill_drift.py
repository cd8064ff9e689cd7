"""Drift of the device paths from the f64 oracle over a whole prompt (no
K/V hook): GEMM prefill (3- and 2-term) vs the persistent kernel's own
decode-as-prefill, several prompts, toy / tiny shapes.

    python tools/prefill_drift.py [--n 24] [--prompts 8]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from gpu_helpers import device_from_store, rel_err  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--prompts", type=int, default=8)
ap.add_argument("--preset", default="llama31_8b-toy")
a = ap.parse_args()
cfg = O.preset(a.preset)
if a.preset == "tiny":
    cfg = cfg.replace(layers=2)
rows = []
for seed in range(a.prompts):
    toks = np.random.default_rng(seed).integers(0, cfg.vocab_size, size=(a.n, 1))
    ora = O.OracleStore(cfg, 42, a.n + 2)
    for t in range(a.n):
        want = ora.forward(toks[t], t)
    res = {}
    for label, terms in (("prefill3", 3), ("prefill2", 2), ("loop", 0)):
        st = O.OracleStore(cfg, 42, a.n + 2)
        with device_from_store(st, a.n + 2) as m:
            if terms:
                m.set_option("prefill_terms", terms)
                lg, _ = m.prefill(toks, 0)
            else:
                for t in range(a.n):
                    lg, _ = m.step(toks[t], t)
            k, v = m.kv_export(0, a.n)
        res[label] = (rel_err(lg[0], want[0]), k, v)
    K, V = ora.kv()
    kd = {lab: int((res[lab][1][:, :, :, :, :] != K[:, :, :, :a.n]).sum()) for lab in res}
    line = "  ".join(f"{lab} {res[lab][0]:.2e} ({kd[lab]} kv diffs)" for lab in res)
    print(f"prompt {seed}: {line}", flush=True)
    rows.append([res[lab][0] for lab in res])
r = np.array(rows)
print("median rel_err prefill3 %.2e prefill2 %.2e loop %.2e" % tuple(np.median(r, axis=0)))
print("max    rel_err prefill3 %.2e prefill2 %.2e loop %.2e" % tuple(np.max(r, axis=0)))
