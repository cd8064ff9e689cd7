"""Developer diagnostic: per-prefill error vs the oracle and K/V flip counts."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as O
from gpu_helpers import device_from_store, rel_err
TOY = O.preset("llama31_8b-toy")
for prefill in (0, 1, 2, 3, 5, 17, 255, 256, 300):
    st = O.OracleStore(TOY, 42, prefill + 4); st.synthetic_prefill(prefill, 7)
    m = device_from_store(st)
    got = m.forward([17], prefill)
    want = st.forward([17], prefill)
    K, V = st.kv()
    flips = 0; tot = 0
    for l in range(TOY.layers):
        for h in range(TOY.n_kv_heads):
            k, v = m.kv_get(0, l, h, prefill)
            flips += int((k != K[0, l, h, prefill]).sum() + (v != V[0, l, h, prefill]).sum()); tot += 2 * k.size
    print(f"prefill {prefill:4d} rel_err {rel_err(got[0], want[0]):.3e} kv flips {flips}/{tot}", flush=True)
    m.close()
