"""Debug: batch-16 determinism / mode agreement on the toy shape (multi-step)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
from gpu_helpers import device_from_store
from paper_2505_22758_b200 import RunMode
TOY = O.preset("llama31_8b-toy")
TOK = [17, 3, 99, 400, 11, 250, 7, 501, 42, 1, 333, 64, 128, 5, 77, 260]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
res = {}
for mode in [RunMode.FUSED_OVERLAP, RunMode.FUSED, RunMode.BASELINE]:
    st = O.OracleStore(TOY.replace(batch=B), 9, 110)
    st.synthetic_prefill(100, 5)
    with device_from_store(st, mode=mode) as m:
        steps = []
        for i in range(4):
            lg, g = m.step(TOK[:B], 100 + i)
            steps.append(lg)
        res[mode.name] = steps
for k, v in res.items():
    for i in range(4):
        d = np.abs(v[i] - res["FUSED_OVERLAP"][i])
        print(k, "step", i, "max diff", float(d.max()), "rows", np.nonzero(d.max(axis=1))[0].tolist()[:8])

# where does BASELINE diverge: K rows at positions 100 / 101 per layer
kv = {}
for mode in [RunMode.FUSED_OVERLAP, RunMode.BASELINE]:
    st = O.OracleStore(TOY.replace(batch=B), 9, 110)
    st.synthetic_prefill(100, 5)
    with device_from_store(st, mode=mode) as m:
        m.step(TOK[:B], 100)
        m.step(TOK[:B], 101)
        kv[mode.name] = {(b, l, pos): m.kv_get(b, l, 0, pos)[0] for b in range(B) for l in range(4)
                         for pos in (100, 101)}
for key in sorted(kv["BASELINE"]):
    d = float(np.abs(kv["BASELINE"][key] - kv["FUSED_OVERLAP"][key]).max())
    if d > 0:
        print("K differs at (b, l, pos)", key, d)
