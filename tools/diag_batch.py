"""Developer diagnostic: appended K/V ulp distances vs the oracle per batch row."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as O
from gpu_helpers import device_from_store, appended_kv, bf16_ulp_distance
TOY = O.preset("llama31_8b-toy")
for B in (1, 2, 4):
    st = O.OracleStore(TOY.replace(batch=B), 21, 64); st.synthetic_prefill(40, 3)
    m = device_from_store(st)
    tokens = [11, 400, 7, 99][:B]
    got = m.forward(tokens, 40); want = st.forward(tokens, 40)
    kd, vd = appended_kv(m, 40); K, V = st.kv()
    for b in range(B):
        for l in range(TOY.layers):
            uk = bf16_ulp_distance(kd[b, l], K[b, l, :, 40]); uv = bf16_ulp_distance(vd[b, l], V[b, l, :, 40])
            if uk.max() > 1 or uv.max() > 1:
                i = np.unravel_index(np.argmax(uk), uk.shape)
                print(f"B{B} b{b} l{l} K ulp max {uk.max()} at {i}: dev {kd[b,l][i]} ora {K[b,l,:,40][i]}; V ulp max {uv.max()}")
        print(f"B{B} b{b} logits rel {np.abs(got[b]-want[b]).max()/np.abs(want[b]).max():.3g}")
    m.close()
