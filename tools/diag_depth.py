"""Parity error vs depth (diagnostic): strict rel_err of one decode step
(device K/V rows fed to the oracle) for the first L layers of a config."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
from gpu_helpers import appended_kv, device_from_store, rel_err  # noqa: E402

name = sys.argv[1]
qb = int(sys.argv[2])
batch = int(sys.argv[3])
ctx = int(sys.argv[4])
for L in [int(x) for x in sys.argv[5].split(",")]:
    cfg = O.preset(name).replace(layers=L, quant_bits=qb, batch=batch)
    st = O.OracleStore(cfg, 1234, ctx + 4)
    if batch == 1:
        st.synthetic_prefill(ctx, 7)
    else:
        from test_gpu_fulldepth import fast_prefill
        fast_prefill(st, ctx, 11)
    toks = list(range(17, 17 + batch))
    with device_from_store(st) as m:
        got = m.forward(toks, ctx)
        k, v = appended_kv(m, ctx)
    for l in range(L):
        st.set_length(l, ctx)
    want = st.forward(toks, ctx, k_app=k, v_app=v)
    errs = [rel_err(got[b], want[b]) for b in range(batch)]
    scale = np.abs(want).max()
    print(f"{name} q{qb} b{batch} L={L}: strict rel_err max {max(errs):.2e} "
          f"(per row {np.round(np.array(errs) * 1e6, 1).tolist()} e-6), max|logit| {scale:.3f}",
          flush=True)
    st.close()
