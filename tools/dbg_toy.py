"""Developer check: per-layer appended K/V and logits error of the toy preset
against the oracle, per run mode (python tools/dbg_toy.py [batch])."""
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle as O
from gpu_helpers import device_from_store, appended_kv, rel_err
from paper_2505_22758_b200 import RunMode
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
TOY = O.preset("llama31_8b-toy").replace(batch=B)
toks = [11, 400, 7, 99][:B]
for prefill in (0, 1, 2, 40):
  for mode in (RunMode.BASELINE, RunMode.FUSED, RunMode.FUSED_OVERLAP):
    st = O.OracleStore(TOY, 42, prefill + 4); st.synthetic_prefill(prefill, 7)
    with device_from_store(st, mode=mode) as m:
        import os
        if "PF" in os.environ:
            m.set_option("l2_prefetch_bytes", int(os.environ["PF"]))
        if "RANK0" in os.environ:
            m.set_option("sm_rank", 0)
        got = m.forward(toks, prefill)
        kd, vd = appended_kv(m, prefill)
    want = st.forward(toks, prefill)
    K, V = st.kv()
    ko = K[:, :, :, prefill]; vo = V[:, :, :, prefill]
    print(prefill, mode.name, "logit err", max(rel_err(got[b], want[b]) for b in range(B)),
          "k err [b][l]", [[round(float(np.abs(kd[b, l] - ko[b, l]).max()), 4) for l in range(TOY.layers)] for b in range(B)])
