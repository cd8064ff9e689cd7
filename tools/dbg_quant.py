import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle as O
from gpu_helpers import device_from_store, appended_kv, rel_err
from paper_2505_22758_b200 import RunMode
qb = int(sys.argv[1]) if len(sys.argv) > 1 else 8
TOY = O.preset("llama31_8b-toy").replace(quant_bits=qb)
for prefill in (0, 1, 2, 40, 300):
  for mode in (RunMode.BASELINE, RunMode.FUSED, RunMode.FUSED_OVERLAP):
    st = O.OracleStore(TOY, 42, prefill + 4); st.synthetic_prefill(prefill, 7)
    with device_from_store(st, mode=mode) as m:
        got = m.forward([17], prefill)
        kd, vd = appended_kv(m, prefill)
    want = st.forward([17], prefill)
    K, V = st.kv()
    print(prefill, mode.name, "logit err %.2e" % rel_err(got[0], want[0]),
          "k err/layer", [round(float(np.abs(kd[0, l] - K[0, l, :, prefill]).max()), 5) for l in range(TOY.layers)])
