import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle as O
from gpu_helpers import device_from_store, rel_err
from paper_2505_22758_b200 import RunMode
name = "llama31_8b-toy"
for B in (1, 4):
  for L in (2, 3, 4):
    for ms in (4, 8):
      cfg = O.preset(name).replace(batch=B, layers=L)
      toks = [11, 400, 7, 99][:B]
      res = []
      for mode in (RunMode.FUSED, RunMode.FUSED_OVERLAP):
        st = O.OracleStore(cfg, 42, ms); st.synthetic_prefill(0, 7)
        with device_from_store(st, mode=mode) as m:
            got = m.forward(toks, 0)
        want = st.forward(toks, 0)
        res.append(max(rel_err(got[b], want[b]) for b in range(B)))
      print(name, "B", B, "L", L, "max_seq", ms, "fused %.2e overlap %.2e" % tuple(res))
