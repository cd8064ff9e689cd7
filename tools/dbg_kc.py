"""Debug: batch-16 K-chunk geometry on small shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
from gpu_helpers import device_from_store, check_step
shape = sys.argv[1] if len(sys.argv) > 1 else "a"
cfg = {"a": O.ModelCfg(2, 512, 2048, 64, 8, 2, 1024),
       "g1": O.ModelCfg(2, 2048, 2048, 64, 32, 8, 1024),
       "e": O.preset("llama31_8b").replace(layers=1, vocab_size=4096)}[shape].replace(batch=16)
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 64
st = O.OracleStore(cfg, 3, ctx + 6)
st.synthetic_prefill(ctx, 1)
TOK = [17, 3, 99, 400, 11, 250, 7, 501, 42, 1, 333, 64, 128, 5, 77, 260]
with device_from_store(st) as m:
    print(shape, check_step(st, m, TOK, ctx))
