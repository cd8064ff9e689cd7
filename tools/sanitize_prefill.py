"""compute-sanitizer target for the prefill kernels (csrc/prefill.cu): toy
shapes, bf16 / int4 / int8 and batch 16, prompts on top of existing context.

    compute-sanitizer --tool memcheck python tools/sanitize_prefill.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from gpu_helpers import device_from_store  # noqa: E402

CASES = [("llama31_8b-toy", 0, 1, 0, 37), ("llama31_8b-toy", 0, 2, 20, 9), ("llama31_8b-toy", 4, 1, 5, 11),
         ("llama31_8b-toy", 8, 1, 0, 7), ("llama31_8b-toy", 0, 16, 3, 5),
         ("llama31_8b", 4, 1, 3, 6), ("llama31_8b", 8, 1, 0, 5)]  # 8B width: tensor-core code order
for name, qb, batch, ctx, n in CASES:
    cfg = O.preset(name).replace(quant_bits=qb, batch=batch)
    if name == "llama31_8b":
        cfg = cfg.replace(layers=1, vocab_size=4096)
    st = O.OracleStore(cfg, 3, ctx + n + 2)
    if ctx:
        st.synthetic_prefill(ctx, 7)
    with device_from_store(st) as m:
        toks = np.random.default_rng(1).integers(0, cfg.vocab_size, size=(n, batch))
        lg, g = m.prefill(toks, ctx)
        assert np.isfinite(lg).all()
        m.step(list(range(batch)), ctx + n)
    print(f"{name} q{qb} b{batch} ctx {ctx} n {n}: ok", flush=True)
