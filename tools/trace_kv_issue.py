"""When does the producer issue a CTA's attention K/V chunks, relative to
the consumers staging q and finding the ring slots ready?  Needs a library
built with -DFFB_TRACE_PRODUCER (tools/build_variant.sh), which records, per
(CTA, layer), in the S_AOUT trace row: slot 5 = producer reached the first
K/V chunk, 6 = first K/V chunk issued (slot free), 7 = last K/V chunk issued."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2505_22758_b200 import DecodeModel, model_preset

model = sys.argv[1] if len(sys.argv) > 1 else "llama31_8b"
cfg = model_preset(model)
ctx = 4096 if model == "llama31_8b" else 1024
m = DecodeModel(cfg, ctx + 8)
m.init_synthetic(1)
for l in range(cfg.layers):
    m.set_length(l, ctx)
m.calibrate(8)
m.set_trace(True)
for _ in range(3):
    for l in range(cfg.layers):
        m.set_length(l, ctx)
    m.step([17], ctx, logits=False)
tr = m.trace().astype(np.int64)
rows = []
for l in range(cfg.layers):
    a, o, q = tr[:, l * 5 + 1], tr[:, l * 5 + 2], tr[:, l * 5 + 0]
    ok = (a[:, 5] > 0) & (o[:, 6] > 0)
    rel = lambda x: (x[ok] - a[ok, 5]) / 1e3  # relative to q staged
    rows.append([np.median(rel(q[:, 2])),   # QKV done (this CTA)
                 np.median(rel(a[:, 1])),   # ATTN dependency met
                 np.median(rel(o[:, 5])),   # producer reached first K/V chunk
                 np.median(rel(o[:, 6])),   # first K/V chunk issued
                 np.median(rel(o[:, 7])),   # last K/V chunk issued
                 np.median(rel(a[:, 6]))])  # consumer: ring slots ready
r = np.array(rows).mean(0)
print(f"{model}: times relative to q staged (us, median over CTAs, mean over layers)")
for n, v in zip(["QKV done (own)", "ATTN dep met", "prod reached 1st K/V", "1st K/V issued",
                 "last K/V issued", "ring ready"], r):
    print(f"  {n:22s} {v:7.2f}")
