"""Per-CTA timeline of the LM-head stage (the step's last, 1 GB at 8B):
dependency met / done relative to the first CTA's met, ring starvation,
rows, and the same for one GLU stage, from the kernel's %globaltimer trace."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2505_22758_b200 import DecodeModel, model_preset

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama31_8b")
ap.add_argument("--ctx", type=int, default=4096)
ap.add_argument("--calibrate", type=int, default=8)
a = ap.parse_args()
cfg = model_preset(a.model)
m = DecodeModel(cfg, a.ctx + 8)
m.init_synthetic(1)
for l in range(cfg.layers):
    m.set_length(l, a.ctx)
if a.calibrate:
    m.calibrate(a.calibrate)
w = m.plan_weights()
m.set_trace(True)
for _ in range(3):
    for l in range(cfg.layers):
        m.set_length(l, a.ctx)
    m.step([17], a.ctx, logits=False)
tr = m.trace().astype(np.int64)
S = tr.shape[1]
for name, s in (("lmhead", S - 1), ("glu l16", 16 * 5 + 3)):
    met, done, starve = tr[:, s, 1], tr[:, s, 2], tr[:, s, 4]
    t0 = met.min()
    dm, dd = (met - t0) / 1e3, (done - t0) / 1e3
    o = np.argsort(-dd)
    print(f"{name}: met spread {dm.max():.2f} us; done median {np.median(dd):.2f} max {dd.max():.2f} "
          f"min {dd.min():.2f} us; starve median {np.median(starve) / 1e3:.2f} us")
    print("  last:", ", ".join(f"cta {c} done {dd[c]:.1f} starve {starve[c] / 1e3:.1f} w {w[c]:.3f}" for c in o[:6]))
    print("  first:", ", ".join(f"cta {c} done {dd[c]:.1f} starve {starve[c] / 1e3:.1f} w {w[c]:.3f}" for c in o[-4:]))
    q = np.percentile(dd, [10, 25, 50, 75, 90, 99])
    print("  done percentiles 10/25/50/75/90/99:", " ".join(f"{x:.1f}" for x in q))
    print(f"  corr(done, weight) {np.corrcoef(dd, w)[0, 1]:.2f}")
