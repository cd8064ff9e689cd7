"""Developer diagnostics: sync-API step per mode with error checks."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2505_22758_b200 import DecodeModel, RunMode, model_preset

for name, ctx in [("tiny", 128), ("llama32_1b", 1024), ("llama31_8b", 4096)]:
    cfg = model_preset(name)
    m = DecodeModel(cfg, ctx + 8)
    m.init_synthetic(1)
    outs = {}
    for mode in (RunMode.BASELINE, RunMode.FUSED, RunMode.FUSED_OVERLAP):
        m.set_mode(mode)
        for l in range(cfg.layers): m.set_length(l, ctx)
        t = time.time()
        lg, g = m.step([17], ctx)
        dt = time.time() - t
        outs[mode] = lg
        print(name, mode.name, "greedy", g, "argmax", lg.argmax(), "finite", np.isfinite(lg).all(),
              "absmax %.4g" % np.abs(lg).max(), "wall %.2f ms" % (dt * 1e3), flush=True)
    b = outs[RunMode.BASELINE]
    for mode in (RunMode.FUSED, RunMode.FUSED_OVERLAP):
        print("  max|%s - baseline| = %.3g" % (mode.name, np.abs(outs[mode] - b).max()))
    m.close()
