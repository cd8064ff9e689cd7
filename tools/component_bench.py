"""Component ablation (Table 8): stacked attention blocks
and stacked GLU blocks of the Llama-3.1-8B shape, 1 / 4 / 32 layers, in the
three run modes -- the same persistent kernel with a stage mask (DecodeParams::
stage_mask: 0x07 = QKV + attention + O-projection per layer, 0x18 = GLU +
W2), batch 1, and the achieved HBM bandwidth of each block type (the paper's
"stacked GLU blocks exceed 90 % of peak, attention about 50 %").

    python tools/component_bench.py [--ctx 3072] [--steps 50] [--out profiles/components_r02.json]

The vocabulary is cut to 256 rows so the LM-head tail (2 MB) stays out of
the numbers; bytes per step = the blocks' weights (+ the K/V of the attention
blocks).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2505_22758_b200 import DecodeModel, RunMode, model_preset  # noqa: E402

# PAPER.md Table 8 (H100, ms): module -> layers -> (baseline, fused, +overlap)
PAPER = {"attn": {1: (0.089, 0.089, 0.090), 4: (0.357, 0.264, 0.256), 32: (2.857, 1.761, 1.683)},
         "glu": {1: (0.122, 0.122, 0.122), 4: (0.488, 0.466, 0.464), 32: (3.905, 3.689, 3.661)}}
MASK = {"attn": 0x07, "glu": 0x18}

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=3072)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--out", default="")
a = ap.parse_args()
peak = 6650.0
try:
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass

base = model_preset("llama31_8b")
D, DI, dh, nq, nkv = base.d_model, base.d_inter, base.d_head, base.n_q_heads, base.n_kv_heads
rows = []
for mod in ("attn", "glu"):
    for L in (1, 4, 32):
        cfg = base.replace(layers=L, vocab_size=256)
        m = DecodeModel(cfg, a.ctx + 8)
        m.init_synthetic(3)
        m.set_option("stage_mask", MASK[mod])
        if mod == "attn":
            nbytes = L * ((nq + 2 * nkv) * dh * D * 2 + D * nq * dh * 2 + nkv * 2 * dh * 2 * (a.ctx + 1))
        else:
            nbytes = L * 3 * DI * D * 2
        s = torch.cuda.Stream()
        tok = torch.full((1,), 17, dtype=torch.int64, device="cuda")

        def loop(n):
            for _ in range(n):
                for l in range(L):
                    m.set_length(l, a.ctx)
                m.step_device(tok.data_ptr(), a.ctx, 0, 0, s.cuda_stream)

        res = {"module": mod, "layers": L, "ctx": a.ctx, "bytes_per_step": nbytes}
        for name, mode in (("baseline", RunMode.BASELINE), ("fused", RunMode.FUSED),
                           ("fused_overlap", RunMode.FUSED_OVERLAP)):
            m.set_mode(mode)
            loop(5)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            loop(a.steps)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            res[name + "_ms"] = round(ms, 4)
            res[name + "_gbs"] = round(nbytes / ms / 1e6, 1)
        res["frac_of_peak_overlap"] = round(res["fused_overlap_gbs"] / peak, 3)
        res["paper_h100_ms"] = PAPER[mod][L]
        print(json.dumps(res), flush=True)
        rows.append(res)
        m.close()

md = [f"# Component ablation (PAPER.md Table 8) on one B200: Llama-3.1-8B shape, batch 1, ctx {a.ctx}", "",
      "Stacked blocks of one kind in one persistent kernel (stage mask); ms per step, and in brackets the",
      "paper's H100 ms; GB/s = block weights (+ K/V) per step over the FusedOverlap time; peak "
      f"{peak:.0f} GB/s.", "",
      "| module | layers | baseline | fused | +overlap | GB/s (overlap) | of peak |", "|---|---|---|---|---|---|---|"]
for r in rows:
    p = r["paper_h100_ms"]
    md.append(f"| {r['module']} | {r['layers']} | {r['baseline_ms']:.3f} ({p[0]}) | {r['fused_ms']:.3f} ({p[1]}) | "
              f"{r['fused_overlap_ms']:.3f} ({p[2]}) | {r['fused_overlap_gbs']:.0f} | {r['frac_of_peak_overlap']:.2f} |")
print("\n".join(md))
if a.out:
    with open(a.out, "w") as f:
        json.dump({"ctx": a.ctx, "peak_gbs": peak, "rows": rows}, f, indent=1)
    with open(a.out.replace(".json", ".md"), "w") as f:
        f.write("\n".join(md) + "\n")
