"""The paper's stacked-linear fusion ablation (Table "Latencies
of stacked linear layers") on one B200: square bf16 layers, batch 1, as
   baseline  -- one kernel launch per layer (RunMode::Baseline),
   fused     -- one persistent launch, producer waits at layer boundaries,
   overlap   -- one persistent launch streaming across layer boundaries,
next to the paper's published H100 latencies.  Weights are synthetic
(device-side seeded init), 2 GB of bf16 per 32 layers at 8K.

    python tools/linear_bench.py [--reps 50] [--out profiles/linear_r01.json]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_22758_b200 import DecodeModel, ModelConfig, RunMode

# PAPER.md:178-190 (H100, ms): (dim, layers) -> (baseline, fused, overlap)
PAPER_H100 = {(2048, 1): (0.013, 0.013, 0.012), (2048, 4): (0.050, 0.029, 0.027),
              (2048, 32): (0.403, 0.169, 0.154), (4096, 1): (0.021, 0.021, 0.021),
              (4096, 4): (0.084, 0.060, 0.060), (4096, 32): (0.675, 0.423, 0.423),
              (8192, 1): (0.062, 0.062, 0.062), (8192, 4): (0.250, 0.221, 0.218),
              (8192, 32): (1.998, 1.543, 1.513)}

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--out", default="")
a = ap.parse_args()
rows = []
s = torch.cuda.Stream()
for (d, L), paper in PAPER_H100.items():
    m = DecodeModel(ModelConfig(L, d, 0, 0, 0, 0, 0, kind=1), 1)
    m.init_synthetic(7)
    res = {}
    for name, mode in (("baseline", RunMode.BASELINE), ("fused", RunMode.FUSED),
                       ("overlap", RunMode.FUSED_OVERLAP)):
        m.set_mode(mode)
        for _ in range(5):
            m.linear_forward_device(0, 0, s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(a.reps):
            m.linear_forward_device(0, 0, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / a.reps
    nb = L * d * d * 2
    row = {"dim": d, "layers": L, "weight_bytes": nb,
           **{f"{k}_ms": round(v, 4) for k, v in res.items()},
           "overlap_gbs": round(nb / res["overlap"] / 1e6, 1),
           "paper_h100_ms": dict(zip(("baseline", "fused", "overlap"), paper)),
           "speedup_vs_paper_overlap": round(paper[2] / res["overlap"], 2),
           "fusion_gain": round(res["baseline"] / res["overlap"], 2)}
    rows.append(row)
    print(json.dumps(row), flush=True)
    m.close()
if a.out:
    json.dump({"rows": rows}, open(a.out, "w"), indent=1)
