"""Device time per decode step for every BASELINE.json config that fits one
B200 (SURVEY.md §8 tags S, E b1/b4, Q int4/int8, H TP1, plus H as a TP2
group co-located on one GPU), with the roofline fraction of each:

    python tools/config_sweep.py [--steps 50] [--out profiles/configs.json]

Bytes per step = SURVEY.md §8(d): streamed weights + KV read incl. the
current token + embedding rows + f32 norm gains.  Weights are synthetic
(device-side seeded init); the model is calibrated (ffb_calibrate) first.
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_22758_b200 import DecodeModel, TPGroup, model_preset

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--out", default="")
ap.add_argument("--only", default="")
a = ap.parse_args()
PEAK = 6650.0
try:
    PEAK = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass

CONFIGS = [  # tag, model, ctx, batch, quant, tp
    ("T", "tiny", 192, 1, 0, 1),
    ("S", "llama32_1b", 1024, 1, 0, 1),
    ("E-b1", "llama31_8b", 4096, 1, 0, 1),
    ("E-b2", "llama31_8b", 4096, 2, 0, 1),
    ("E-b4", "llama31_8b", 4096, 4, 0, 1),
    ("E-b8", "llama31_8b", 4096, 8, 0, 1),
    ("E-b16", "llama31_8b", 4096, 16, 0, 1),
    ("Q-int8", "llama31_8b", 4096, 1, 8, 1),
    ("Q-int4", "llama31_8b", 4096, 1, 4, 1),
    ("H-tp1", "llama31_70b", 4096, 1, 0, 1),
    ("H-tp2-colocated", "llama31_70b", 4096, 1, 0, 2),
]


def step_bytes(cfg, ctx, tp=1):
    kv = cfg.batch * cfg.layers * cfg.n_kv_heads * 2 * cfg.d_head * 2 * (ctx + 1)
    return (cfg.streamed_weight_bytes() + kv + cfg.batch * cfg.d_model * 2 +
            (2 * cfg.layers + 1) * cfg.d_model * 4)


rows = []
for tag, name, ctx, batch, quant, tp in CONFIGS:
    if a.only and tag not in a.only.split(","):
        continue
    cfg = model_preset(name).replace(batch=batch, quant_bits=quant)
    t0 = time.time()
    if tp == 1:
        m = DecodeModel(cfg, ctx + 8)
        m.init_synthetic(1)
        for l in range(cfg.layers):
            m.set_length(l, ctx)
        m.calibrate(3)
        s = torch.cuda.Stream()
        tok = torch.arange(17, 17 + batch, dtype=torch.int64, device="cuda")

        def loop(n):
            for _ in range(n):
                for l in range(cfg.layers):
                    m.set_length(l, ctx)
                m.step_device(tok.data_ptr(), ctx, 0, 0, s.cuda_stream)
    else:
        m = TPGroup(cfg, ctx + 8, tp)
        m.init_synthetic(1)
        s = None

        def loop(n):
            for _ in range(n):
                for l in range(cfg.layers):
                    m.set_length(l, ctx)
                m.step([17] * batch, ctx)
    loop(5)
    torch.cuda.synchronize()
    if s is not None:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s); loop(a.steps); e1.record(s); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
    else:  # host-synchronised group steps (includes the logits gather)
        t = time.perf_counter(); loop(a.steps); ms = (time.perf_counter() - t) * 1e3 / a.steps
    nb = step_bytes(cfg, ctx, tp)
    gbs = nb / ms / 1e6
    row = {"config": tag, "model": name, "ctx": ctx, "batch": batch, "quant_bits": quant, "tp": tp,
           "ms_per_step": round(ms, 4), "ms_per_token": round(ms / batch, 4),
           "tokens_per_s": round(1e3 * batch / ms, 1), "bytes_per_step": nb,
           "achieved_gbs": round(gbs, 1), "frac_of_peak": round(gbs / PEAK, 4),
           "frac_of_8TBs": round(gbs / 8000, 4), "setup_s": round(time.time() - t0, 1)}
    rows.append(row)
    print(json.dumps(row), flush=True)
    m.close()
    del m
    torch.cuda.empty_cache()
if a.out:
    json.dump({"peak_gbs": PEAK, "rows": rows}, open(a.out, "w"), indent=1)
