"""Developer performance probe: device time per decode step for each run
mode, the streaming-only schedule (ffb_set_debug(1)) and an L2-prefetch
window sweep."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_22758_b200 import DecodeModel, RunMode, model_preset

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama31_8b")
ap.add_argument("--ctx", type=int, default=4096)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--quant", type=int, default=0, help="weight bits: 0 (bf16), 4, 8")
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--sweep", default="", help="comma list of l2_prefetch_bytes")
ap.add_argument("--ncu", action="store_true", help="few launches, for profiling")
ap.add_argument("--calibrate", type=int, default=0, help="ffb_calibrate iterations first")
ap.add_argument("--masks", default="", help="comma list of calib_mask values to compare")
ap.add_argument("--ab", default="", help="option=v0,v1: interleaved A/B of one option")
ap.add_argument("--sets", default="", help="'k=v,k=v|k=v,...': option sets timed interleaved (3 reps)")
ap.add_argument("--pf-stages", type=int, default=0x3f, help="l2_prefetch_stages mask for --sweep")
a = ap.parse_args()

cfg = model_preset(a.model).replace(batch=a.batch, quant_bits=a.quant)
m = DecodeModel(cfg, a.ctx + 8)
m.init_synthetic(1)
if a.calibrate:
    for l in range(cfg.layers):
        m.set_length(l, a.ctx)
    m.calibrate(a.calibrate)
    w = m.plan_weights()
    print(f"calibrated weights: min {w.min():.3f} max {w.max():.3f} std {w.std():.3f}")
s = torch.cuda.Stream()
tok = torch.full((a.batch,), 17, dtype=torch.int64, device="cuda")
kv = a.batch * cfg.layers * cfg.n_kv_heads * 2 * cfg.d_head * 2 * (a.ctx + 1)
nbytes = cfg.streamed_weight_bytes() + kv

def loop(n):
    for _ in range(n):
        for l in range(cfg.layers):
            m.set_length(l, a.ctx)
        m.step_device(tok.data_ptr(), a.ctx, 0, 0, s.cuda_stream)

if a.ncu:
    loop(4)
    torch.cuda.synchronize()
    sys.exit(0)

def timeit(name):
    loop(5); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s); loop(a.steps); e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(f"{a.model} b{a.batch} ctx{a.ctx} {name:22s} {ms:.4f} ms/step {nbytes / ms / 1e9:6.2f} TB/s", flush=True)

if a.ab:
    key, vals = a.ab.split("=")
    m.set_mode(RunMode.FUSED_OVERLAP)
    for rep in range(3):
        for v in [int(x, 0) for x in vals.split(",")]:
            m.set_option(key, v)
            timeit(f"{key}={v}")
    sys.exit(0)
if a.sets:
    m.set_mode(RunMode.FUSED_OVERLAP)
    sets = [[kv.split("=") for kv in grp.split(",") if kv] for grp in a.sets.split("|")]
    for rep in range(3):
        for grp in sets:
            for k, v in grp:
                m.set_option(k.strip(), int(v, 0))
            timeit(",".join(f"{k.strip()}={v}" for k, v in grp))
    sys.exit(0)
if a.masks:
    m.set_mode(RunMode.FUSED_OVERLAP)
    for rep in range(2):
        for mk in [int(x, 0) for x in a.masks.split(",")]:
            m.set_option("calib_mask", mk)
            timeit(f"calib_mask={mk:#x}")
    sys.exit(0)
if a.sweep:
    m.set_mode(RunMode.FUSED_OVERLAP)
    m.set_option("l2_prefetch_stages", a.pf_stages)
    for w in [int(x) for x in a.sweep.split(",")]:
        m.set_option("l2_prefetch_bytes", w)
        timeit(f"overlap l2pf={w >> 10}K")
    sys.exit(0)
for name, mode, dbg in [("fused_overlap", RunMode.FUSED_OVERLAP, 0), ("fused", RunMode.FUSED, 0),
                        ("baseline", RunMode.BASELINE, 0),
                        ("stream_only", RunMode.FUSED_OVERLAP, 1)]:
    m.set_mode(mode); m.set_debug(dbg)
    timeit(name)
m.set_debug(0)
