"""Per-stage timeline of one decode step from the kernel's %globaltimer trace.

Trace slots per (CTA, stage): 0 entry, 1 dependency met, 2 done (arrived),
3 stage mark (QKV: activations normalised; ATTN: ring chunks done),
4 ns starved waiting for ring data (consumer thread 0).
Per stage type, mean over layers of medians over CTAs:
  wait = met - entry ; mark = mark - met ; starve = slot 4 ; work = done - met
  span = last done - first met ; gap = first met - previous stage's last done
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2505_22758_b200 import DecodeModel, RunMode, model_preset

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama31_8b")
ap.add_argument("--ctx", type=int, default=4096)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--quant", type=int, default=0, help="weight bits: 0 (bf16), 4, 8")
ap.add_argument("--mode", default="fused_overlap")
ap.add_argument("--reverse", action="store_true", help="plan_reverse option")
ap.add_argument("--calibrate", type=int, default=0, help="ffb_calibrate iterations first")
ap.add_argument("--mask", type=lambda v: int(v, 0), default=0x1f, help="stage_mask (component ablation)")
ap.add_argument("--vocab", type=int, default=0, help="vocabulary rows (0: the preset's)")
ap.add_argument("--opt", action="append", default=[], help="ffb_set_option key=value (repeatable)")
a = ap.parse_args()
cfg = model_preset(a.model).replace(batch=a.batch, quant_bits=a.quant)
if a.vocab:
    cfg = cfg.replace(vocab_size=a.vocab)
m = DecodeModel(cfg, a.ctx + 8, mode={"fused_overlap": RunMode.FUSED_OVERLAP, "fused": RunMode.FUSED,
                                      "baseline": RunMode.BASELINE}[a.mode])
m.init_synthetic(1)
if a.mask != 0x1f:
    m.set_option("stage_mask", a.mask)
for kv in a.opt:
    k, v = kv.split("=")
    m.set_option(k, int(v, 0))
if a.reverse:
    m.set_option("plan_reverse", 1)
if a.calibrate:
    for l in range(cfg.layers):
        m.set_length(l, a.ctx)
    m.calibrate(a.calibrate)
m.set_trace(True)
for _ in range(3):
    for l in range(cfg.layers):
        m.set_length(l, a.ctx)
    m.step([17] * a.batch, a.ctx, logits=False)
tr = m.trace().astype(np.int64)  # [grid][S][8]
S = tr.shape[1]
t0 = tr[:, 0, 0][tr[:, 0, 0] > 0].min()
names = ["qkv", "attn", "aout", "glu", "red"]
rows = {n: [] for n in names + ["lmhead"]}
prev_done = None
for s in range(S):
    ent, met, done, mk, starve = (tr[:, s, i] for i in range(5))
    ok = met > 0
    dn = done > 0
    name = "lmhead" if s == S - 1 else names[s % 5]
    if ok.sum() == 0:
        continue
    med = lambda x, sel: float(np.median(x[sel])) / 1e3 if sel.any() else 0.0
    km = (mk > 0) & ok
    last = done[dn].max() if dn.any() else met[ok].max()
    rows[name].append((med(met - ent, ok), med(mk - met, km), med(starve, dn),
                       med(done - met, dn), (last - met[ok].min()) / 1e3,
                       (met[ok].min() - prev_done) / 1e3 if prev_done is not None else 0.0))
    prev_done = last
print(f"{a.model} b{a.batch} ctx {a.ctx} {a.mode}: step span {(tr[:, :, 2].max() - t0) / 1e3:.1f} us")
print(f"{'stage':8s} {'n':>3s} {'wait':>7s} {'mark':>7s} {'starve':>7s} {'work':>7s} {'span':>7s} {'gap':>6s}  us")
for n, v in rows.items():
    if v:
        v = np.array(v)
        print(f"{n:8s} {len(v):3d} " + " ".join(f"{x:7.2f}" for x in v.mean(0)))
pf = tr[:, S - 1, 5]
print(f"L2-prefetched bytes per CTA per step: median {np.median(pf) / 1e6:.2f} MB, "
      f"max {pf.max() / 1e6:.2f} MB, total {pf.sum() / 1e9:.2f} GB")
# per-CTA GLU balance: which CTAs finish GLU last, and does it follow the SM?
glu = [s for s in range(S - 1) if s % 5 == 3]
work = np.stack([(tr[:, s, 2] - tr[:, s, 1]) for s in glu], 1) / 1e3   # [grid][L]
starve = np.stack([tr[:, s, 4] for s in glu], 1) / 1e3
done_rel = np.stack([(tr[:, s, 2] - tr[:, s, 2].min()) for s in glu], 1) / 1e3
sm = tr[:, S - 1, 6]
order = np.argsort(-done_rel.mean(1))
print("GLU: CTAs finishing last (mean over layers): cta sm done_after_first(us) work starve")
for c in order[:8]:
    print(f"  cta {c:3d} sm {sm[c]:3d} {done_rel[c].mean():6.2f} {work[c].mean():6.2f} {starve[c].mean():6.2f}")
print("  fastest:", ", ".join(f"cta {c} sm {sm[c]} {done_rel[c].mean():.2f}" for c in order[-4:]))
print(f"  corr(done, cta)={np.corrcoef(done_rel.mean(1), np.arange(len(sm)))[0,1]:.2f} "
      f"corr(done, sm)={np.corrcoef(done_rel.mean(1), sm)[0,1]:.2f}; "
      f"per-layer spread of done: {np.mean(done_rel.max(0)):.2f} us")
for s_name, s_idx in (("qkv", 0), ("aout", 2)):
    ss = [s for s in range(S - 1) if s % 5 == s_idx]
    dr = np.stack([(tr[:, s, 2] - tr[:, s, 2].min()) for s in ss], 1) / 1e3
    o = np.argsort(-dr.mean(1))
    print(f"{s_name}: done spread {np.mean(dr.max(0)):.2f} us; slowest ctas {list(o[:6])}; "
          f"corr(done, cta)={np.corrcoef(dr.mean(1), np.arange(len(sm)))[0,1]:.2f}")
if os.environ.get("QKV_CTAS"):  # per-CTA QKV timeline of the slowest / a typical CTA
    ss = [s for s in range(S - 1) if s % 5 == 0]
    base = np.stack([tr[:, s, 1].astype(np.int64) for s in ss], 1)
    base = base - base.min(0, keepdims=True)
    for c in list(np.argsort(-np.stack([tr[:, s, 2] - tr[:, s, 2].min() for s in ss], 1).mean(1))[:6]) + [10, 60]:
        ent = np.mean([(tr[c, s, 0] - tr[:, s, 1].min()) / 1e3 for s in ss])
        met = np.mean([(tr[c, s, 1] - tr[:, s, 1].min()) / 1e3 for s in ss])
        mk = np.mean([(tr[c, s, 3] - tr[:, s, 1].min()) / 1e3 for s in ss])
        dn = np.mean([(tr[c, s, 2] - tr[:, s, 1].min()) / 1e3 for s in ss])
        stv = np.mean([tr[c, s, 4] / 1e3 for s in ss])
        print(f"  qkv cta {c:3d} sm {int(tr[c, S - 1, 6]):3d} unit {'attn' if c < 144 else 'idle'}: entry {ent:6.2f} met {met:6.2f} mark {mk:6.2f} done {dn:6.2f} starve {stv:5.2f} us "
              f"(rel. to the first CTA's dependency met)")
# attention breakdown (slots 5: q staged, 6: ring slots ready, 3: pass done,
# 7: partial written; 2: combine done, last arriver only)
att = [s for s in range(S - 1) if s % 5 == 1]
def seg(a, b, sel=None):
    v = []
    for s in att:
        x = tr[:, s, a].astype(np.int64); y = tr[:, s, b].astype(np.int64)
        ok = (x > 0) & (y > x)
        if ok.any():
            v.append(np.median((y - x)[ok]) / 1e3)
    return np.mean(v) if v else float("nan")
print(f"attn: dep->q {seg(1, 5):.2f}  q->ring {seg(5, 6):.2f}  pass {seg(6, 3):.2f}  "
      f"partial {seg(3, 7):.2f}  combine(last) {seg(7, 2):.2f} us")
if os.environ.get("PHASES"):
    print(f"attn phases: ring->A {seg(6, 5):.2f}  A->B {seg(5, 7):.2f}  B->C/end {seg(7, 3):.2f} us")

if os.environ.get("COMBINE"):
    print(f"combine: partial->atomic-done {seg(7, 5):.2f}  ->ml-loaded {seg(5, 6):.2f}  ->done {seg(6, 2):.2f} us")

if os.environ.get("GLUSPLIT"):
    g = [s for s in range(S - 1) if s % 5 == 3]
    def seg2(a, b):
        v = []
        for s in g:
            x = tr[:, s, a].astype(np.int64); y = tr[:, s, b].astype(np.int64)
            ok = (x > 0) & (y > x)
            if ok.any(): v.append(np.median((y - x)[ok]) / 1e3)
        return np.mean(v) if v else float("nan")
    print(f"glu: dep->ffn1 done {seg2(1, 3):.2f}  ffn1->done {seg2(3, 2):.2f} us")

if os.environ.get("ATTNCTA"):  # q -> ring wait per CTA: by attention member index and by head
    qr = np.stack([(tr[:, s, 6].astype(np.int64) - tr[:, s, 5].astype(np.int64)) for s in att], 1) / 1e3
    dq = np.stack([(tr[:, s, 5].astype(np.int64) - tr[:, s, 1].astype(np.int64)) for s in att], 1) / 1e3
    wt = np.stack([(tr[:, s, 1].astype(np.int64) - tr[:, s, 0].astype(np.int64)) for s in att], 1) / 1e3
    ok = (tr[:, att[0], 5] > 0)
    cta = np.arange(tr.shape[0])
    for name, key in (("member", cta % 18), ("head", cta // 18)):
        print(f"q->ring by {name}:", " ".join(f"{k}:{np.median(qr[ok & (key == k)]):.2f}" for k in range(int(key[ok].max()) + 1)))
    print("attn dependency wait by head:", " ".join(f"{k}:{np.median(wt[ok & (cta // 18 == k)]):.2f}" for k in range(8)))
    print(f"q->ring percentiles 10/50/90: {np.percentile(qr[ok], 10):.2f} {np.percentile(qr[ok], 50):.2f} {np.percentile(qr[ok], 90):.2f}; "
          f"starve in QKV median {np.median(tr[ok, 0, 4]) / 1e3:.2f}")
