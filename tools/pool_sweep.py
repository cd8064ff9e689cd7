"""Developer sweep of the GLU work-pool knobs (device time per step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_22758_b200 import DecodeModel, model_preset
name = sys.argv[1] if len(sys.argv) > 1 else "llama31_8b"
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = model_preset(name)
m = DecodeModel(cfg, ctx + 8); m.init_synthetic(1)
s = torch.cuda.Stream(); tok = torch.full((1,), 17, dtype=torch.int64, device="cuda")
def loop(n):
    for _ in range(n):
        for l in range(cfg.layers): m.set_length(l, ctx)
        m.step_device(tok.data_ptr(), ctx, 0, 0, s.cuda_stream)
for pm, ct in [(0, 4), (60, 4), (120, 4), (200, 4), (120, 8), (200, 8), (300, 4)]:
    m.set_option("glu_pool_permille", pm); m.set_option("glu_pool_chunk", ct)
    loop(5); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s); loop(50); e1.record(s); torch.cuda.synchronize()
    print(f"{name} pool {pm}/1000 chunk {ct}: {e0.elapsed_time(e1) / 50:.4f} ms/step", flush=True)
