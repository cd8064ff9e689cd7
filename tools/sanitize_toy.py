"""Driver for compute-sanitizer (racecheck / synccheck / memcheck): the toy
decoder (llama31_8b-toy) for two decode steps in each run mode, checked
against the CPU oracle.  Run with a library built with a long spin watchdog
(tools/build_variant.sh san "-DFFB_SPIN_NS=...") because the sanitizer slows
every CTA by orders of magnitude while the others spin on its flags."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle as O
from gpu_helpers import device_from_store, rel_err
from paper_2505_22758_b200 import RunMode

# optional: QB to run the 8B-width int4 / int8 shape (1 layer) -- the
# integer-MMA tensor-core GEMV (decode_kernel.cuh tc_slot) only exists there
QB = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = O.preset("llama31_8b-toy")
modes = (RunMode.FUSED_OVERLAP, RunMode.FUSED, RunMode.BASELINE)
if QB:
    cfg = O.preset("llama31_8b").replace(layers=1, vocab_size=4096, quant_bits=QB)
    modes = (RunMode.FUSED_OVERLAP,)
for mode in modes:
    st = O.OracleStore(cfg, 42, 40)
    st.synthetic_prefill(9, 7)
    with device_from_store(st) as m:
        m.set_mode(mode)
        for i, tok in enumerate((17, 3)):
            logits, greedy = m.step([tok], 9 + i)
            want = st.forward([tok], 9 + i)
            err = rel_err(logits[0], want[0])
            print(f"mode {int(mode)} step {i}: rel_err {err:.2e} greedy {int(greedy[0])}", flush=True)
            assert err < 5e-4 and int(greedy[0]) == int(np.argmax(want[0]))
print("sanitize_toy ok")
