"""The host-NCCL multi-kernel tensor-parallel baseline (RunMode.BASELINE_NCCL,
SURVEY.md §8(e) "Baseline: host ncclAllReduce between per-layer kernels"):
two ranks, one process and one GPU each, every stage its own launch, the two
per-layer residual sums as ncclAllReduce on the launch stream and the argmax
as ncclAllGather.  Checked like the in-kernel exchange (tests/
test_gpu_tp_mp.py): gathered logits and the global greedy token of every
step against the f64 oracle fed the ranks' appended K/V rows.  Needs two
GPUs (NCCL does not run two ranks on one device)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import oracle as O
from gpu_helpers import rel_err

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CFG = O.preset("tiny").replace(layers=2)
PREFILL = 40
N_STEPS = 6


def test_tp2_host_nccl_baseline_matches_oracle():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one NCCL rank per device)")
    d = tempfile.mkdtemp(prefix="ffb_nccl_")
    init = os.path.join(d, "pg_init")
    outs = [os.path.join(d, f"rank{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "tp_mp_worker.py"), str(r), "2",
                               init, outs[r], str(N_STEPS), "nccl"], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(2)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=300)[0].decode()[-3000:])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("NCCL TP worker timed out")
    assert all(p.returncode == 0 for p in procs), logs
    res = [np.load(o) for o in outs]
    np.testing.assert_array_equal(res[0]["greedy"], res[1]["greedy"])
    st = O.OracleStore(CFG, 42, PREFILL + N_STEPS + 2)
    st.synthetic_prefill(PREFILL, 7)
    for i in range(N_STEPS):
        logits = np.concatenate([r["logits"][i] for r in res])
        k = np.concatenate([r["k"][i] for r in res], axis=2)
        v = np.concatenate([r["v"][i] for r in res], axis=2)
        want = st.forward([int(res[0]["tokens"][i])], PREFILL + i, k_app=k, v_app=v)[0]
        assert rel_err(logits, want) < 2e-5, i
        assert int(res[0]["greedy"][i]) == int(np.argmax(want)), i
