"""Multi-PROCESS tensor parallelism on one B200: two ranks
in two processes -- separate CUDA contexts, the peer's exchange buffers and
flags opened with cudaIpcOpenMemHandle, system-scope release / acquire flags
across the processes -- exactly the cross-process path bench.py takes with
one process per GPU, here with both ranks on GPU 0 run concurrently under an
MPS daemon (private pipe directory; skipped where MPS is unavailable).  The
gathered logits and the global greedy token of every step are checked
against the f64 oracle of the whole model fed the ranks' appended K/V rows."""
import os
import shutil
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


@pytest.fixture
def mps_env():
    ctl = shutil.which("nvidia-cuda-mps-control")
    if ctl is None:
        pytest.skip("nvidia-cuda-mps-control not available")
    d = tempfile.mkdtemp(prefix="ffb_mps_")
    env = dict(os.environ, CUDA_MPS_PIPE_DIRECTORY=os.path.join(d, "pipe"),
               CUDA_MPS_LOG_DIRECTORY=os.path.join(d, "log"))
    os.makedirs(env["CUDA_MPS_PIPE_DIRECTORY"])
    os.makedirs(env["CUDA_MPS_LOG_DIRECTORY"])
    r = subprocess.run([ctl, "-d"], env=env, capture_output=True, timeout=30)
    if r.returncode != 0:
        pytest.skip(f"MPS daemon did not start: {r.stderr.decode()[:200]}")
    try:
        yield env, d
    finally:
        subprocess.run([ctl], input=b"quit\n", env=env, capture_output=True, timeout=60)
        shutil.rmtree(d, ignore_errors=True)


def test_tp2_two_processes_cuda_ipc_matches_oracle(mps_env):
    env, d = mps_env
    init = os.path.join(d, "pg_init")
    outs = [os.path.join(d, f"rank{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "tp_mp_worker.py"), str(r), "2",
                               init, outs[r], str(N_STEPS)], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(2)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=300)[0].decode()[-3000:])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("TP worker timed out")
    assert all(p.returncode == 0 for p in procs), logs
    res = [np.load(o) for o in outs]
    np.testing.assert_array_equal(res[0]["greedy"], res[1]["greedy"])  # global argmax agrees
    st = O.OracleStore(CFG, 42, PREFILL + N_STEPS + 2)
    st.synthetic_prefill(PREFILL, 7)
    worst = 0.0
    for i in range(N_STEPS):
        logits = np.concatenate([r["logits"][i] for r in res])  # vocab slices in rank order
        k = np.concatenate([r["k"][i] for r in res], axis=2)     # kv heads in rank order
        v = np.concatenate([r["v"][i] for r in res], axis=2)
        want = st.forward([int(res[0]["tokens"][i])], PREFILL + i, k_app=k, v_app=v)[0]
        e = rel_err(logits, want)
        worst = max(worst, e)
        assert e < 2e-5, (i, e)
        assert int(res[0]["greedy"][i]) == int(np.argmax(want)), i
    print(f"TP2 across two processes (CUDA IPC, MPS): {N_STEPS} greedy steps identical, "
          f"max rel_err {worst:.2e}")


def test_bench_two_ranks_tp2_under_mps(mps_env):
    """bench.py's N > 1 contract (torchrun, one process per rank, the TP-2
    sharded model, max over ranks) on a one-GPU box: both ranks on the GPU
    under MPS; checks the JSON line, not the timing."""
    env, d = mps_env
    root = os.path.dirname(HERE)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                        "--model", "tiny", "--ctx", "192", "--steps", "5", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-2000:]
    import json
    line = json.loads(lines[-1])
    assert line["n_gpus"] == 2 and line["n_ranks_tp"] == 2 and line["value"] > 0
    assert line["config"]["parallelism"] == "tp2" and "shared_gpu" in line
