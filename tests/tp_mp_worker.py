"""One rank of a multi-PROCESS tensor-parallel group (test helper for
tests/test_gpu_tp_mp.py): its own process, its own CUDA context, the peer's
exchange buffers opened through CUDA IPC (ffb_tp_connect), the blobs
all-gathered over a gloo process group -- the wiring bench.py uses across
GPUs, here with every rank on GPU 0 under MPS so the persistent kernels of
the two processes run side by side.

    python tp_mp_worker.py RANK WORLD INIT_FILE OUT_NPZ N_STEPS [ipc|nccl]

`nccl`: every rank on its own GPU (device = rank), the host-NCCL multi-
kernel baseline (RunMode.BASELINE_NCCL: per-stage launches, ncclAllReduce of
the residual deltas between them) instead of the in-kernel exchange.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as O  # noqa: E402
from gpu_helpers import to_model_cfg  # noqa: E402
from paper_2505_22758_b200 import (DecodeModel, RunMode, all_gather_tp_blobs,  # noqa: E402
                                   broadcast_nccl_id)

CFG = O.preset("tiny").replace(layers=2)
PREFILL = 40


def main():
    rank, world, init_file, out, n_steps = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3],
                                            sys.argv[4], int(sys.argv[5]))
    mode = sys.argv[6] if len(sys.argv) > 6 else "ipc"
    dev = rank if mode == "nccl" else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    st = O.OracleStore(CFG, 42, PREFILL + n_steps + 2)
    st.synthetic_prefill(PREFILL, 7)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    m = DecodeModel(to_model_cfg(CFG), st.max_seq_len, device=dev, tp_rank=rank, tp_size=world,
                    grid=sms if mode == "nccl" else sms // world)
    m.upload_store(st)
    k, v = st.kv()
    m.kv_import(k, v, PREFILL)
    if mode == "nccl":
        m.tp_nccl_init(broadcast_nccl_id())
        m.set_mode(RunMode.BASELINE_NCCL)
    else:
        m.tp_connect(all_gather_tp_blobs(m.tp_blob()))
    dist.barrier()
    tok, rec = 17, {"logits": [], "greedy": [], "k": [], "v": [], "tokens": []}
    for i in range(n_steps):
        rec["tokens"].append(tok)
        logits, greedy = m.step([tok], PREFILL + i)
        ka, va = m.kv_export(PREFILL + i, 1)
        rec["logits"].append(logits[0])
        rec["greedy"].append(int(greedy[0]))
        rec["k"].append(ka[:, :, :, 0])
        rec["v"].append(va[:, :, :, 0])
        tok = int(greedy[0])
    dist.barrier()
    np.savez(out, **{key: np.asarray(val) for key, val in rec.items()})
    m.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
