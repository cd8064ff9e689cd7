"""CPU checks of the tensor-parallel host logic: the shard
partition of every reference tensor (paper_2505_22758_b200.tp_shard, the host
restatement of runtime.cu's resolve) covers each weight exactly once, and the
multi-process wiring -- every rank all-gathers the others' exchange-buffer
blobs over torch.distributed -- runs with world size 2 on the gloo backend."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2505_22758_b200 as P
from gpu_helpers import to_model_cfg


@pytest.mark.parametrize("tp", [2, 4])
def test_shards_partition_every_tensor(tp):
    cfg = O.preset("tiny").replace(layers=1, n_kv_heads=4)
    st = O.OracleStore(cfg, 3, 4)
    mc = to_model_cfg(cfg)
    for name in P.tensor_names(mc):
        full = st.tensor(name)
        shards = [P.tp_shard(mc, name, full, r, tp) for r in range(tp)]
        np.testing.assert_array_equal(P.tp_unshard(mc, name, shards), full)
        if name.endswith(("wqkv", "wffn1", "wffn2t")) or name == "lm_head":
            assert sum(s.shape[0] for s in shards) == full.shape[0]
        if name.endswith("waout"):
            assert all(s.shape == (full.shape[0], full.shape[1] // tp) for s in shards)


def test_wqkv_shard_holds_its_heads_rows():
    cfg = P.model_preset("llama31_8b")
    rows = np.arange(cfg.qkv_rows)[:, None].astype(np.float32)
    s1 = P.tp_shard(cfg, "layer.0.wqkv", rows, 1, 2)[:, 0].astype(int)
    dh = cfg.d_head
    # rank 1 of 2: q heads 16..31, kv heads 4..7 (k then v)
    assert list(s1[:16 * dh]) == list(range(16 * dh, 32 * dh))
    assert list(s1[16 * dh:20 * dh]) == list(range(32 * dh + 4 * dh, 32 * dh + 8 * dh))
    assert list(s1[20 * dh:]) == list(range(40 * dh + 4 * dh, 40 * dh + 8 * dh))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = O.preset("tiny").replace(layers=1)
        mc = to_model_cfg(cfg)
        st = O.OracleStore(cfg, 11, 4)
        # every rank keeps its shard, the group reassembles the whole tensor
        ok = True
        for name in ["layer.0.wqkv", "layer.0.waout", "layer.0.wffn1", "layer.0.wffn2t", "lm_head"]:
            mine = P.tp_shard(mc, name, st.tensor(name), rank, world)
            got = [None] * world
            dist.all_gather_object(got, mine)
            ok &= np.array_equal(P.tp_unshard(mc, name, got), st.tensor(name))
        # the blob exchange of bench.py / INTEGRATION.md (fake blobs: no GPU)
        blob = bytes([rank]) * 64
        blobs = P.all_gather_tp_blobs(blob)
        ok &= blobs == [bytes([r]) * 64 for r in range(world)]
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_reassembly_and_blob_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
