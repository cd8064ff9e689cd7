"""Store files, device images and bulk KV export through the C-ABI
(§8(b) kv import/export):

* ffb_load_store reads the reference's "FSTW" v1 container (the restatement
  writes files byte-identical to fusesim::save_store, tests/test_oracle.py)
  and gives the same device state as uploading the TensorStore tensor by
  tensor (bit-identical logits);
* ffb_save_image / ffb_load_image round-trip the packed device weights
  (bf16, int4, batch-16 chunk-major, a TP shard) and refuse an image of
  another shape or shard;
* ffb_kv_export returns the reference layout [B][L][Hkv][n][dh] and equals
  per-position ffb_kv_get (KVCache::k_at / v_at, tensor_store.hpp:109-125).
"""
import numpy as np
import pytest

import oracle as O
from gpu_helpers import device_from_store, to_model_cfg
from paper_2505_22758_b200 import (DecodeModel, TPGroup, UsageError, ValidationError)

pytestmark = pytest.mark.gpu

TOY = O.preset("llama31_8b-toy")


@pytest.mark.parametrize("quant", [0, 4])
def test_load_store_file_equals_upload(tmp_path, quant):
    st = O.OracleStore(TOY.replace(quant_bits=quant), 11, 40)
    st.synthetic_prefill(30, 3)
    path = str(tmp_path / "store.fstw")
    st.save(path)
    with device_from_store(st) as a:
        want = a.forward([9], 30)
    with DecodeModel(to_model_cfg(st.cfg), 40) as b:
        b.load_store(path)
        k, v = st.kv()
        b.kv_import(k, v, 30)
        got = b.forward([9], 30)
        assert b.info()["quant_inexact_groups"] == 0
    np.testing.assert_array_equal(got, want)


def test_load_store_rejects_other_shapes_and_bad_files(tmp_path):
    st = O.OracleStore(TOY, 11, 8)
    path = tmp_path / "store.fstw"
    st.save(str(path))
    with DecodeModel(to_model_cfg(TOY.replace(layers=2)), 8) as m:
        with pytest.raises(ValidationError, match="different model shape"):
            m.load_store(str(path))
    with DecodeModel(to_model_cfg(TOY), 8) as m:
        bad = tmp_path / "bad.fstw"
        bad.write_bytes(b"\0" * 16)
        with pytest.raises(UsageError, match="bad magic"):
            m.load_store(str(bad))
        bad.write_bytes(path.read_bytes()[:4096])
        with pytest.raises(UsageError, match="truncated"):
            m.load_store(str(bad))
        with pytest.raises(UsageError, match="cannot open"):
            m.load_store(str(tmp_path / "missing"))


@pytest.mark.parametrize("quant,batch", [(0, 1), (4, 1), (8, 1), (0, 16)])
def test_device_image_round_trip(tmp_path, quant, batch):
    cfg = TOY.replace(quant_bits=quant, batch=batch)
    st = O.OracleStore(cfg, 5, 24)
    st.synthetic_prefill(20, 2)
    toks = list(range(3, 3 + batch))
    path = str(tmp_path / "img.bin")
    with device_from_store(st) as a:
        a.save_image(path)
        want = a.forward(toks, 20)
    with DecodeModel(to_model_cfg(cfg), 24) as b:
        b.load_image(path)
        k, v = st.kv()
        b.kv_import(k, v, 20)
        np.testing.assert_array_equal(b.forward(toks, 20), want)
    # another specialisation refuses the image
    with DecodeModel(to_model_cfg(cfg.replace(quant_bits=4 if quant == 0 else 0, batch=1)), 24) as c:
        with pytest.raises(ValidationError):
            c.load_image(path)


def test_device_image_of_a_tp_shard(tmp_path):
    cfg = O.preset("tiny").replace(layers=2)
    st = O.OracleStore(cfg, 42, 24)
    st.synthetic_prefill(16, 7)
    with TPGroup(to_model_cfg(cfg), 24, 2) as g:
        g.upload_store(st)
        k, v = st.kv()
        g.kv_import(k, v, 16)
        paths = [str(tmp_path / f"r{r}.img") for r in range(2)]
        for r, m in enumerate(g.ranks):
            m.save_image(paths[r])
        want = g.forward([17], 16)
    with TPGroup(to_model_cfg(cfg), 24, 2) as g:
        with pytest.raises(ValidationError):  # rank 1's image on rank 0
            g.ranks[0].load_image(paths[1])
        for r, m in enumerate(g.ranks):
            m.load_image(paths[r])
        g.kv_import(k, v, 16)
        np.testing.assert_array_equal(g.forward([17], 16), want)


def test_kv_export_matches_kv_get_and_reference_layout():
    cfg = TOY.replace(batch=2)
    st = O.OracleStore(cfg, 3, 40)
    st.synthetic_prefill(33, 9)
    with device_from_store(st) as m:
        k, v = m.kv_export(0, 33)
        K, V = st.kv()
        np.testing.assert_array_equal(k, K[:, :, :, :33])
        np.testing.assert_array_equal(v, V[:, :, :, :33])
        m.forward([1, 2], 33)
        ka, va = m.kv_export(33, 1)
        for b in range(2):
            for l in range(cfg.layers):
                for h in range(cfg.n_kv_heads):
                    kg, vg = m.kv_get(b, l, h, 33)
                    np.testing.assert_array_equal(ka[b, l, h, 0], kg)
                    np.testing.assert_array_equal(va[b, l, h, 0], vg)
        with pytest.raises(ValidationError):
            m.kv_export(39, 5)


def test_kv_export_chunked_path_large_block():
    """More than the 32 MiB staging block: the per-(row, layer) chunked path."""
    cfg = O.preset("llama32_1b").replace(layers=2, vocab_size=512)
    st = O.OracleStore(cfg, 3, 8200)
    k, v = st.kv()
    rng = np.random.default_rng(0)
    k[:] = rng.standard_normal(k.shape, dtype=np.float32).astype(np.float32)
    v[:] = -k
    with device_from_store(st, max_seq_len=8200) as m:
        m.kv_import(k, v, 8200)
        ke, ve = m.kv_export(0, 8200)
        kr = k.view(np.uint32)
        kb = (((kr.astype(np.uint64) + 0x7FFF + ((kr >> 16) & 1)) >> 16) << 16).astype(np.uint32)
        np.testing.assert_array_equal(ke, kb.view(np.float32))
        np.testing.assert_array_equal(ve, -ke)


def test_device_token_out_of_range_latches_validation_error():
    """ADVICE: device-resident ids are not checked before the launch; an
    out-of-range id reads row 0 and is reported by the next ffb_sync /
    ffb_decode_step like reference_forward's ValidationError."""
    import torch
    st = O.OracleStore(TOY, 5, 16)
    st.synthetic_prefill(4, 1)
    with device_from_store(st) as m:
        bad = torch.tensor([TOY.vocab_size + 5], dtype=torch.int64, device="cuda:0")
        torch.cuda.synchronize()
        m.step_device(bad.data_ptr(), 4)
        with pytest.raises(ValidationError, match="out of range"):
            m.sync()
        m.sync()  # latch cleared
        good = torch.tensor([3], dtype=torch.int64, device="cuda:0")
        torch.cuda.synchronize()
        m.step_device(good.data_ptr(), 5)
        m.sync()
        m.step([3], 6)  # host path still validates ids itself
        with pytest.raises(ValidationError, match="out of range"):
            m.step([TOY.vocab_size], 7)
