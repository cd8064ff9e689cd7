"""CPU checks of the drop-in boundary (include/flashformer_b200.h):
the in-tree library loads, exports exactly the declared entry points, the
shape registry answers, and compute calls fail loudly without a B200."""
import ctypes as C
import os
import re

import pytest

import paper_2505_22758_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flashformer_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ffb_[a-z0-9_]+)\s*\(", src)))


def test_library_is_in_tree_and_loads():
    assert os.path.exists(P.LIB_PATH)
    assert P.LIB_PATH.startswith(ROOT)
    assert P.lib().ffb_version().decode().startswith("ffb200")


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 15
    lib = C.CDLL(P.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert re.search(r"sm_(?!100a)\d+", out) is None


@pytest.mark.parametrize("name", ["llama31_8b-toy", "tiny", "llama32_1b", "llama31_8b"])
def test_compiled_shapes_supported(name):
    assert P.DecodeModel.supported(P.model_preset(name))


def test_unsupported_shape_reported():
    cfg = P.model_preset("llama31_8b").replace(d_inter=12288)
    assert not P.DecodeModel.supported(cfg)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.DeviceError, match="no CPU fallback"):
        P.DecodeModel(P.model_preset("tiny"), 64)


def test_validation_mirrors_reference():
    with pytest.raises(P.ValidationError, match="GQA"):
        P.DecodeModel(P.model_preset("tiny").replace(n_kv_heads=3), 64)
    with pytest.raises(P.ValidationError, match="d_model must equal"):
        P.DecodeModel(P.model_preset("tiny").replace(d_head=32), 64)


def test_byte_accounting():
    cfg = P.model_preset("llama31_8b")
    assert cfg.streamed_weight_bytes() == 32 * 436207616 + 1050673152  # test_store.cpp:73-86
    assert cfg.replace(quant_bits=4).streamed_weight_bytes() == 3986849792


def test_nccl_unique_id_without_gpu():
    """The host-NCCL baseline loads NCCL at run time (dlopen); making the
    communicator id needs no GPU."""
    import paper_2505_22758_b200 as P
    a, b = P.nccl_unique_id(), P.nccl_unique_id()
    assert len(a) == 128 and a != b
