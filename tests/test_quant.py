"""CPU checks of the weight-only quantization packer (ffb_pack_quant_rows,
the host side of the int4 / int8 weight formats, quant.hpp:17-60).

The reference snaps its weights to the int4 g128 grid and discards the codes
(tensor_store.hpp:275-287); the packer must re-derive (code, scale, zero) so
that (code - zero) * scale reproduces every stored f32 value bit for bit.
The int8 format is the reference's formula with 255 levels (an extension the
reference does not pin; the C oracle restates it)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_2505_22758_b200 as P


@pytest.mark.parametrize("qb", [4, 8])
@pytest.mark.parametrize("preset", ["llama31_8b-toy", "tiny"])
def test_packer_reproduces_reference_grid_bit_exact(preset, qb):
    cfg = O.preset(preset).replace(quant_bits=qb, layers=1)
    st = O.OracleStore(cfg, 42, 8)
    for name in ["layer.0.wqkv", "layer.0.waout", "layer.0.wffn1", "layer.0.wffn2t", "lm_head"]:
        w = st.tensor(name)
        packed, inexact = P.pack_quant_rows(w, qb)
        assert inexact == 0, name
        assert packed.shape == (w.shape[0], P.lib().ffb_quant_row_bytes(w.shape[1], qb))
        np.testing.assert_array_equal(P.unpack_quant_rows(packed, w.shape[1], qb), w)


@pytest.mark.parametrize("qb", [4, 8])
def test_tensor_core_code_order_round_trip(qb):
    """Layout 1 (the mma.sync A-fragment order) stores every code exactly once
    and reproduces the same f32 weights as the plain order."""
    pos = P.tc_code_positions(qb)
    assert sorted(pos.tolist()) == list(range(128))
    cfg = O.preset("llama31_8b").replace(quant_bits=qb, layers=1, d_inter=256, vocab_size=64)
    st = O.OracleStore(cfg, 42, 8)
    w = st.tensor("lm_head")
    plain, ie0 = P.pack_quant_rows(w, qb, 0)
    tc, ie1 = P.pack_quant_rows(w, qb, 1)
    assert ie0 == ie1 == 0
    assert not np.array_equal(plain, tc)
    np.testing.assert_array_equal(P.unpack_quant_rows(tc, w.shape[1], qb, 1), w)
    np.testing.assert_array_equal(plain[:, w.shape[1] // (2 if qb == 4 else 1):],
                                  tc[:, w.shape[1] // (2 if qb == 4 else 1):])


def test_row_bytes_match_the_device_format():
    # codes + f32 scale + u8 zero per group of 128, padded to 16 bytes
    assert P.lib().ffb_quant_row_bytes(4096, 4) == 2048 + 32 * 5
    assert P.lib().ffb_quant_row_bytes(4096, 8) == 4096 + 32 * 5
    assert P.lib().ffb_quant_row_bytes(256, 4) == 144
    assert P.lib().ffb_quant_row_bytes(4096, 0) == 8192
    assert P.lib().ffb_quant_row_bytes(100, 4) == -1
    assert P.lib().ffb_quant_row_bytes(4096, 3) == -1


def test_codes_scales_zeros_follow_quantize_group():
    """The packed group equals fo_quantize_group's (codes, scale, zero) for a
    group on the grid; nibbles are little-endian within a byte."""
    rng = np.random.default_rng(3)
    vals = rng.standard_normal(128).astype(np.float32) * 0.05
    deq = np.empty_like(vals)
    codes = np.empty(128, np.uint8)
    s, z = C.c_float(), C.c_float()
    O.lib().fo_quantize_group(vals.ctypes.data_as(C.POINTER(C.c_float)), 128, 15,
                              codes.ctypes.data_as(C.POINTER(C.c_uint8)), C.byref(s),
                              C.byref(z), deq.ctypes.data_as(C.POINTER(C.c_float)))
    s, z = s.value, z.value
    packed, inexact = P.pack_quant_rows(deq[None, :], 4)
    assert inexact == 0
    row = packed[0]
    np.testing.assert_array_equal(row[:64] & 0xF, codes[0::2])
    np.testing.assert_array_equal(row[:64] >> 4, codes[1::2])
    assert row[64:68].view(np.float32)[0] == np.float32(s)
    assert row[68] == int(z)


def test_off_grid_values_are_packed_lossily_and_counted():
    rng = np.random.default_rng(0)
    w = rng.standard_normal((3, 256)).astype(np.float32)
    for qb, tol in ((4, 0.25), (8, 0.02)):
        packed, inexact = P.pack_quant_rows(w, qb)
        assert inexact == 6
        assert np.abs(P.unpack_quant_rows(packed, 256, qb) - w).max() < tol
    zeros = np.zeros((2, 128), np.float32)
    packed, inexact = P.pack_quant_rows(zeros, 4)
    assert inexact == 0 and not P.unpack_quant_rows(packed, 128, 4).any()
