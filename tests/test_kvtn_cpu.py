"""KVTN tensor files (reference tensor_io.py:100-143): our writer produces the
reference writer's bytes (tests/golden/kvtn.npz, from make_golden.py
kvtn_cases), our reader inverts them, and malformed files raise
TensorFormatError like the reference's tests/test_tensor_io.py cases."""
import os

import numpy as np
import pytest

import paper_2509_00579_b200 as kv

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(HERE, "golden", "kvtn.npz"))


@pytest.mark.parametrize("nm", ["f16", "f32"])
def test_bytes_equal_reference(tmp_path, g, nm):
    path = tmp_path / "t.kvtn"
    kv.write_tensor(kv.CacheTensor(g[nm + "_values"]), path)
    assert path.read_bytes() == g[nm + "_file"].tobytes()
    path.write_bytes(g[nm + "_file"].tobytes())
    back = kv.read_tensor(path)
    assert back.dtype == g[nm + "_values"].dtype
    assert np.array_equal(back.values.view(np.uint8), g[nm + "_values"].view(np.uint8))


def test_torch_values(tmp_path, g):
    import torch
    path = tmp_path / "t.kvtn"
    kv.write_tensor(kv.CacheTensor(torch.from_numpy(g["f32_values"])), path)
    assert path.read_bytes() == g["f32_file"].tobytes()


@pytest.mark.parametrize("edit,match", [
    (lambda b: b"XXXX" + b[4:], "magic"),
    (lambda b: b[:-2], "truncated"),
    (lambda b: b + b"\x00", "trailing"),
    (lambda b: b[:4] + b"\x02" + b[5:], "version"),
    (lambda b: b[:5] + b"\x07" + b[6:], "dtype"),
    (lambda b: b[:10], "header"),
    (lambda b: b[:6] + (0).to_bytes(8, "little") + b[14:], "positive"),
])
def test_malformed(tmp_path, g, edit, match):
    path = tmp_path / "t.kvtn"
    path.write_bytes(edit(g["f32_file"].tobytes()))
    with pytest.raises(kv.TensorFormatError, match=match):
        kv.read_tensor(path)


def test_nan_payload(tmp_path):
    path = tmp_path / "t.kvtn"
    kv.write_tensor(kv.CacheTensor(np.zeros((1, 1, 2), np.float32)), path)
    b = bytearray(path.read_bytes())
    b[-4:] = np.array([np.nan], np.float32).tobytes()
    path.write_bytes(bytes(b))
    with pytest.raises(kv.TensorFormatError, match="NaN"):
        kv.read_tensor(path)
