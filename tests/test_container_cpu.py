"""KVCZ header parsing and format errors (host-only paths; no GPU needed)."""
import numpy as np
import pytest

from golden_cases import load


def test_read_header_reference_file(tmp_path):
    from paper_2509_00579_b200 import QuantMode, read_header
    g = load("c_fp16_d128")
    p = tmp_path / "r.kvcz"
    p.write_bytes(g["kvcz"].tobytes())
    h = read_header(p)
    ctx, H, D = (int(x) for x in g["cfg"][:3])
    assert (h["head_num"], h["head_dim"]) == (H, D)
    assert h["context_len"] == ctx + int(g["cfg"][5])
    assert h["cfg_k"].mode is QuantMode.K_BLOCK and h["cfg_v"].mode is QuantMode.V_TOKEN
    assert h["dtype"] == np.dtype("<f2")


def test_read_header_kchannel(tmp_path):
    from paper_2509_00579_b200 import QuantMode, read_header
    g = load("c_kchannel")
    p = tmp_path / "r.kvcz"
    p.write_bytes(g["kvcz"].tobytes())
    assert read_header(p)["cfg_k"].mode is QuantMode.K_CHANNEL


def test_bad_magic_and_short_file(tmp_path):
    from paper_2509_00579_b200 import ContainerFormatError, read_header
    g = load("c_fp16_d128")
    raw = bytearray(g["kvcz"].tobytes())
    raw[0:4] = b"XXXX"
    p = tmp_path / "bad.kvcz"
    p.write_bytes(bytes(raw))
    with pytest.raises(ContainerFormatError):
        read_header(p)
    p.write_bytes(b"KVCZ")
    with pytest.raises(ContainerFormatError):
        read_header(p)


def test_cursor_bounds_and_config_codes():
    """The bounds-checked reader and the config / dtype code tables."""
    import struct
    from paper_2509_00579_b200 import ContainerFormatError, QuantConfig, QuantMode
    from paper_2509_00579_b200.container import (_QCFG, _Cursor, _config_fields, _config_from,
                                                 _dtype_code)
    cur = _Cursor(b"\x01\x02\x03")
    assert bytes(cur.take(2, "x")) == b"\x01\x02"
    with pytest.raises(ContainerFormatError):
        cur.take(2, "x")
    for cfg in (QuantConfig(QuantMode.K_BLOCK), QuantConfig(QuantMode.K_CHANNEL, 8, 0.3, 16),
                QuantConfig(QuantMode.V_TOKEN, 64, 1 / 255)):
        raw = _QCFG.pack(*_config_fields(cfg))
        assert _config_from(_QCFG.unpack(raw)) == cfg
    with pytest.raises(ContainerFormatError):
        _config_from((7, 64, 128, 0.05))
    assert _dtype_code(np.float16) == 0 and _dtype_code(np.float32) == 1
    with pytest.raises(ContainerFormatError):
        _dtype_code(np.float64)


def test_truncated_reference_file(tmp_path):
    from paper_2509_00579_b200 import ContainerFormatError, read_header
    g = load("c_fp16_d128")
    p = tmp_path / "t.kvcz"
    p.write_bytes(g["kvcz"].tobytes()[:40])
    with pytest.raises(ContainerFormatError):
        read_header(p)
