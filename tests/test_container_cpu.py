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


def test_arena_counters_from_blocks():
    """Counters rebuilt from block headers equal the reference's running totals."""
    from paper_2509_00579_b200.container import _arena_counters
    g = load("c_fp16_d128")
    c = _arena_counters(g["fin_k_arena"].tobytes(), g["fin_k_offsets"], 128)
    assert [c.payload_bits, c.payload_bytes] == g["fin_counters"][3:5].tolist()
    assert c.cursor == g["fin_k_arena"].size
