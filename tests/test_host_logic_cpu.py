"""Host-side logic added for the device decode loop and the drop-in API that
needs no GPU: the arenas' max-extent bound (stage sizes without
synchronising), 1.25x growth, the report rows / CSV of the simulation API,
and metadata_overhead."""
import csv

import numpy as np
import pytest
import torch

from paper_2509_00579_b200 import codec


@pytest.fixture
def cpu_pool(monkeypatch):
    p = codec._SlabPool(torch.device("cpu"))
    p.slab_bytes = 4 << 20
    monkeypatch.setitem(codec._POOLS, ("cpu", None), p)
    return p


def test_max_extent_bound_is_conservative_until_read(cpu_pool):
    a = codec.DeviceArena(torch.device("cpu"), None, initial_bytes=1 << 12, initial_blocks=4)
    assert a.max_extent_bound() == 0
    # blocks appended on the device: their worst case bounds the stage size
    a.note_append(3, 3 * 7000, block_worst=7000)
    assert a.max_extent_bound() == 7000
    # a counters read makes the bound exact again (here: what the "device" wrote)
    cnt = codec._lib.ArenaCounters(cursor=9000, n_blocks=3, payload_bits=0, payload_bytes=0,
                                   max_extent=5200, err=0)
    a._counters.copy_(torch.frombuffer(bytearray(bytes(cnt)), dtype=torch.uint8))
    assert a.counters().max_extent == 5200
    assert a.max_extent_bound() == 5200
    a.note_append(1, 6000, block_worst=6000)
    assert a.max_extent_bound() == 6000


def test_arena_growth_is_1_25x(cpu_pool):
    a = codec.DeviceArena(torch.device("cpu"), None, initial_bytes=100_000, initial_blocks=4)
    cap0 = a.alloc_capacity
    a.reserve(1, cap0 + 10)          # just past the allocation
    assert cap0 + 10 <= a.alloc_capacity <= int(1.26 * cap0) + 64
    a.reserve(2, 10 * cap0)          # a large request is served exactly
    assert a.alloc_capacity >= 10 * cap0


def test_bench_rows_and_csv(tmp_path):
    from paper_2509_00579_b200 import (BenchRow, QuantConfig, QuantMode, config_label,
                                       equivalent_decompression_throughput, write_csv)
    ck, cv = QuantConfig(QuantMode.K_BLOCK), QuantConfig(QuantMode.V_TOKEN)
    label = config_label(ck, cv, 8, 128)
    assert label == "mode=kblock;block=64;buffer=128;rsk=0.05;rsv=0.15;heads=8;dim=128"
    rows = [BenchRow(label, 4096, 1000, 200, 50, 4.0, 2.5),
            BenchRow(label, 4096, 1000, 200, 50, 4.0, 2.5, fused_time=0.001,
                     multistage_time=0.004, reference_matvec_time=0.002,
                     equivalent_decompression_throughput=equivalent_decompression_throughput(
                         1000, 0.001, 0.002))]
    p = tmp_path / "r.csv"
    write_csv(rows, p)
    got = list(csv.reader(open(p)))
    assert got[0][0] == "config" and got[0][-1] == "equivalent_decompression_throughput"
    assert got[1][7:] == ["", "", "", ""]
    assert got[2][-1] == "fused-faster" and got[2][7] == "0.001"
    assert equivalent_decompression_throughput(1000, 0.003, 0.001) == pytest.approx(500000.0)


def test_metadata_overhead_arithmetic():
    from paper_2509_00579_b200 import CodecError, metadata_overhead

    class B:
        def __init__(self, n, bits):
            self.n_slices, self.total_bits = n, bits
    comp, orig = metadata_overhead([B(64, 64 * 256), B(64, 64 * 256)], 128)
    assert comp == pytest.approx(16 / 256) and orig == pytest.approx(1 / 128)
    with pytest.raises(CodecError):
        metadata_overhead([], 128)
