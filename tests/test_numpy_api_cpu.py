"""The kvpack facade with host outputs (paper_2509_00579_b200.numpy_api):
module layout and the tensor -> numpy conversion, without a GPU."""
import sys

import numpy as np
import torch

from paper_2509_00579_b200 import numpy_api


def test_install_registers_modules():
    top = numpy_api.install()
    try:
        import kvpack
        import kvpack.codec
        assert kvpack is top
        assert kvpack.codec.iter_decoded_blocks is not None
        assert kvpack.LayerCacheState is numpy_api.LayerCacheState
        assert kvpack.bench.FUSED_FASTER == "fused-faster"
    finally:
        for k in [k for k in sys.modules if k == "kvpack" or k.startswith("kvpack.")]:
            del sys.modules[k]


def test_to_host_converts_nested_results():
    qb = numpy_api.QuantizedBlock(codes=torch.arange(6, dtype=torch.uint8).reshape(2, 3),
                                  unit_mins=torch.zeros(3), unit_scales=torch.ones(3),
                                  block_index=4, head_index=0, ctx_start=0)
    out = numpy_api.to_host((qb, [torch.ones(2)], 7))
    assert isinstance(out, tuple) and out[2] == 7
    assert isinstance(out[0].codes, np.ndarray) and out[0].codes.dtype == np.uint8
    assert np.array_equal(out[0].codes, np.arange(6, dtype=np.uint8).reshape(2, 3))
    assert isinstance(out[1][0], np.ndarray)
    cb = numpy_api.CompressedBlock(block_index=1, slice_bit_counts=torch.tensor([3, 5]),
                                   unit_mins=torch.zeros(2), unit_scales=torch.ones(2),
                                   payload=torch.tensor([1, 2], dtype=torch.uint8))
    h = numpy_api.to_host(cb)
    assert h.payload == b"\x01\x02" and h.total_bits == 8
