"""Quantisation configuration + block quantisation on the device.

Mirrors the reference's quantizer.py (QuantMode :37-47, QuantConfig :56-85,
QuantizedBlock :88-104, quantize_block :162-209, dequantize_block :212-223);
the arithmetic runs in the sm_100a kernel ``kvc_quantize`` (store.cu), which
is bit-exact with the reference's binary64 numpy code.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from .errors import CodecError, ConfigError

MIN_REL_SCALE = 1.0 / 255.0
DEFAULT_REL_SCALE = {"kblock": 0.05, "kchannel": 0.25, "vtoken": 0.15}


class QuantMode(enum.Enum):
    K_BLOCK = "kblock"
    K_CHANNEL = "kchannel"
    V_TOKEN = "vtoken"

    @property
    def is_key(self) -> bool:
        return self in (QuantMode.K_BLOCK, QuantMode.K_CHANNEL)

    @property
    def abi(self) -> int:
        return {QuantMode.K_BLOCK: _lib.KVC_K_BLOCK, QuantMode.V_TOKEN: _lib.KVC_V_TOKEN,
                QuantMode.K_CHANNEL: _lib.KVC_K_CHANNEL}[self]


class QuantUnitMeta(NamedTuple):
    min_value: float
    scale: float


@dataclass(frozen=True)
class QuantConfig:
    """Same fields, defaults and validation as quantizer.py:56-85."""

    mode: QuantMode
    block_size: int = 64
    rel_quant_scale: Optional[float] = None
    buffer_size: Optional[int] = None

    def __post_init__(self):
        if self.rel_quant_scale is None:
            object.__setattr__(self, "rel_quant_scale", DEFAULT_REL_SCALE[self.mode.value])
        if self.buffer_size is None:
            object.__setattr__(self, "buffer_size", 2 * self.block_size)
        if self.block_size < 1:
            raise ConfigError("block_size must be positive")
        if not MIN_REL_SCALE <= self.rel_quant_scale <= 1.0:
            raise ConfigError(
                f"rel_quant_scale {self.rel_quant_scale} outside [1/255, 1]; "
                "codes must fit an unsigned 8-bit integer")
        if self.buffer_size < self.block_size:
            raise ConfigError("buffer_size must be at least block_size")
        if self.buffer_size % self.block_size != 0:
            raise ConfigError("buffer_size must be a multiple of block_size")

    @property
    def max_code(self) -> int:
        return int(math.ceil(1.0 / self.rel_quant_scale))


@dataclass(frozen=True)
class QuantizedBlock:
    codes: torch.Tensor        # (block_size, head_dim) uint8, device
    unit_mins: torch.Tensor    # (n_units,) float32
    unit_scales: torch.Tensor  # (n_units,) float32
    block_index: int
    head_index: int
    ctx_start: int


def as_device_tensor(x, device=None) -> torch.Tensor:
    """f16/f32 torch tensor on the CUDA device (numpy input is copied over)."""
    if not isinstance(x, torch.Tensor):  # numpy arrays, nested lists
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    if x.dtype not in (torch.float16, torch.float32):
        x = x.to(torch.float32)
    dev = torch.device(device) if device is not None else (
        x.device if x.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    return x.to(dev).contiguous()


def dtype_code(t: torch.Tensor) -> int:
    return _lib.KVC_F16 if t.dtype == torch.float16 else _lib.KVC_F32


def quantize_tokens(x: torch.Tensor, n_chunks: int, head_num: int, head_dim: int, bs: int,
                    mode: QuantMode, rel: float, hist: Optional[torch.Tensor] = None,
                    k_ranges: Optional[torch.Tensor] = None):
    """Device quantisation of x[t, h, :] for t < n_chunks*bs, blocks in
    chunk-major / head-minor order (kvcache.py:242-268).  Returns (codes
    [nb, bs, D] u8, metas [nb, n_units, 2] f32).  K_CHANNEL takes the
    whole-context ranges as a device f32 tensor [2, H, D]."""
    if mode is QuantMode.K_CHANNEL:
        if k_ranges is None:
            raise ConfigError("K_CHANNEL quantization requires whole-context channel_ranges")
        k_ranges = k_ranges.to(x.device, torch.float32).contiguous()
        if tuple(k_ranges.shape) != (2, head_num, head_dim):
            raise ConfigError("channel ranges must have shape (2, head_num, head_dim)")
    nb = n_chunks * head_num
    n_units = bs if mode is QuantMode.V_TOKEN else head_dim
    codes = torch.empty((nb, bs, head_dim), dtype=torch.uint8, device=x.device)
    metas = torch.empty((nb, n_units, 2), dtype=torch.float32, device=x.device)
    if nb:
        st = _lib.lib().kvc_quantize(
            x.data_ptr(), dtype_code(x), head_num * head_dim, n_chunks, head_num, head_dim, bs,
            mode.abi, float(rel), k_ranges.data_ptr() if mode is QuantMode.K_CHANNEL else None,
            codes.data_ptr(), metas.data_ptr(),
            hist.data_ptr() if hist is not None else None,
            torch.cuda.current_stream(x.device).cuda_stream)
        _lib.check(st, "kvc_quantize")
    return codes, metas


def quantize_unit(values, rel_quant_scale: float, device=None):
    """quantizer.py:144-160 on the device: one unit (a flat group of values
    sharing min/scale), binary64 arithmetic on the float64 values ->
    (codes uint8 device tensor, QuantUnitMeta(min, scale))."""
    if isinstance(values, torch.Tensor):
        v = values.detach().reshape(-1)
        dev = torch.device(device) if device is not None else (
            v.device if v.is_cuda else torch.device("cuda", torch.cuda.current_device()))
        v = v.to(dev, torch.float64).contiguous()
    else:
        a = np.asarray(values, dtype=np.float64).reshape(-1)
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        v = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if v.numel() == 0:
        raise CodecError("cannot quantize an empty unit")
    if not bool(torch.isfinite(v).all()):
        raise CodecError("non-finite values in quantization unit")
    if not MIN_REL_SCALE <= rel_quant_scale <= 1.0:
        raise ConfigError(f"rel_quant_scale {rel_quant_scale} outside [1/255, 1]")
    n = v.numel()
    codes = torch.empty(n, dtype=torch.uint8, device=dev)
    meta = torch.empty(2, dtype=torch.float32, device=dev)
    # the unit as one V_TOKEN row: min/max over the row, one (min, scale)
    st = _lib.lib().kvc_quantize(v.data_ptr(), _lib.KVC_F64, n, 1, 1, n, 1, _lib.KVC_V_TOKEN,
                                 float(rel_quant_scale), None, codes.data_ptr(), meta.data_ptr(),
                                 None, torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(st, "quantize_unit")
    m = meta.cpu().numpy()
    return codes, QuantUnitMeta(float(m[0]), float(m[1]))


def quantize_block(block, mode: QuantMode, cfg: QuantConfig, head_index: int, ctx_start: int,
                   head_num: int, channel_ranges=None, device=None) -> QuantizedBlock:
    """quantizer.py:162-209 on the device."""
    x = as_device_tensor(block, device)
    if x.ndim != 2 or x.shape[0] != cfg.block_size:
        raise CodecError(f"block shape {tuple(x.shape)} does not match block_size {cfg.block_size}")
    if mode is not cfg.mode:
        raise ConfigError(f"mode {mode} does not match config mode {cfg.mode}")
    if ctx_start % cfg.block_size != 0:
        raise CodecError("ctx_start must be a multiple of block_size")
    if not 0 <= head_index < head_num:
        raise CodecError("head_index out of range")
    if mode is QuantMode.K_CHANNEL and channel_ranges is None:
        raise ConfigError("K_CHANNEL quantization requires whole-context channel_ranges")
    D = x.shape[1]
    ranges = None
    if mode is QuantMode.K_CHANNEL:  # quantizer.py:191-197: (mins, maxs) of length head_dim
        ranges = torch.stack([torch.as_tensor(np.asarray(r, np.float32)) if not isinstance(
            r, torch.Tensor) else r.to(torch.float32).cpu() for r in channel_ranges])
        if tuple(ranges.shape) != (2, D):
            raise ConfigError("channel_ranges must be two arrays of length head_dim")
        ranges = ranges.reshape(2, 1, D).to(x.device)
    codes, metas = quantize_tokens(x.reshape(cfg.block_size, 1, D), 1, 1, D, cfg.block_size, mode,
                                   cfg.rel_quant_scale, k_ranges=ranges)
    return QuantizedBlock(codes=codes[0], unit_mins=metas[0, :, 0].clone(),
                          unit_scales=metas[0, :, 1].clone(),
                          block_index=(ctx_start // cfg.block_size) * head_num + head_index,
                          head_index=head_index, ctx_start=ctx_start)


def dequantize_block(q: QuantizedBlock, mode: QuantMode) -> torch.Tensor:
    """quantizer.py:212-223: min + code * scale in float64."""
    codes = torch.as_tensor(q.codes).to(torch.float64)
    mins = torch.as_tensor(q.unit_mins).to(torch.float64)
    scales = torch.as_tensor(q.unit_scales).to(torch.float64)
    if mode is QuantMode.V_TOKEN:
        if mins.shape[0] != codes.shape[0]:
            raise CodecError("token-mode metadata count must equal block_size")
        return mins[:, None] + codes * scales[:, None]
    if mins.shape[0] != codes.shape[1]:
        raise CodecError("channel-mode metadata count must equal head_dim")
    return mins[None, :] + codes * scales[None, :]
