"""Dense KV tensors and synthetic KV generation (reference tensor_io.py:30-157).

``generate_synthetic`` reproduces the reference generator bit-for-bit (same
PCG64 streams, float32 normals, outlier channels) so oracle-checked inputs
are identical; ``generate_synthetic_device`` draws the same distribution on
the GPU (torch RNG, not bit-identical) for full-size benchmark inputs.
``write_tensor`` / ``read_tensor`` handle the reference's KVTN files
(tensor_io.py:100-143): a 30-byte little-endian header (b"KVTN", version 1,
dtype code 0 = f16 / 1 = f32, three u64 dimensions) and the raw values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import TensorFormatError


@dataclass(frozen=True)
class CacheTensor:
    """Dense [context_len, head_num, head_dim] f16/f32 tensor (numpy or torch)."""

    values: object

    def __post_init__(self):
        v = self.values
        if isinstance(v, torch.Tensor):
            if v.ndim != 3 or min(v.shape) < 1:
                raise TensorFormatError("values must be a 3-d tensor with positive dimensions")
            if v.dtype not in (torch.float16, torch.float32):
                raise TensorFormatError(f"unsupported dtype {v.dtype}")
            return
        if not isinstance(v, np.ndarray) or v.ndim != 3:
            raise TensorFormatError("values must be a 3-d ndarray [context_len, head_num, head_dim]")
        if min(v.shape) < 1:
            raise TensorFormatError(f"all dimensions must be positive, got shape {v.shape}")
        if v.dtype not in (np.float16, np.float32):
            raise TensorFormatError(f"unsupported dtype {v.dtype}; expected float16 or float32")
        if not np.all(np.isfinite(v)):
            raise TensorFormatError("NaN/Inf values are not accepted into the pipeline")

    @property
    def context_len(self) -> int:
        return int(self.values.shape[0])

    @property
    def head_num(self) -> int:
        return int(self.values.shape[1])

    @property
    def head_dim(self) -> int:
        return int(self.values.shape[2])

    @property
    def dtype(self):
        return self.values.dtype

    def as_float32(self):
        if isinstance(self.values, torch.Tensor):
            return self.values.to(torch.float32).contiguous()
        return np.ascontiguousarray(self.values, dtype=np.float32)

    def numpy(self) -> np.ndarray:
        v = self.values
        return v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v


@dataclass(frozen=True)
class SyntheticSpec:
    context_len: int
    head_num: int
    head_dim: int
    seed: int = 0
    channel_outlier_fraction: float = 0.05
    outlier_magnitude: float = 8.0
    base_std: float = 1.0

    def __post_init__(self):
        if min(self.context_len, self.head_num, self.head_dim) < 1:
            raise TensorFormatError("context_len, head_num and head_dim must be positive")
        if not 0.0 <= self.channel_outlier_fraction <= 1.0:
            raise TensorFormatError("channel_outlier_fraction must lie in [0, 1]")
        if self.outlier_magnitude <= 0 or self.base_std <= 0:
            raise TensorFormatError("outlier_magnitude and base_std must be positive")
        if not 0 <= self.seed < 2 ** 64:
            raise TensorFormatError("seed must fit an unsigned 64-bit integer")


def _outlier_mask(spec: SyntheticSpec) -> np.ndarray:
    rng = np.random.default_rng([spec.seed, 0x6F75746C])
    return rng.random((spec.head_num, spec.head_dim)) < spec.channel_outlier_fraction


def generate_synthetic(spec: SyntheticSpec) -> CacheTensor:
    """Bit-identical to tensor_io.py:142-157."""
    outliers = _outlier_mask(spec)
    rng = np.random.default_rng([spec.seed, 0x76616C73])
    values = rng.standard_normal((spec.context_len, spec.head_num, spec.head_dim),
                                 dtype=np.float32)
    values *= np.float32(spec.base_std)
    values[:, outliers] *= np.float32(spec.outlier_magnitude)
    return CacheTensor(values)


def generate_synthetic_device(spec: SyntheticSpec, device="cuda", dtype=torch.float16,
                              out: torch.Tensor = None) -> torch.Tensor:
    """Same distribution on the device (seeded torch RNG; not bit-identical)."""
    g = torch.Generator(device=device)
    g.manual_seed(int(spec.seed) & 0x7FFFFFFFFFFFFFFF)
    scale = torch.full((spec.head_num, spec.head_dim), spec.base_std, dtype=torch.float32)
    scale[torch.from_numpy(_outlier_mask(spec))] *= spec.outlier_magnitude
    scale = scale.to(device)
    shape = (spec.context_len, spec.head_num, spec.head_dim)
    if out is None:
        out = torch.empty(shape, dtype=dtype, device=device)
    step = max(1, (1 << 26) // (spec.head_num * spec.head_dim))
    for t0 in range(0, spec.context_len, step):
        t1 = min(spec.context_len, t0 + step)
        x = torch.randn((t1 - t0, spec.head_num, spec.head_dim), generator=g, device=device,
                        dtype=torch.float32)
        out[t0:t1] = (x * scale).to(dtype)
    return out


# KVTN header (tensor_io.py:22-26) as a packed little-endian record
_KVTN = np.dtype([("magic", "S4"), ("version", "u1"), ("code", "u1"), ("dims", "<u8", (3,))])
_KVTN_VERSION = 1
_KVTN_TYPES = (np.dtype("<f2"), np.dtype("<f4"))  # indexed by the dtype code


def write_tensor(t: CacheTensor, path) -> None:
    """tensor_io.py:100-111: header + C-order values.  Device tensors are
    copied to the host first."""
    v = t.values
    if isinstance(v, torch.Tensor):
        v = v.detach().cpu().numpy()
    v = np.asarray(v)
    if v.dtype not in (np.float16, np.float32):
        raise TensorFormatError(f"cannot write dtype {v.dtype}")
    code = 0 if v.dtype == np.float16 else 1
    hdr = np.zeros((), _KVTN)
    hdr["magic"], hdr["version"], hdr["code"] = b"KVTN", _KVTN_VERSION, code
    hdr["dims"] = v.shape
    with open(path, "wb") as fh:
        fh.write(hdr.tobytes())
        fh.write(np.ascontiguousarray(v, dtype=_KVTN_TYPES[code]).tobytes())


def read_tensor(path) -> CacheTensor:
    """tensor_io.py:114-143: the inverse of write_tensor, validating the
    header, the payload length and finiteness (TensorFormatError)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _KVTN.itemsize:
        raise TensorFormatError(f"KVTN header needs {_KVTN.itemsize} bytes, file has {len(blob)}")
    hdr = np.frombuffer(blob, _KVTN, count=1)[0]
    if bytes(hdr["magic"]) != b"KVTN":
        raise TensorFormatError(f"not a KVTN file (magic {bytes(hdr['magic'])!r})")
    if int(hdr["version"]) != _KVTN_VERSION:
        raise TensorFormatError(f"KVTN version {int(hdr['version'])} is not supported")
    code = int(hdr["code"])
    if code >= len(_KVTN_TYPES):
        raise TensorFormatError(f"KVTN dtype code {code} is not supported")
    dims = tuple(int(d) for d in hdr["dims"])
    if min(dims) < 1:
        raise TensorFormatError(f"KVTN dimensions {dims} must be positive")
    dt = _KVTN_TYPES[code]
    need = dims[0] * dims[1] * dims[2] * dt.itemsize
    have = len(blob) - _KVTN.itemsize
    if have < need:
        raise TensorFormatError(f"truncated KVTN payload ({have} of {need} bytes)")
    if have > need:
        raise TensorFormatError(f"{have - need} trailing bytes after the KVTN payload")
    vals = np.frombuffer(blob, dt, offset=_KVTN.itemsize).reshape(dims).copy()
    if not np.isfinite(vals).all():
        raise TensorFormatError("KVTN payload holds NaN/Inf")
    return CacheTensor(vals)
