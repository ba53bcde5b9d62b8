"""``kvpack`` with host outputs: the package's API with every torch tensor a
call returns converted to a numpy array (recursively through dataclasses,
tuples, lists and generators), for callers written against the reference,
whose functions return numpy (kvpack/__init__.py:9-75).  The kernels and
device state are the same; only the returned values are copied to the host.

    import paper_2509_00579_b200.numpy_api as kvpack
    kvpack.install()   # optional: also answer ``import kvpack`` / ``kvpack.codec`` ...

The device API (tensors stay on the GPU) remains ``paper_2509_00579_b200``.
"""

from __future__ import annotations

import dataclasses
import functools
import sys
import types

import torch

import paper_2509_00579_b200 as _pkg
from . import (attention, bench, codebook, codec, container, errors, kvcache, quantizer,
               tensor_io)

_MODULES = {"attention": attention, "bench": bench, "codebook": codebook, "codec": codec,
            "container": container, "errors": errors, "kvcache": kvcache,
            "quantizer": quantizer, "tensor_io": tensor_io}


def to_host(x):
    """torch tensors -> numpy, recursively; private dataclass fields (device
    caches such as a block's serialised image) are left as they are."""
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    if dataclasses.is_dataclass(x) and not isinstance(x, type):
        ch = {f.name: to_host(getattr(x, f.name)) for f in dataclasses.fields(x)
              if f.init and not f.name.startswith("_")}
        if isinstance(x, codec.CompressedBlock):
            ch["payload"] = ch["payload"].tobytes()  # bytes, as the reference's block
        return dataclasses.replace(x, **ch)
    if isinstance(x, tuple) and hasattr(x, "_fields"):
        return type(x)(*map(to_host, x))
    if isinstance(x, (tuple, list)):
        return type(x)(map(to_host, x))
    if isinstance(x, types.GeneratorType):
        return (to_host(v) for v in x)
    return x


def _wrap(fn):
    @functools.wraps(fn)
    def call(*args, **kwargs):
        return to_host(fn(*args, **kwargs))
    return call


class LayerCacheState(kvcache.LayerCacheState):
    """kvcache.LayerCacheState whose host-facing reads return numpy."""

    def fetch_dequantized(self):
        return to_host(super().fetch_dequantized())


def _is_ours(obj) -> bool:
    return getattr(obj, "__module__", "").startswith(_pkg.__name__)


def _facade(mod):
    """A copy of ``mod`` with its functions wrapped and LayerCacheState
    replaced; classes, constants and exceptions are shared."""
    out = types.ModuleType(mod.__name__.replace(_pkg.__name__, "kvpack"), mod.__doc__)
    for name in dir(mod):
        if name.startswith("__"):
            continue
        obj = getattr(mod, name)
        if obj is kvcache.LayerCacheState:
            obj = LayerCacheState
        elif isinstance(obj, types.FunctionType) and _is_ours(obj):
            obj = _wrap(obj)
        setattr(out, name, obj)
    return out


_SUB = {name: _facade(m) for name, m in _MODULES.items()}
_TOP = _facade(_pkg)
for _name, _m in _SUB.items():
    setattr(_TOP, _name, _m)

# this module's public surface is the facade's
for _name in dir(_TOP):
    if not _name.startswith("__"):
        globals().setdefault(_name, getattr(_TOP, _name))
globals().update(_SUB)


def install() -> types.ModuleType:
    """Register the facade as ``kvpack`` and ``kvpack.<module>``."""
    sys.modules["kvpack"] = _TOP
    for name, m in _SUB.items():
        sys.modules["kvpack." + name] = m
    return _TOP
