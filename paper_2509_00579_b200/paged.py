"""Paged arena memory (the paper's paged-cache integration).

vLLM-style block tables give every sequence a list of fixed-size physical
pages from one shared pool, so memory is committed as a cache grows and
returned when it shrinks, with no per-sequence maximum reservation.  Here
the page table is the GPU's own: a ``PagedArena`` reserves a large virtual
range once (CUDA virtual memory, ``csrc/vmm.cu``) and maps physical pages
from a ``PagePool`` into it as it grows.  Growth never copies and never moves
the arena (so descriptors stay valid), ``compact`` returns the unused tail
pages to the pool, and every kernel still sees one contiguous arena with u32
offsets -- the Store and Fetch kernels are unchanged.

    pool = PagePool(device, page_bytes=2 << 20)
    st = LayerCacheState.prefill(k, v, cfg_k, cfg_v, page_pool=pool)
"""

from __future__ import annotations

import threading
from typing import Optional

import torch

from . import _lib
from .codec import TMA_SLACK, DeviceArena
from .errors import ArenaFullError

VA_BYTES = (4 << 30) + (64 << 20)   # u32 offsets cap an arena at 4 GiB; + TMA slack


class _CudaSpan:
    """A device byte range for torch.as_tensor (__cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class PagePool:
    """Physical pages (cuMemCreate) shared by the paged arenas of one device.
    Pages handed back by an arena are reused before new ones are created;
    ``max_pages`` caps the pool (ArenaFullError past it)."""

    def __init__(self, device=None, page_bytes: int = 2 << 20, max_pages: Optional[int] = None):
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.index = self.device.index if self.device.index is not None else \
            torch.cuda.current_device()
        lib = _lib.lib()
        import ctypes
        g = ctypes.c_size_t(0)
        _lib.check(lib.kvc_vmm_granularity(self.index, ctypes.byref(g)), "PagePool")
        gran = int(g.value)
        self.page_bytes = max(gran, (int(page_bytes) + gran - 1) // gran * gran)
        self.max_pages = max_pages
        self.free = []
        self.created = 0
        self.lock = threading.Lock()

    @property
    def pages_in_use(self) -> int:
        return self.created - len(self.free)

    def take(self) -> int:
        with self.lock:
            if self.free:
                return self.free.pop()
            if self.max_pages is not None and self.created >= self.max_pages:
                raise ArenaFullError(f"page pool exhausted ({self.max_pages} pages of "
                                     f"{self.page_bytes} B)")
            import ctypes
            h = ctypes.c_uint64(0)
            _lib.check(_lib.lib().kvc_vmm_create(self.index, self.page_bytes, ctypes.byref(h)),
                       "PagePool")
            self.created += 1
            return int(h.value)

    def give(self, handle: int) -> None:
        with self.lock:
            self.free.append(handle)

    def trim(self) -> int:
        """Release the pool's free pages to the driver; returns how many."""
        with self.lock:
            n = len(self.free)
            for h in self.free:
                _lib.lib().kvc_vmm_release(h)
            self.created -= n
            self.free.clear()
            return n


class _Mapping:
    """The pages mapped into one arena's virtual range (finalizer target)."""

    def __init__(self, pool: PagePool):
        import ctypes
        self.pool = pool
        va = ctypes.c_uint64(0)
        _lib.check(_lib.lib().kvc_vmm_reserve(VA_BYTES, ctypes.byref(va)), "PagedArena")
        self.va = int(va.value)
        self.pages = []

    def grow(self, nbytes: int) -> None:
        pb = self.pool.page_bytes
        need = (int(nbytes) + pb - 1) // pb
        if need * pb > VA_BYTES:
            raise ArenaFullError("paged arena exceeds its 4 GiB virtual range")
        while len(self.pages) < need:
            h = self.pool.take()
            st = _lib.lib().kvc_vmm_map(self.va + len(self.pages) * pb, pb, h, self.pool.index)
            if st != _lib.KVC_OK:
                self.pool.give(h)
                _lib.check(st, "PagedArena")
            self.pages.append(h)

    def shrink(self, nbytes: int) -> None:
        """Unmap the pages wholly past nbytes (the caller has synchronised)."""
        pb = self.pool.page_bytes
        keep = max(1, (int(nbytes) + pb - 1) // pb)
        while len(self.pages) > keep:
            h = self.pages.pop()
            _lib.lib().kvc_vmm_unmap(self.va + len(self.pages) * pb, pb)
            self.pool.give(h)

    @property
    def mapped(self) -> int:
        return len(self.pages) * self.pool.page_bytes

    def close(self) -> None:
        if not self.va:
            return
        try:
            if self.pages:
                torch.cuda.synchronize(self.pool.device)  # no kernel still reads the pages
            self.shrink(0)
            if self.pages:
                h = self.pages.pop()
                _lib.lib().kvc_vmm_unmap(self.va, self.pool.page_bytes)
                self.pool.give(h)
            _lib.lib().kvc_vmm_free_va(self.va, VA_BYTES)
        except Exception:  # interpreter / CUDA context teardown: the driver reclaims it
            pass
        self.va = 0


class PagedArena(DeviceArena):
    """A DeviceArena whose bytes are pages of a PagePool mapped into one
    fixed virtual range: growth maps pages (no copy, the address never
    changes), compaction returns pages."""

    def __init__(self, device, capacity: Optional[int] = None, initial_bytes: int = 1 << 16,
                 initial_blocks: int = 256, counters: Optional[torch.Tensor] = None,
                 pool: Optional[PagePool] = None):
        import weakref
        self._map = _Mapping(pool if pool is not None else PagePool(device))
        weakref.finalize(self, self._map.close)
        super().__init__(device, capacity, initial_bytes=initial_bytes,
                         initial_blocks=initial_blocks, counters=counters)

    def _set_buf(self, nbytes: int, keep: int = 0) -> None:
        self._map.grow(nbytes)
        self._buf = torch.as_tensor(_CudaSpan(self._map.va, self._map.mapped),
                                    device=self.device)

    def compact(self, headroom: int = 0) -> None:
        if self.capacity is not None:
            return
        cur = int(self.counters().cursor)  # synchronises the stream
        self._map.shrink(cur + headroom + TMA_SLACK)
        self._buf = torch.as_tensor(_CudaSpan(self._map.va, self._map.mapped),
                                    device=self.device)

    @property
    def pages(self) -> int:
        return len(self._map.pages)
