"""Device-resident compressed arena (reference codec.py:271-348) and counters.

The arena bytes are exactly the reference's serialisation (codec.py:229-244),
block after block in block_index order, so ``snapshot()`` is byte-comparable
with ``CompressedArena.snapshot()``.  Offsets and running totals live on the
device (``kvc_arena_counters``) and are advanced by the Store kernels; the
host reads them only when asked (stats, snapshot, error checks).
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from .errors import ArenaFullError, CodecError

TMA_SLACK = 64  # bytes after the cursor the fetch kernel may over-read


class _SlabPool:
    """Arena byte buffers carved from large per-device slabs.

    Compressed states live for the whole decode, so with the caching allocator
    every prefill's arenas are fresh cudaMalloc calls (~0.3 ms each, with
    multi-ms outliers).  Arenas instead take extents of 1 GiB slabs
    (``KVC_ARENA_SLAB_MB``): bump-allocated from a slab's free tail, first fit
    over the holes only when no tail fits; an extent returns to its slab when
    the arena grows, shrinks or is collected.  Extents are stream-ordered like the caching allocator's blocks:
    a released extent may be reused by work enqueued after the release.
    """

    ALIGN = 256

    def __init__(self, device: torch.device):
        import os
        import threading
        # states may be built and dropped from several threads, and an arena's
        # finalizer can run inside alloc (a GC pass): releases that find the
        # lock taken are queued and applied by the next alloc / release
        self.lock = threading.Lock()
        self.pending = []
        self.cur = 0  # slab whose free tail serves the next allocation
        self.device = device
        self.slab_bytes = int(os.environ.get("KVC_ARENA_SLAB_MB", "1024")) << 20
        self.slabs = []   # torch uint8 tensors
        self.free = []    # per slab: sorted list of [offset, size]

    def alloc(self, nbytes: int):
        with self.lock:
            self._drain()
            return self._alloc(nbytes)

    def _drain(self) -> None:
        while self.pending:
            self._release(*self.pending.pop())

    def _alloc(self, nbytes: int):
        n = max(self.ALIGN, (int(nbytes) + self.ALIGN - 1) // self.ALIGN * self.ALIGN)
        # 1. bump allocation from the free tail of the current slab, then of any
        #    slab (O(#slabs)); 2. first fit over all free extents only when no
        #    tail fits.  Compacted arenas leave many small holes behind, and a
        #    first-fit walk over them on every prefill grew to milliseconds
        #    (config 5: 64 sequences x 2 arenas per layer).
        order = [self.cur] + [si for si in range(len(self.free)) if si != self.cur] \
            if self.cur < len(self.free) else range(len(self.free))
        for si in order:
            fl = self.free[si]
            if fl and fl[-1][0] + fl[-1][1] == self.slabs[si].numel() and fl[-1][1] >= n:
                off, size = fl[-1]
                if size == n:
                    fl.pop()
                else:
                    fl[-1] = [off + n, size - n]
                self.cur = si
                return self.slabs[si][off: off + n], _Extent(self, si, off, n)
        for si, fl in enumerate(self.free):
            for i, (off, size) in enumerate(fl):
                if size >= n:
                    if size == n:
                        del fl[i]
                    else:
                        fl[i] = [off + n, size - n]
                    return self.slabs[si][off: off + n], _Extent(self, si, off, n)
        slab = max(self.slab_bytes, (n + (2 << 20) - 1) // (2 << 20) * (2 << 20))
        self.slabs.append(torch.empty(slab, dtype=torch.uint8, device=self.device))
        self.free.append([[n, slab - n]] if slab > n else [])
        self.cur = len(self.slabs) - 1
        return self.slabs[-1][:n], _Extent(self, len(self.slabs) - 1, 0, n)

    def release(self, si: int, off: int, n: int) -> None:
        self.pending.append((si, off, n))
        if self.lock.acquire(blocking=False):
            try:
                self._drain()
            finally:
                self.lock.release()

    def _release(self, si: int, off: int, n: int) -> None:
        fl = self.free[si]
        lo, hi = 0, len(fl)
        while lo < hi:
            mid = (lo + hi) // 2
            if fl[mid][0] < off:
                lo = mid + 1
            else:
                hi = mid
        fl.insert(lo, [off, n])
        if lo + 1 < len(fl) and fl[lo][0] + fl[lo][1] == fl[lo + 1][0]:
            fl[lo][1] += fl[lo + 1][1]
            del fl[lo + 1]
        if lo > 0 and fl[lo - 1][0] + fl[lo - 1][1] == fl[lo][0]:
            fl[lo - 1][1] += fl[lo][1]
            del fl[lo]


class _Extent:
    __slots__ = ("pool", "si", "off", "n", "live")

    def __init__(self, pool, si, off, n):
        self.pool, self.si, self.off, self.n, self.live = pool, si, off, n, True

    def release(self) -> None:
        if self.live:
            self.live = False
            self.pool.release(self.si, self.off, self.n)

    def shrink(self, nbytes: int) -> None:
        """Return the extent's tail beyond nbytes (aligned up) to the pool, in
        place: no new allocation, no copy."""
        keep = max(_SlabPool.ALIGN, (int(nbytes) + _SlabPool.ALIGN - 1) // _SlabPool.ALIGN
                   * _SlabPool.ALIGN)
        if self.live and keep < self.n:
            self.pool.release(self.si, self.off + keep, self.n - keep)
            self.n = keep


_POOLS = {}


def reserve_arena_pool(nbytes: int, device=None) -> int:
    """Pre-grow the arena slab pool of `device` to >= nbytes of free space.

    Fresh device memory costs ~3-5 us per MB to map (cudaMalloc), so a serving
    process reserves its compressed-cache memory once at startup (as paged KV
    managers reserve their block pool) instead of inside each prefill.
    Returns the pool's total free bytes."""
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    pool = _pool(dev)
    with pool.lock:
        pool._drain()
        free = sum(sz for fl in pool.free for _, sz in fl)
        while free < nbytes:
            slab = pool.slab_bytes
            pool.slabs.append(torch.empty(slab, dtype=torch.uint8, device=pool.device))
            pool.free.append([[0, slab]])
            free += slab
    return free


def pooled_zeros(shape, dtype, device):
    """A zero-filled tensor carved from the arena slab pool (long-lived state
    buffers: no caching-allocator segment growth per state).  Returns
    (tensor, extent); the owner releases the extent when it dies."""
    dev = torch.device(device)
    nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    raw, ext = _pool(dev).alloc(max(nbytes, 1))
    t = raw[:nbytes].view(dtype).view(*shape)
    t.zero_()
    return t, ext


def _pool(device: torch.device) -> _SlabPool:
    idx = device.index
    if idx is None and device.type == "cuda":
        idx = torch.cuda.current_device()
    key = (device.type, idx)
    p = _POOLS.get(key)
    if p is None:
        p = _POOLS[key] = _SlabPool(torch.device(device.type, idx) if idx is not None
                                    else torch.device(device.type))
    return p


@dataclass
class DataMovement:
    """Byte/scratch counters (codec.py:44-55)."""

    bytes_read: int = 0
    peak_scratch_values: int = 0

    def add_read(self, n: int) -> None:
        self.bytes_read += int(n)

    def note_scratch(self, n: int) -> None:
        self.peak_scratch_values = max(self.peak_scratch_values, int(n))


def worst_block_bytes(bs: int, n_units: int, head_dim: int, max_len: int) -> int:
    raw = 6 + 2 * bs + 8 * n_units + (bs * head_dim * max_len + 7) // 8
    return (raw + 3) & ~3


class DeviceArena:
    """Append-only device byte arena + u32 block offsets + device counters."""

    # Bytes past the cursor and offsets past n_blocks are never read as data
    # (TMA over-reads of the last block's rounded extent and the decoder's window
    # tail are don't-care bits), so the buffers are allocated without a memset.
    def __init__(self, device, capacity: Optional[int] = None, initial_bytes: int = 1 << 16,
                 initial_blocks: int = 256):
        self.device = torch.device(device)
        self.capacity = capacity  # user limit (None = grow on demand)
        alloc = initial_bytes if capacity is None else capacity
        self._extent = None
        self._set_buf(alloc + TMA_SLACK)
        # offsets and counters from the slab pool as well: per-state small
        # allocations otherwise grow the caching allocator's small pool (a
        # cudaMalloc per few states)
        self._offsets, self._off_ext = self._pooled(max(initial_blocks, 1) * 4, torch.int32)
        self._counters, self._cnt_ext = self._pooled(ctypes.sizeof(_lib.ArenaCounters),
                                                     torch.uint8, zero=True)
        self.n_blocks = 0          # host mirror (deterministic)
        self._bound = 0            # host upper bound on the cursor

    def _pooled(self, nbytes: int, dtype, zero: bool = False):
        """A device tensor of nbytes (as dtype) from the slab pool, released
        when this arena dies; plain torch memory off the GPU."""
        if self.device.type != "cuda":
            t = torch.zeros(nbytes, dtype=torch.uint8, device=self.device).view(dtype)
            return t, None
        raw, ext = _pool(self.device).alloc(nbytes)
        t = raw[:nbytes].view(dtype)
        if zero:
            t.zero_()
        weakref.finalize(self, ext.release)
        return t, ext

    def _set_buf(self, nbytes: int, keep: int = 0) -> None:
        """(Re)allocate the byte buffer from the slab pool, copying the first
        ``keep`` bytes; the previous extent goes back to the pool."""
        buf, ext = _pool(self.device).alloc(nbytes)
        buf = buf[:nbytes]
        if keep:
            buf[:keep] = self._buf[:keep]
        old = self._extent
        self._buf, self._extent = buf, ext
        weakref.finalize(self, ext.release)
        if old is not None:
            old.release()

    # ---- growth -------------------------------------------------------
    def reserve(self, n_blocks: int, worst_bytes: int) -> None:
        """Make room for n_blocks more blocks of at most worst_bytes total."""
        need_blocks = self.n_blocks + n_blocks
        if need_blocks > self._offsets.numel():
            new, ext = self._pooled(max(need_blocks, 2 * self._offsets.numel()) * 4, torch.int32)
            new[: self.n_blocks] = self._offsets[: self.n_blocks]
            old_ext = self._off_ext
            self._offsets, self._off_ext = new, ext
            if old_ext is not None:
                old_ext.release()
        if self.capacity is not None:
            return  # fixed capacity: the device reports ArenaFullError
        need = self._bound + worst_bytes
        if need > self._buf.numel() - TMA_SLACK:
            new_cap = max(need, 2 * (self._buf.numel() - TMA_SLACK))
            self._set_buf(new_cap + TMA_SLACK, keep=self._buf.numel())

    def compact(self, headroom: int = 0) -> None:
        """Shrink the allocation to the written bytes (+headroom) after a big prefill."""
        if self.capacity is not None:
            return
        cur = int(self.counters().cursor)
        size = cur + headroom
        if size + TMA_SLACK < self._buf.numel():
            if self._extent is not None:
                # in place: the extent's tail goes back to the pool (a copy into
                # a new extent would leave the old one behind as a hole)
                self._extent.shrink(size + TMA_SLACK)
                self._buf = self._buf[: size + TMA_SLACK]
            else:
                self._set_buf(size + TMA_SLACK, keep=cur)

    def load(self, data: bytes, offsets: np.ndarray, counters: bytes, headroom: int = 1 << 16):
        """Replace the contents with serialised blocks (container restore)."""
        n = len(data)
        cap = n + headroom if self.capacity is None else self.capacity
        if self.capacity is not None and n > self.capacity:
            raise ArenaFullError("restored arena exceeds capacity")
        buf = torch.zeros(cap + TMA_SLACK, dtype=torch.uint8)
        buf[:n] = torch.frombuffer(bytearray(data), dtype=torch.uint8) if n else buf[:0]
        self._set_buf(cap + TMA_SLACK)
        self._buf.copy_(buf)
        nb = len(offsets)
        offs = torch.zeros(max(nb, 1), dtype=torch.int32)
        if nb:
            offs[:nb] = torch.from_numpy(np.asarray(offsets, np.uint32).view(np.int32).copy())
        for e in (self._off_ext, self._cnt_ext):
            if e is not None:
                e.release()
        self._off_ext = self._cnt_ext = None
        self._offsets = offs.to(self.device)
        self._counters = torch.frombuffer(bytearray(counters), dtype=torch.uint8).to(self.device)
        self.n_blocks = nb
        self._bound = n

    def note_append(self, n_blocks: int, worst_bytes: int) -> None:
        self.n_blocks += n_blocks
        self._bound += worst_bytes

    @property
    def alloc_capacity(self) -> int:
        return self.capacity if self.capacity is not None else self._buf.numel() - TMA_SLACK

    # ---- device pointers ---------------------------------------------
    # the three device tensors keep their data pointers cached: descriptors of
    # every state are rebuilt-checked on each decode-step launch
    @property
    def _buf(self) -> torch.Tensor:
        return self.__buf

    @_buf.setter
    def _buf(self, t: torch.Tensor) -> None:
        self.__buf, self._buf_ptr = t, t.data_ptr()

    @property
    def _offsets(self) -> torch.Tensor:
        return self.__offsets

    @_offsets.setter
    def _offsets(self, t: torch.Tensor) -> None:
        self.__offsets, self._off_ptr = t, t.data_ptr()

    @property
    def _counters(self) -> torch.Tensor:
        return self.__counters

    @_counters.setter
    def _counters(self, t: torch.Tensor) -> None:
        self.__counters, self._cnt_ptr = t, t.data_ptr()

    @property
    def buf_ptr(self) -> int:
        return self._buf_ptr

    @property
    def offsets_ptr(self) -> int:
        return self._off_ptr

    @property
    def counters_ptr(self) -> int:
        return self._cnt_ptr

    # ---- host views (synchronising) ----------------------------------
    def counters(self) -> _lib.ArenaCounters:
        raw = self._counters.cpu().numpy().tobytes()
        c = _lib.ArenaCounters.from_buffer_copy(raw)
        self._bound = int(c.cursor)
        return c

    def check(self, what: str = "arena") -> None:
        c = self.counters()
        if c.err:
            _lib.raise_device_error(c.err, what)

    def __len__(self) -> int:
        return self.n_blocks

    @property
    def write_cursor(self) -> int:
        return int(self.counters().cursor)

    @property
    def size_bytes(self) -> int:
        return self.write_cursor

    @property
    def payload_bits(self) -> int:
        return int(self.counters().payload_bits)

    @property
    def payload_bytes(self) -> int:
        return int(self.counters().payload_bytes)

    @property
    def max_extent(self) -> int:
        return int(self.counters().max_extent)

    @property
    def block_offsets(self) -> np.ndarray:
        return self._offsets[: self.n_blocks].cpu().numpy().view(np.uint32).copy()

    def snapshot(self) -> bytes:
        cur = self.write_cursor
        return self._buf[:cur].cpu().numpy().tobytes()

    def extent(self, ordinal: int) -> Tuple[int, int]:
        if not 0 <= ordinal < self.n_blocks:
            raise CodecError(f"block ordinal {ordinal} out of range")
        offs = self.block_offsets
        end = int(offs[ordinal + 1]) if ordinal + 1 < self.n_blocks else self.write_cursor
        return int(offs[ordinal]), end

    def raw_tensor(self) -> torch.Tensor:
        return self._buf

    def offsets_tensor(self) -> torch.Tensor:
        return self._offsets


def full_error(what="arena"):
    return ArenaFullError(f"{what}: capacity exhausted")
