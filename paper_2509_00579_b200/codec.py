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
from dataclasses import dataclass, field
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
                 initial_blocks: int = 256, counters: Optional[torch.Tensor] = None):
        self.device = torch.device(device)
        self.capacity = capacity  # user limit (None = grow on demand)
        alloc = initial_bytes if capacity is None else capacity
        self._extent = None
        self._set_buf(alloc + TMA_SLACK)
        # offsets and counters from the slab pool as well: per-state small
        # allocations otherwise grow the caching allocator's small pool (a
        # cudaMalloc per few states)
        self._offsets, self._off_ext = self._pooled(max(initial_blocks, 1) * 4, torch.int32)
        if counters is not None:  # zeroed device bytes owned by the caller (the state)
            self._counters, self._cnt_ext = counters, None
        else:
            self._counters, self._cnt_ext = self._pooled(ctypes.sizeof(_lib.ArenaCounters),
                                                         torch.uint8, zero=True)
        self.n_blocks = 0          # host mirror (deterministic)
        self._bound = 0            # host upper bound on the cursor
        # host mirror of counters.max_extent (the fused fetch sizes its
        # shared-memory stages from it): exact after a counters() read; after
        # appends it is refreshed by an asynchronous readback, and until that
        # lands stage sizes use the appended blocks' worst case
        self._ext_host = 0
        self._ext_worst = 0        # worst extent of blocks appended since the last read
        self._ext_pending = None   # (pinned slot, event) of an in-flight readback

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
            # 1.25x growth: a compacted config-2 arena is ~90 MB and a decode
            # step's overflow event adds ~0.3 MB, so doubling would map (and
            # copy) gigabytes per event across a batch of states
            cur = self._buf.numel() - TMA_SLACK
            new_cap = max(need, cur + cur // 4, 1 << 16)
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
        self._buf[: buf.numel()].copy_(buf)
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
        self._ext_pending = None
        self._ext_host = _lib.ArenaCounters.from_buffer_copy(bytes(counters)).max_extent
        self._ext_worst = 0

    def note_append(self, n_blocks: int, worst_bytes: int, block_worst: int = 0) -> None:
        """Host mirrors after an append of n_blocks (worst_bytes in total,
        block_worst per block); starts the asynchronous max-extent readback."""
        self.n_blocks += n_blocks
        self._bound += worst_bytes
        if n_blocks:
            self._ext_worst = max(self._ext_worst, block_worst or worst_bytes)
            self._ext_stale = True  # a readback starts at the next bound query

    def max_extent_bound(self) -> int:
        """An upper bound of every block extent, without synchronising: the
        exact device value once known, else the worst case of the blocks
        appended since it was last read (and an asynchronous readback of the
        counters is started)."""
        if getattr(self, "_ext_stale", False):
            self._ext_stale = False
            if self.device.type == "cuda":
                self._ext_pending = _counters_readback(self._counters)
        if self._ext_pending is not None:
            buf, ev = self._ext_pending
            if ev.query():
                c = _lib.ArenaCounters.from_buffer_copy(buf.numpy().tobytes())
                self._ext_pending = None
                self._ext_host, self._ext_worst = int(c.max_extent), 0
        return max(self._ext_host, self._ext_worst)

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
        self._ext_host, self._ext_worst, self._ext_pending = int(c.max_extent), 0, None
        self._ext_stale = False
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


class _PinnedRing:
    """Pinned host slots for asynchronous counter readbacks; a slot is
    rewritten only after the event of its previous copy has completed."""

    def __init__(self, slot_bytes: int, slots: int = 1024):
        self.buf = torch.empty((slots, slot_bytes), dtype=torch.uint8, pin_memory=True)
        self.events = [None] * slots
        self.i = 0


_CNT_RING = None


def _counters_readback(counters: torch.Tensor):
    global _CNT_RING
    if _CNT_RING is None:
        _CNT_RING = _PinnedRing(ctypes.sizeof(_lib.ArenaCounters))
    r = _CNT_RING
    i = r.i
    r.i = (i + 1) % len(r.events)
    if r.events[i] is not None:
        r.events[i].synchronize()
    slot = r.buf[i]
    slot.copy_(counters, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(counters.device))
    r.events[i] = ev
    return slot, ev


# pinned slots of batched readbacks: [host buffer, event, weakrefs of the arenas served]
_BATCH_SLOTS: list = []


def readback_extents(arenas) -> None:
    """Start one asynchronous counter readback for many arenas at once (a
    stacked device copy, one D2H copy, one event) instead of one per arena:
    after a batch's overflow event the per-arena copies were thousands of
    tiny transfers whose pinned ring also throttled the host.  Arenas without
    a stale extent are skipped; max_extent_bound() consumes the result."""
    todo = [a for a in arenas if getattr(a, "_ext_stale", False) and a.device.type == "cuda"]
    if len(todo) < 2:
        return
    rows = torch.stack([a._counters.view(torch.uint8).reshape(-1) for a in todo])
    nb = rows.numel()
    slot = None
    for sl in _BATCH_SLOTS:
        if sl[0].numel() >= nb and (sl[1] is None or sl[1].query()):
            slot = sl
            break
    if slot is None:
        slot = [torch.empty(max(nb, 1 << 16), dtype=torch.uint8, pin_memory=True), None, []]
        _BATCH_SLOTS.append(slot)
    # arenas that have not read their result from this slot yet do so now
    # (its copy has completed), before it is overwritten
    for r in slot[2]:
        a = r()
        if a is not None and a._ext_pending is not None and a._ext_pending[1] is slot[1]:
            a.max_extent_bound()
    host = slot[0][:nb].view(len(todo), -1)
    host.copy_(rows, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(todo[0].device))
    slot[1], slot[2] = ev, [weakref.ref(a) for a in todo]  # weak: arenas may be freed
    for i, a in enumerate(todo):
        a._ext_stale = False
        a._ext_pending = (host[i], ev)


def full_error(what="arena"):
    return ArenaFullError(f"{what}: capacity exhausted")


# ---------------------------------------------------------------------------
# Per-block codec surface (reference codec.py:59-226, :308-341, :351-472).
# The Store/Fetch hot path never builds these objects; they are the
# reference's single-block API, backed by the same device kernels
# (kvc_encode_append for encoding, kvc_decode_blocks / kvc_decode_slices_tree
# for decoding, kvc_arena_append / kvc_arena_restore for the arena).
# ---------------------------------------------------------------------------

MAX_SLICE_BITS = 0xFFFF


def _dev(device=None) -> torch.device:
    return torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _to_dev(x, dtype, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(dev, dtype).contiguous()
    if isinstance(x, (bytes, bytearray, memoryview)):
        x = np.frombuffer(bytes(x), dtype=np.uint8)
    return torch.as_tensor(np.ascontiguousarray(x)).to(dev, dtype).contiguous()


@dataclass(frozen=True)
class CompressedBlock:
    """One entropy-coded block (codec.py:59-74): per-slice bit counts, unit
    metadata and the byte-padded payload, as device tensors.  Blocks made by
    ``compress_block`` also carry their serialised image, so
    ``DeviceArena.append`` is a device copy."""

    block_index: int
    slice_bit_counts: torch.Tensor  # (n_slices,) int32 (u16 values)
    unit_mins: torch.Tensor         # (n_units,) float32
    unit_scales: torch.Tensor       # (n_units,) float32
    payload: torch.Tensor           # (ceil(bits/8),) uint8
    _total_bits: Optional[int] = field(default=None, compare=False, repr=False)
    _image: Optional[torch.Tensor] = field(default=None, compare=False, repr=False)

    @property
    def n_slices(self) -> int:
        return int(self.slice_bit_counts.shape[0])

    @property
    def total_bits(self) -> int:
        if self._total_bits is not None:
            return self._total_bits
        return int(torch.as_tensor(np.asarray(self.slice_bit_counts) if not isinstance(
            self.slice_bit_counts, torch.Tensor) else self.slice_bit_counts).to(torch.int64).sum())


def _encode_one_block(codes: torch.Tensor, metas: torch.Tensor, block_index: int, cb):
    """kvc_encode_append on a private one-block arena: returns (image, bits).
    Missing codes / 16-bit slice overflow raise CodecError (codec.py:85-102)."""
    dev = codes.device
    bs, D = codes.shape
    n_units = metas.shape[0]
    lib = _lib.lib()
    arena = DeviceArena(dev, None, initial_bytes=worst_block_bytes(bs, n_units, D,
                                                                   cb.max_code_length) + TMA_SLACK,
                        initial_blocks=1)
    ws = torch.empty(lib.kvc_encode_workspace_bytes(1, bs), dtype=torch.uint8, device=dev)
    st = lib.kvc_encode_append(codes.data_ptr(), metas.data_ptr(), 1, 1, 1, 0, int(block_index),
                               bs, D, n_units, cb.max_code_length,
                               cb.device_tables(dev).data_ptr(), arena.buf_ptr,
                               arena.alloc_capacity, arena.offsets_ptr, arena.counters_ptr,
                               ws.data_ptr(), _stream(dev))
    _lib.check(st, "compress_block")
    c = arena.counters()
    if c.err:
        _lib.raise_device_error(c.err, "compress_block")
    return arena.raw_tensor()[: int(c.cursor)].clone(), int(c.payload_bits)


def _check_codes(codes: torch.Tensor, cb) -> torch.Tensor:
    """codec.py:77-91: every code must be present in the codebook; returns
    the per-code lengths (device)."""
    lens = torch.as_tensor(cb.code_lengths.astype(np.int64)).to(codes.device)[codes.long()]
    absent = lens == 0
    if bool(absent.any()):
        missing = int(codes[absent].reshape(-1)[0])
        raise CodecError(f"code {missing} is absent from the codebook")
    return lens


def encode_slice(codes, cb) -> Tuple[torch.Tensor, int]:
    """codec.py:94-103: one slice -> (its codeword bits as a 0/1 uint8 device
    tensor, bit count)."""
    dev = codes.device if isinstance(codes, torch.Tensor) and codes.is_cuda else _dev()
    arr = _to_dev(codes, torch.uint8, dev).reshape(-1)
    if arr.numel() == 0:
        raise CodecError("cannot encode an empty slice")
    total = int(_check_codes(arr, cb).sum())
    if total > MAX_SLICE_BITS:
        raise CodecError(f"slice bit count {total} overflows 16 bits")
    image, bits = _encode_one_block(arr.reshape(1, -1),
                                    torch.zeros((1, 2), dtype=torch.float32, device=dev), 0, cb)
    hdr = 6 + 2 + 8
    payload = image[hdr: hdr + (bits + 7) // 8]
    shifts = torch.arange(7, -1, -1, device=dev, dtype=torch.uint8)
    out = ((payload[:, None] >> shifts) & 1).reshape(-1)[:bits]
    return out.contiguous(), bits


def scan_offsets(bit_counts) -> Tuple[torch.Tensor, int]:
    """codec.py:106-116: exclusive bit offsets from the inclusive scan, and
    the total (CodecError past 32 bits)."""
    c = bit_counts if isinstance(bit_counts, torch.Tensor) else torch.as_tensor(
        np.asarray(bit_counts, dtype=np.int64))
    c = c.to(torch.int64)
    if c.is_cpu:
        c = c.to(_dev())
    if c.numel() == 0:
        raise CodecError("scan over an empty bit-count array")
    inclusive = torch.cumsum(c.reshape(-1), 0)
    total = int(inclusive[-1])
    if total > 0xFFFFFFFF:
        raise CodecError("total bit count overflows 32 bits")
    return inclusive - c.reshape(-1), total


def compress_block(q, cb) -> CompressedBlock:
    """codec.py:119-138 on the device (the Store's block encoder)."""
    codes = q.codes
    dev = codes.device if isinstance(codes, torch.Tensor) and codes.is_cuda else _dev()
    codes = _to_dev(codes, torch.uint8, dev)
    if codes.ndim != 2:
        raise CodecError("block codes must be a (n_slices, head_dim) matrix")
    _check_codes(codes, cb)
    mins = _to_dev(q.unit_mins, torch.float32, dev).reshape(-1)
    scales = _to_dev(q.unit_scales, torch.float32, dev).reshape(-1)
    metas = torch.stack([mins, scales], dim=1).contiguous()
    image, bits = _encode_one_block(codes, metas, q.block_index, cb)
    bs = codes.shape[0]
    counts = image[6: 6 + 2 * bs].view(torch.int16).to(torch.int32) & 0xFFFF
    p0 = 6 + 2 * bs + 8 * metas.shape[0]
    return CompressedBlock(block_index=int(q.block_index), slice_bit_counts=counts,
                           unit_mins=mins, unit_scales=scales,
                           payload=image[p0: p0 + (bits + 7) // 8].clone(), _total_bits=bits,
                           _image=image)


def _tree_decode(bits: torch.Tensor, packed: bool, n_bits: int, offs: torch.Tensor,
                 counts: torch.Tensor, tree, out_len: int) -> torch.Tensor:
    dev = bits.device
    n = offs.numel()
    children, is_symbol, symbols = tree.device(dev)
    out = torch.zeros((n, out_len), dtype=torch.uint8, device=dev)
    bad = torch.full((1,), n, dtype=torch.int32, device=dev)
    st = _lib.lib().kvc_decode_slices_tree(bits.data_ptr(), int(packed), int(n_bits),
                                           offs.data_ptr(), counts.data_ptr(), n,
                                           children.data_ptr(), is_symbol.data_ptr(),
                                           symbols.data_ptr(), tree.n_nodes, out_len,
                                           out.data_ptr(), bad.data_ptr(), _stream(dev))
    _lib.check(st, "decode_slices")
    b = int(bad.item())
    if b < n:
        raise CodecError(f"corrupt slice {b}: the stream does not decode to {out_len} symbols "
                         f"in {int(counts[b])} bits")
    return out


def decode_slice(payload, bit_offset: int, bit_count: int, tree, out_len: int) -> torch.Tensor:
    """codec.py:141-173: one slice of a packed MSB-first payload, decoded
    with the array-form tree on the device."""
    dev = payload.device if isinstance(payload, torch.Tensor) and payload.is_cuda else _dev()
    data = _to_dev(payload, torch.uint8, dev).reshape(-1)
    if bit_offset < 0 or bit_offset + bit_count > data.numel() * 8:
        raise CodecError("bit range outside payload")
    offs = torch.tensor([bit_offset], dtype=torch.int64, device=dev)
    cnt = torch.tensor([bit_count], dtype=torch.int64, device=dev)
    return _tree_decode(data, True, data.numel() * 8, offs, cnt, tree, out_len)[0]


def decode_slices(bits, bit_offsets, bit_counts, tree, out_len: int) -> torch.Tensor:
    """codec.py:176-226: many slices of an unpacked 0/1 bit array, one device
    thread per slice (the reference's lockstep loop)."""
    dev = bits.device if isinstance(bits, torch.Tensor) and bits.is_cuda else _dev()
    b = _to_dev(bits, torch.uint8, dev).reshape(-1)
    offs = _to_dev(bit_offsets, torch.int64, dev).reshape(-1)
    counts = _to_dev(bit_counts, torch.int64, dev).reshape(-1)
    if offs.numel() == 0:
        return torch.zeros((0, out_len), dtype=torch.uint8, device=dev)
    if bool((offs < 0).any()) or bool((offs + counts > b.numel()).any()):
        raise CodecError("bit range outside payload")
    return _tree_decode(b, False, b.numel(), offs, counts, tree, out_len)


def units_per_block(mode, head_dim: int, block_size: int) -> int:
    """codec.py:344-346: one metadata unit per channel (K) or token (V)."""
    from .quantizer import QuantMode
    return block_size if mode is QuantMode.V_TOKEN else head_dim


def decompress_block(arena: "DeviceArena", ordinal: int, cb, *, mode, head_num: int,
                     head_dim: int, block_size: int):
    """codec.py:351-391: the exact inverse of compress_block + append, on the
    device (kvc_decode_blocks)."""
    from .quantizer import QuantizedBlock
    if not 0 <= ordinal < arena.n_blocks:
        raise CodecError(f"block ordinal {ordinal} out of range")
    dev = arena.device
    n_units = units_per_block(mode, head_dim, block_size)
    codes = torch.empty((1, block_size, head_dim), dtype=torch.uint8, device=dev)
    metas = torch.empty((1, n_units, 2), dtype=torch.float32, device=dev)
    bidx = torch.zeros(1, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    ords = torch.tensor([ordinal], dtype=torch.int32, device=dev)
    st = _lib.lib().kvc_decode_blocks(arena.buf_ptr, arena.offsets_ptr, arena.counters_ptr,
                                      ords.data_ptr(), 1, block_size, n_units, head_dim,
                                      cb.device_tables(dev).data_ptr(), codes.data_ptr(),
                                      metas.data_ptr(), bidx.data_ptr(), err.data_ptr(),
                                      _stream(dev))
    _lib.check(st, "decompress_block")
    _lib.raise_device_error(int(err.item()), "decompress_block")
    block_index = int(bidx.item()) & 0xFFFFFFFF
    return QuantizedBlock(codes=codes[0], unit_mins=metas[0, :, 0].clone(),
                          unit_scales=metas[0, :, 1].clone(), block_index=block_index,
                          head_index=block_index % head_num,
                          ctx_start=(block_index // head_num) * block_size)


DECODE_GROUP_SLICES = 8192  # codec.py:38


def iter_decoded_blocks(arena: "DeviceArena", cb, *, n_units: int, head_dim: int, ordinals=None,
                        group_slices: int = DECODE_GROUP_SLICES, movement=None):
    """codec.py:394-452 on the device: arena blocks decoded by
    kvc_decode_blocks in groups of about ``group_slices`` slices (one launch
    per group, so scratch stays bounded).  Yields ``(ordinal, block_index,
    codes [n_slices, head_dim] u8, mins, scales)`` in the order of
    ``ordinals``; tensors live on the arena's device.  A block whose header,
    counters or payload disagree with the codebook raises CodecError."""
    n = len(arena)
    if n == 0:
        return
    which = list(range(n)) if ordinals is None else [int(o) for o in ordinals]
    if not which:
        return
    offs = arena.block_offsets
    cursor = arena.write_cursor

    def extent(o: int) -> Tuple[int, int]:
        if not 0 <= o < n:
            raise CodecError(f"block ordinal {o} out of range")
        return int(offs[o]), (int(offs[o + 1]) if o + 1 < n else cursor)

    # slices per block: the u16 after the block index in the first header
    s0, e0 = extent(which[0])
    if e0 - s0 < 6:
        raise CodecError("block extent shorter than its header")
    bs = int.from_bytes(arena.raw_tensor()[s0 + 4: s0 + 6].cpu().numpy().tobytes(), "little")
    if bs < 1:
        raise CodecError("block with zero slices")
    dev = arena.device
    tables = cb.device_tables(dev)
    per_group = max(1, -(-group_slices // bs))
    for g in range(0, len(which), per_group):
        grp = which[g: g + per_group]
        for o in grp:
            s, e = extent(o)
            if movement is not None:
                movement.add_read(e - s)
        m = len(grp)
        codes = torch.empty((m, bs, head_dim), dtype=torch.uint8, device=dev)
        metas = torch.empty((m, n_units, 2), dtype=torch.float32, device=dev)
        bidx = torch.zeros(m, dtype=torch.int32, device=dev)  # u32 block indices
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        ords = torch.tensor(grp, dtype=torch.int32, device=dev)
        st = _lib.lib().kvc_decode_blocks(arena.buf_ptr, arena.offsets_ptr, arena.counters_ptr,
                                          ords.data_ptr(), m, bs, n_units, head_dim,
                                          tables.data_ptr(), codes.data_ptr(), metas.data_ptr(),
                                          bidx.data_ptr(), err.data_ptr(), _stream(dev))
        _lib.check(st, "iter_decoded_blocks")
        _lib.raise_device_error(int(err.item()), "iter_decoded_blocks")
        if movement is not None:
            movement.note_scratch(codes.numel())
        block_ids = bidx.cpu().numpy().view(np.uint32).tolist()
        for i, o in enumerate(grp):
            yield o, int(block_ids[i]), codes[i], metas[i, :, 0], metas[i, :, 1]


def metadata_overhead(cblocks, head_dim: int) -> Tuple[float, float]:
    """codec.py:455-472: 16-bit slice counters as fractions of the payload and
    of the original 16-bit values."""
    if not cblocks:
        raise CodecError("metadata_overhead needs at least one block")
    n_slices = sum(b.n_slices for b in cblocks)
    payload_bits = sum(b.total_bits for b in cblocks)
    if payload_bits == 0:
        raise CodecError("empty payloads have no meaningful overhead ratio")
    counter_bits = 16 * n_slices
    return counter_bits / payload_bits, counter_bits / (n_slices * head_dim * 16)


def _block_image(cb: CompressedBlock) -> torch.Tensor:
    """_serialize_block (codec.py:229-244) of a block built from its fields."""
    if cb._image is not None:
        return cb._image
    dev = cb.payload.device if isinstance(cb.payload, torch.Tensor) and cb.payload.is_cuda else _dev()
    hdr = np.zeros(6, np.uint8)
    hdr[:4] = np.frombuffer(np.uint32(cb.block_index).tobytes(), np.uint8)
    hdr[4:6] = np.frombuffer(np.uint16(cb.n_slices).tobytes(), np.uint8)
    counts = _to_dev(cb.slice_bit_counts, torch.int32, dev).to(torch.int16).view(torch.uint8)
    metas = torch.stack([_to_dev(cb.unit_mins, torch.float32, dev).reshape(-1),
                         _to_dev(cb.unit_scales, torch.float32, dev).reshape(-1)], 1)
    parts = [torch.from_numpy(hdr).to(dev), counts, metas.contiguous().view(torch.uint8).reshape(-1),
             _to_dev(cb.payload, torch.uint8, dev).reshape(-1)]
    raw = sum(p.numel() for p in parts)
    parts.append(torch.zeros((-raw) % 4, dtype=torch.uint8, device=dev))
    return torch.cat(parts)


def _serialize_block(cblock: CompressedBlock) -> bytes:
    """codec.py:229-244 as bytes (the reference's tests compare block images
    through this helper)."""
    return _block_image(cblock).cpu().numpy().tobytes()


def _arena_append(self: "DeviceArena", cblock: CompressedBlock) -> int:
    """CompressedArena.append (codec.py:308-326): serialise and append one
    block on the device; returns its arrival ordinal.  A full arena raises
    ArenaFullError and is left unchanged."""
    image = _block_image(cblock).to(self.device)
    n = image.numel()
    bits = cblock.total_bits
    self.reserve(1, n)
    st = _lib.lib().kvc_arena_append(image.data_ptr(), n, bits, (bits + 7) // 8, self.buf_ptr,
                                     self.alloc_capacity, self.offsets_ptr, self.counters_ptr,
                                     _stream(self.device))
    _lib.check(st, "CompressedArena.append")
    if self.capacity is not None or self._bound + n > 0xFFFFFFFF:
        c = self.counters()
        if c.err == _lib.KVC_ERR_ARENA_FULL:
            self._counters[36:40].zero_()  # the refused append changed nothing
            raise ArenaFullError(f"arena capacity {self.capacity} exhausted at offset "
                                 f"{int(c.cursor)}")
    ordinal = self.n_blocks
    self.note_append(1, n)
    return ordinal


def _arena_restore(cls, data, offsets, n_units: int, device=None) -> "DeviceArena":
    """CompressedArena.restore (codec.py:329-341): serialised bytes + offsets
    -> a device arena whose counters are recomputed (and every extent
    validated) on the device."""
    dev = _dev(device)
    raw = bytes(data) if not isinstance(data, torch.Tensor) else data.cpu().numpy().tobytes()
    offs = np.asarray([int(o) for o in offsets], dtype=np.uint32)
    arena = cls(device=dev, capacity=None, initial_bytes=max(len(raw), 1),
                initial_blocks=max(len(offs), 1))
    arena.load(raw, offs, bytes(ctypes.sizeof(_lib.ArenaCounters)))
    nsl = torch.zeros(1, dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    st = _lib.lib().kvc_arena_restore(arena.buf_ptr, len(raw), arena.offsets_ptr, len(offs),
                                      int(n_units), arena.counters_ptr, nsl.data_ptr(),
                                      err.data_ptr(), _stream(dev))
    _lib.check(st, "CompressedArena.restore")
    _lib.raise_device_error(int(err.item()), "CompressedArena.restore")
    arena.counters()
    return arena


def _arena_n_slices(self: "DeviceArena") -> int:
    """Running total of slices (codec.py:290): the n_slices header fields."""
    if self.n_blocks == 0:
        return 0
    at = self._offsets[: self.n_blocks].to(torch.int64) & 0xFFFFFFFF
    lo = self._buf[at + 4].to(torch.int64)
    hi = self._buf[at + 5].to(torch.int64)
    return int((lo | (hi << 8)).sum())


DeviceArena.append = _arena_append
DeviceArena.restore = classmethod(_arena_restore)
DeviceArena.n_slices = property(_arena_n_slices)


class CompressedArena(DeviceArena):
    """The reference's constructor signature (codec.py:279-284:
    ``CompressedArena(capacity=None)``) for a device arena on the current
    (or given) CUDA device."""

    def __init__(self, capacity: Optional[int] = None, device=None, initial_bytes: int = 1 << 16,
                 initial_blocks: int = 256):
        super().__init__(_dev(device), capacity, initial_bytes=initial_bytes,
                         initial_blocks=initial_blocks)


# names the reference's codec module also carries (codec.py:19-36 imports)
from .codebook import DecodeTree, HuffmanCodebook  # noqa: E402
from .quantizer import QuantizedBlock, QuantMode  # noqa: E402
