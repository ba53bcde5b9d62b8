"""Device-resident compressed arena (reference codec.py:271-348) and counters.

The arena bytes are exactly the reference's serialisation (codec.py:229-244),
block after block in block_index order, so ``snapshot()`` is byte-comparable
with ``CompressedArena.snapshot()``.  Offsets and running totals live on the
device (``kvc_arena_counters``) and are advanced by the Store kernels; the
host reads them only when asked (stats, snapshot, error checks).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from .errors import ArenaFullError, CodecError

TMA_SLACK = 64  # bytes after the cursor the fetch kernel may over-read


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
        self._buf = torch.empty(alloc + TMA_SLACK, dtype=torch.uint8, device=self.device)
        self._offsets = torch.empty(max(initial_blocks, 1), dtype=torch.int32, device=self.device)
        self._counters = torch.zeros(ctypes.sizeof(_lib.ArenaCounters), dtype=torch.uint8,
                                     device=self.device)
        self.n_blocks = 0          # host mirror (deterministic)
        self._bound = 0            # host upper bound on the cursor

    # ---- growth -------------------------------------------------------
    def reserve(self, n_blocks: int, worst_bytes: int) -> None:
        """Make room for n_blocks more blocks of at most worst_bytes total."""
        need_blocks = self.n_blocks + n_blocks
        if need_blocks > self._offsets.numel():
            new = torch.empty(max(need_blocks, 2 * self._offsets.numel()), dtype=torch.int32,
                              device=self.device)
            new[: self.n_blocks] = self._offsets[: self.n_blocks]
            self._offsets = new
        if self.capacity is not None:
            return  # fixed capacity: the device reports ArenaFullError
        need = self._bound + worst_bytes
        if need > self._buf.numel() - TMA_SLACK:
            new_cap = max(need, 2 * (self._buf.numel() - TMA_SLACK))
            new = torch.empty(new_cap + TMA_SLACK, dtype=torch.uint8, device=self.device)
            new[: self._buf.numel()] = self._buf
            self._buf = new

    def compact(self, headroom: int = 0) -> None:
        """Shrink the allocation to the written bytes (+headroom) after a big prefill."""
        if self.capacity is not None:
            return
        cur = int(self.counters().cursor)
        size = cur + headroom
        if size + TMA_SLACK < self._buf.numel():
            new = torch.empty(size + TMA_SLACK, dtype=torch.uint8, device=self.device)
            new[:cur] = self._buf[:cur]
            self._buf = new

    def load(self, data: bytes, offsets: np.ndarray, counters: bytes, headroom: int = 1 << 16):
        """Replace the contents with serialised blocks (container restore)."""
        n = len(data)
        cap = n + headroom if self.capacity is None else self.capacity
        if self.capacity is not None and n > self.capacity:
            raise ArenaFullError("restored arena exceeds capacity")
        buf = torch.zeros(cap + TMA_SLACK, dtype=torch.uint8)
        buf[:n] = torch.frombuffer(bytearray(data), dtype=torch.uint8) if n else buf[:0]
        self._buf = buf.to(self.device)
        nb = len(offsets)
        offs = torch.zeros(max(nb, 1), dtype=torch.int32)
        if nb:
            offs[:nb] = torch.from_numpy(np.asarray(offsets, np.uint32).view(np.int32).copy())
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
    @property
    def buf_ptr(self) -> int:
        return self._buf.data_ptr()

    @property
    def offsets_ptr(self) -> int:
        return self._offsets.data_ptr()

    @property
    def counters_ptr(self) -> int:
        return self._counters.data_ptr()

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
