"""Multi-GPU (batch, KV-head) sharding of the compressed cache.

One process per GPU; rank r owns KV heads [r*H/P, (r+1)*H/P) of every
(sequence, layer).  The path has exactly two exchange steps, both tiny:

* Store / prefill: codebooks are built from the code histograms of *all*
  heads (reference kvcache.py:116-121), so ranks all-reduce the 2 x 256-bin
  histogram before the host Huffman build.  Every rank then holds identical
  codebooks and its blocks are byte-identical to the single-process arena's
  blocks with the same block_index (quantizer.py:201 numbering is kept
  global via head_base / head_total).
* Fetch: each rank computes attention for its heads only; the per-head
  outputs [B, H/P, D] are all-gathered (NCCL over NVLink on B200).

Appends need no collective (codebooks are fixed after prefill).  The host
helpers here are backend-agnostic so the same code runs over ``gloo`` in the
CPU tests.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import List, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    head_total: int

    def __post_init__(self):
        if self.head_total % self.world:
            raise ValueError(f"{self.head_total} heads do not split over {self.world} ranks")

    @property
    def heads_local(self) -> int:
        return self.head_total // self.world

    @property
    def head_base(self) -> int:
        return self.rank * self.heads_local

    def slice(self, x):
        """This rank's heads of a [ctx, H, D] tensor (contiguous copy)."""
        s = x[:, self.head_base: self.head_base + self.heads_local]
        return s.contiguous() if isinstance(s, torch.Tensor) else np.ascontiguousarray(s)


def allreduce_histograms(hist: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the concatenated K|V code histograms (int64 [512]) over ranks."""
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def gather_head_outputs(out_local: torch.Tensor, group=None) -> torch.Tensor:
    """[B, H/P, D] per rank -> [B, H, D] on every rank (rank order = head order)."""
    if not (dist.is_available() and dist.is_initialized()):
        return out_local
    world = dist.get_world_size(group)
    parts = [torch.empty_like(out_local) for _ in range(world)]
    dist.all_gather(parts, out_local.contiguous(), group=group)
    return torch.cat(parts, dim=1)


_HDR = struct.Struct("<IH")


def split_blocks(arena: bytes, offsets: Sequence[int]) -> List[bytes]:
    ends = list(offsets[1:]) + [len(arena)]
    return [arena[int(s): int(e)] for s, e in zip(offsets, ends)]


def interleave_shard_arenas(shards: Sequence[Tuple[bytes, Sequence[int]]]) -> Tuple[bytes, np.ndarray]:
    """Reassemble per-rank arenas into the single-process arena: blocks are
    self-describing (block_index in the header, codec.py:229-244), so the
    global arena is all blocks sorted by block_index, offsets re-scanned."""
    blocks = []
    for arena, offsets in shards:
        for blk in split_blocks(arena, offsets):
            (bi, _), = [_HDR.unpack_from(blk, 0)]
            blocks.append((bi, blk))
    blocks.sort(key=lambda t: t[0])
    out = bytearray()
    offs = []
    for _, blk in blocks:
        offs.append(len(out))
        out += blk
    return bytes(out), np.asarray(offs, np.uint32)
