"""A multi-layer decode step over resident compressed caches, optionally as
one CUDA graph.

One step appends each layer's new token rows to that layer's batch of
LayerCacheStates (the growing-cache Store, kvcache.py:150-177) and runs the
fused fetch-attention over them -- the reference's decode loop
(bench.py:207-330: attention_step + append_token per step) for a whole model
and batch.  Between overflow events every launch parameter is fixed (the
descriptors are stable, the token counts live on the device), so the step's
~2 launches per layer are captured once and replayed; a step that overflows a
buffer runs eagerly (its Store launches depend on the arena cursors) and the
graph is captured again afterwards.
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from .attention import attention_batched, attention_gqa
from .kvcache import LayerCacheState, _BatchDesc, append_batched


class DecodeLoop:
    """states[l] = the batch of states of layer l (same shape across layers).
    ``step(k_new, v_new, q, out)`` with k_new/v_new [L, B, H, D] (f16/f32) and
    q/out [L, B, H*group, D] f32 device tensors."""

    def __init__(self, states: Sequence[Sequence[LayerCacheState]], group: int = 1,
                 use_graph: bool = True):
        self.states: List[List[LayerCacheState]] = [list(r) for r in states]
        self.group = group
        self.use_graph = use_graph and torch.cuda.is_available()
        self.caches = [_BatchDesc() for _ in self.states]
        self.graph = None
        self.graph_io = None
        self.events = 0        # steps that ran an overflow event
        self.captures = 0
        s0 = self.states[0][0]
        self._ws = torch.empty(0, dtype=torch.uint8, device=s0.device)
        self._stream = torch.cuda.Stream(s0.device) if self.use_graph else None

    # ------------------------------------------------------------------
    def _attend(self, layer: int, q: torch.Tensor, out: torch.Tensor) -> None:
        row = self.states[layer]
        if self.group == 1:
            attention_batched(row, q, desc_cache=self.caches[layer], workspace=self._ws, out=out,
                              want_err=False)
        else:
            attention_gqa(row, q, self.group, desc_cache=self.caches[layer], workspace=self._ws,
                          check=False, out=out)

    def _eager(self, k_new, v_new, q, out) -> None:
        for layer, row in enumerate(self.states):
            append_batched(row, k_new[layer], v_new[layer], desc_cache=self.caches[layer])
            self._attend(layer, q[layer], out[layer])

    def _overflows(self) -> bool:
        return any(r[0].buffered + 1 > r[0].cfg_k.buffer_size for r in self.states) or any(
            s.buffered != r[0].buffered for r in self.states for s in r)

    def _reserve_workspace(self) -> None:
        from . import _lib
        s0 = self.states[0][0]
        B, H = len(self.states[0]), s0.head_num
        mc = max(s.n_chunks for r in self.states for s in r)
        need = _lib.lib().kvc_attention_workspace_bytes(B, H, self.group, s0.head_dim, mc + 8)
        if self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=s0.device)

    def _capture(self, k_new, v_new, q, out) -> None:
        """Record one step as a graph.  The capture itself performs no work:
        the host mirrors it advanced are rolled back."""
        for r in self.states:
            for s in r:
                s.settle()  # exact stage sizes before they are baked into the graph
        self._reserve_workspace()
        # descriptors uploaded (and workspace sized) outside the capture
        for layer, row in enumerate(self.states):
            self.caches[layer].get(row)
        saved = [(s.buffered, s.context_len) for r in self.states for s in r]
        # capture_begin/end directly: the torch.cuda.graph context manager
        # also synchronises, runs gc.collect() and empties the allocator cache
        # (~1 s with a large resident cache), on every re-capture
        dev = self.states[0][0].device
        g = torch.cuda.CUDAGraph()
        self.graph = None  # its private memory pool goes with it
        stream = self._stream
        stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(stream):
            g.capture_begin()
            try:
                self._eager(k_new, v_new, q, out)
            finally:
                g.capture_end()
        torch.cuda.current_stream(dev).wait_stream(stream)
        it = iter(saved)
        for r in self.states:
            for s in r:
                s.buffered, s.context_len = next(it)
        self.graph = g
        self.graph_io = (k_new.data_ptr(), v_new.data_ptr(), q.data_ptr(), out.data_ptr())
        self.captures += 1

    def step(self, k_new: torch.Tensor, v_new: torch.Tensor, q: torch.Tensor,
             out: torch.Tensor) -> torch.Tensor:
        if self._overflows():
            self.graph = None
            self.events += 1
            self._reserve_workspace()
            self._eager(k_new, v_new, q, out)
            return out
        if not self.use_graph:
            self._reserve_workspace()
            self._eager(k_new, v_new, q, out)
            return out
        io = (k_new.data_ptr(), v_new.data_ptr(), q.data_ptr(), out.data_ptr())
        if self.graph is None or io != self.graph_io:
            # re-capture with exact stage sizes: _capture waits for the arenas'
            # max-extent readbacks (the host is usually far ahead of the device
            # here, so the wait overlaps queued work; the device idles only
            # during the capture itself)
            self._capture(k_new, v_new, q, out)
        self.graph.replay()
        for r in self.states:
            for s in r:
                s._after_append()  # cannot overflow: checked above
        return out
