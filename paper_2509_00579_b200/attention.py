"""Fetch: fused decompress + decode attention (reference attention.py:34-228).

``attention_step`` runs the single-pass fused sm_100a kernel (Huffman decode
-> dequantise -> q.K^T -> online softmax -> .V per context split, then a
combine that also folds in the f32 buffered tokens) whenever the shape is
covered (head_dim 128, block_size 64, codes <= 13 bits); other shapes run the
shape-generic decode-in-the-dot-product kernels (kvc_k_scores ->
kvc_softmax_rows -> kvc_v_output).  Both are CUDA; there is no CPU path.
``attention_batched`` is the batch entry point (many sequences, one launch).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .codec import DataMovement
from .errors import CodecError, ConfigError
from .kvcache import LayerCacheState, _BatchDesc, append_batched  # noqa: F401
from .tensor_io import CacheTensor


@dataclass(frozen=True)
class AttentionOutput:
    out: torch.Tensor     # (head_num, head_dim) float32
    scores: torch.Tensor  # (head_num, context_len) float32, pre-softmax


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check_query(state: LayerCacheState, q) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(q, np.float32)) if not isinstance(q, torch.Tensor) else q
    if tuple(t.shape) != (state.head_num, state.head_dim):
        raise CodecError(f"query must have shape {(state.head_num, state.head_dim)}")
    t = t.to(state.device, torch.float32).contiguous()
    if not bool(torch.isfinite(t).all()):
        raise CodecError("non-finite query rejected")
    return t


def _movement_fetch(state: LayerCacheState, movement: Optional[DataMovement], with_w: bool):
    if movement is None:
        return
    movement.add_read(state.head_num * state.head_dim * 4)              # q
    movement.add_read(state.k_arena.size_bytes + state.v_arena.size_bytes)
    movement.add_read(2 * state.buffered * state.head_num * state.head_dim * 4)
    if with_w:
        movement.add_read(state.head_num * state.context_len * 4)


def fused_k_scores(state: LayerCacheState, q, movement: Optional[DataMovement] = None,
                   n_threads: int = 1) -> torch.Tensor:
    """attention.py:59-109 — logits over the whole context, x 1/sqrt(D)."""
    q32 = _check_query(state, q)
    scores = torch.empty((state.head_num, state.context_len), dtype=torch.float32,
                         device=state.device)
    err = torch.zeros(1, dtype=torch.int32, device=state.device)
    st = _lib.lib().kvc_k_scores(state.desc_device().data_ptr(), 1, state.head_num,
                                 state.head_dim, state.cfg_k.block_size, q32.data_ptr(),
                                 scores.data_ptr(), state.context_len, err.data_ptr(),
                                 _stream(state.device))
    _lib.check(st, "kvc_k_scores")
    _lib.raise_device_error(int(err.item()), "fused_k_scores")
    if movement is not None:
        movement.add_read(q32.numel() * 4 + state.k_arena.size_bytes +
                          state.buffered * state.head_num * state.head_dim * 4)
    return scores


def fused_v_output(state: LayerCacheState, weights, movement: Optional[DataMovement] = None,
                   n_threads: int = 1) -> torch.Tensor:
    """attention.py:112-165 — weighted V aggregation decoded block by block."""
    w = weights if isinstance(weights, torch.Tensor) else torch.as_tensor(
        np.asarray(weights, np.float32))
    H, D = state.head_num, state.head_dim
    if tuple(w.shape) != (H, state.context_len):
        raise CodecError(f"weights must have shape {(H, state.context_len)}")
    w = w.to(state.device, torch.float32).contiguous()
    out = torch.empty((H, D), dtype=torch.float32, device=state.device)
    lib = _lib.lib()
    ws = torch.empty(lib.kvc_v_output_workspace_bytes(1, H, D), dtype=torch.uint8,
                     device=state.device)
    err = torch.zeros(1, dtype=torch.int32, device=state.device)
    st = lib.kvc_v_output(state.desc_device().data_ptr(), 1, H, D, state.cfg_v.block_size,
                          w.data_ptr(), state.context_len, out.data_ptr(), ws.data_ptr(),
                          err.data_ptr(), _stream(state.device))
    _lib.check(st, "kvc_v_output")
    _lib.raise_device_error(int(err.item()), "fused_v_output")
    if movement is not None:
        movement.add_read(w.numel() * 4 + state.v_arena.size_bytes +
                          state.buffered * H * D * 4)
    return out


def softmax_rows(logits) -> torch.Tensor:
    """attention.py:168-173 — stable row softmax, on the device."""
    x = logits if isinstance(logits, torch.Tensor) else torch.as_tensor(
        np.asarray(logits, np.float32))
    x = x.to(torch.float32)
    if not x.is_cuda:
        x = x.cuda()
    x = x.contiguous().clone()
    rows = x.shape[0] if x.ndim > 1 else 1
    st = _lib.lib().kvc_softmax_rows(x.data_ptr(), rows, x.shape[-1], x.shape[-1],
                                     _stream(x.device))
    _lib.check(st, "kvc_softmax_rows")
    return x


FUSED_MAX_CODE_LENGTH = 13  # pair LUT (<= 6), 12-bit and 13-bit single-symbol LUTs


def _state_fused_ok(s: LayerCacheState) -> bool:
    return max(s.k_codebook.max_code_length, s.v_codebook.max_code_length) <= FUSED_MAX_CODE_LENGTH


def _fused_supported(states: Sequence[LayerCacheState]) -> bool:
    s0 = states[0]
    if s0.head_dim != 128 or s0.cfg_k.block_size != 64 or s0.cfg_k.buffer_size >= 1024:
        return False
    return all(_state_fused_ok(s) for s in states)


_default_desc_cache = _BatchDesc()


def _check_batch(states: Sequence[LayerCacheState], q: torch.Tensor, n_q_heads_per_kv: int,
                 out: Optional[torch.Tensor]):
    """Shape/dtype/device validation before raw pointers reach the kernels:
    every state shares (H, D, block size, device); q is a contiguous f32
    [B, H*group, D] tensor on that device, out likewise (ConfigError for
    mixed states, CodecError for tensors, as the reference's shape checks,
    attention.py:44-47)."""
    if len(states) == 0:
        raise ConfigError("attention over an empty batch of states")
    s0 = states[0]
    for s in states[1:]:
        if (s.head_num, s.head_dim, s.cfg_k.block_size, s.device) != (
                s0.head_num, s0.head_dim, s0.cfg_k.block_size, s0.device):
            raise ConfigError("batched states must share head_num, head_dim, block_size and device")
    shape = (len(states), s0.head_num * n_q_heads_per_kv, s0.head_dim)
    if not isinstance(q, torch.Tensor) or tuple(q.shape) != shape:
        raise CodecError(f"query must be a tensor of shape {shape}")
    if q.dtype != torch.float32 or q.device != s0.device or not q.is_contiguous():
        raise CodecError("query must be a contiguous float32 tensor on the states' device")
    if out is not None and (tuple(out.shape) != shape or out.dtype != torch.float32
                            or out.device != s0.device or not out.is_contiguous()):
        raise CodecError(f"out must be a contiguous float32 tensor of shape {shape} on the "
                         "states' device")
    for s in states:
        if s.context_len < 1:
            raise CodecError("attention over an empty context")


def attention_batched(states: Sequence[LayerCacheState], q: torch.Tensor,
                      want_scores: bool = False, desc_cache: Optional[_BatchDesc] = None,
                      workspace: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                      want_err: bool = True):
    """One fused launch over a batch of same-shape states.  q: [B, H, D] f32
    on the device.  Returns (out [B, H, D], scores [B, H, max_ctx] or None,
    err [1] int32: the device error word of this call, or None with
    want_err=False -- the decode loop's fire-and-forget path, which skips the
    per-call zero fill)."""
    _check_batch(states, q, 1, out)
    B = len(states)
    s0 = states[0]
    # a batch mixing books the fused kernel covers (codes <= 13 bits) with
    # longer ones (very fine scales): fused launch for the former, the generic
    # kernels for the rest, instead of the whole batch on the generic path
    ok = [_state_fused_ok(s) for s in states]
    shape_ok = s0.head_dim == 128 and s0.cfg_k.block_size == 64 and s0.cfg_k.buffer_size < 1024
    if shape_ok and any(ok) and not all(ok):
        cache = desc_cache if desc_cache is not None else _BatchDesc()
        if getattr(cache, "split", None) is None:
            cache.split = (_BatchDesc(), _BatchDesc())
        if out is None:
            out = torch.empty((B, s0.head_num, s0.head_dim), dtype=torch.float32, device=s0.device)
        max_ctx = max(s.context_len for s in states)
        scores = (torch.zeros((B, s0.head_num, max_ctx), dtype=torch.float32, device=s0.device)
                  if want_scores else None)
        errs = []
        for sub_ok, sub_cache in ((True, cache.split[0]), (False, cache.split[1])):
            idx = [i for i in range(B) if ok[i] == sub_ok]
            it = torch.tensor(idx, device=s0.device)
            o, sc, e = attention_batched([states[i] for i in idx], q.index_select(0, it).contiguous(),
                                         want_scores=want_scores, desc_cache=sub_cache,
                                         want_err=True)
            out.index_copy_(0, it, o)
            if want_scores:
                scores[it, :, : sc.shape[-1]] = sc
            errs.append(e)
        err = torch.maximum(errs[0], errs[1])
        return out, scores, (err if want_err else None)
    H, D, bs = s0.head_num, s0.head_dim, s0.cfg_k.block_size
    dev = s0.device
    lib = _lib.lib()
    max_ctx = max(s.context_len for s in states)
    max_chunks = max(s.n_chunks for s in states)
    if out is None:
        out = torch.empty((B, H, D), dtype=torch.float32, device=dev)
    scores = torch.zeros((B, H, max_ctx), dtype=torch.float32, device=dev) if want_scores else None
    cache = desc_cache if desc_cache is not None else _BatchDesc()
    if want_err or not _fused_supported(states):
        err = torch.zeros(1, dtype=torch.int32, device=dev)
    else:
        if getattr(cache, "scratch_err", None) is None or cache.scratch_err.device != dev:
            cache.scratch_err = torch.zeros(1, dtype=torch.int32, device=dev)
        err = cache.scratch_err
    ddev, dhost = cache.get(states)
    if _fused_supported(states):
        need = lib.kvc_attention_workspace_bytes(B, H, 1, D, max_chunks)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=dev)
        st = lib.kvc_attention(ddev.data_ptr(), ctypes_addr(dhost), B, H, D, bs, 1,
                               q.data_ptr(), out.data_ptr(),
                               scores.data_ptr() if scores is not None else None, max_ctx,
                               workspace.data_ptr(), workspace.numel(), err.data_ptr(),
                               _stream(dev))
        _lib.check(st, "kvc_attention")
    else:
        sc = scores if scores is not None else torch.zeros((B, H, max_ctx), dtype=torch.float32,
                                                           device=dev)
        st = lib.kvc_k_scores(ddev.data_ptr(), B, H, D, bs, q.data_ptr(), sc.data_ptr(), max_ctx,
                              err.data_ptr(), _stream(dev))
        _lib.check(st, "kvc_k_scores")
        w = sc.clone()
        for b, s in enumerate(states):
            st = lib.kvc_softmax_rows(w[b].data_ptr(), H, s.context_len, max_ctx, _stream(dev))
            _lib.check(st, "kvc_softmax_rows")
            if s.context_len < max_ctx:
                w[b, :, s.context_len:] = 0
        ws = torch.empty(lib.kvc_v_output_workspace_bytes(B, H, D), dtype=torch.uint8, device=dev)
        st = lib.kvc_v_output(ddev.data_ptr(), B, H, D, bs, w.data_ptr(), max_ctx, out.data_ptr(),
                              ws.data_ptr(), err.data_ptr(), _stream(dev))
        _lib.check(st, "kvc_v_output")
        scores = sc if want_scores else None
    return out, scores, (err if want_err else None)


def ctypes_addr(arr) -> int:
    import ctypes
    return ctypes.addressof(arr)


def attention_step(state: LayerCacheState, q, movement: Optional[DataMovement] = None,
                   n_threads: int = 1) -> AttentionOutput:
    """attention.py:176-188 — one decode step; returns (out, scores)."""
    if state.context_len < 1:
        raise CodecError("attention over an empty context")
    q32 = _check_query(state, q)
    out, scores, err = attention_batched([state], q32.unsqueeze(0), want_scores=True)
    _lib.raise_device_error(int(err.item()), "attention_step")
    _movement_fetch(state, movement, with_w=False)
    return AttentionOutput(out=out[0], scores=scores[0])


def reference_scores(k: CacheTensor, q, movement: Optional[DataMovement] = None) -> torch.Tensor:
    """attention.py:191-202 — dense matvec on a materialised K (device)."""
    vals = k.values if isinstance(k.values, torch.Tensor) else torch.from_numpy(k.as_float32())
    vals = vals.to(torch.float32).cuda() if not vals.is_cuda else vals.to(torch.float32)
    q32 = (q if isinstance(q, torch.Tensor) else torch.as_tensor(np.asarray(q, np.float32)))
    q32 = q32.to(vals.device, torch.float32)
    if tuple(q32.shape) != (k.head_num, k.head_dim):
        raise CodecError(f"query must have shape {(k.head_num, k.head_dim)}")
    if movement is not None:
        movement.add_read(vals.numel() * 4 + q32.numel() * 4)
    return torch.einsum("thd,hd->ht", vals, q32) * np.float32(1.0 / math.sqrt(k.head_dim))


def reference_output(v: CacheTensor, weights, movement: Optional[DataMovement] = None):
    """attention.py:205-215 — dense weighted V sum on a materialised V (device)."""
    vals = v.values if isinstance(v.values, torch.Tensor) else torch.from_numpy(v.as_float32())
    vals = vals.to(torch.float32).cuda() if not vals.is_cuda else vals.to(torch.float32)
    w = weights if isinstance(weights, torch.Tensor) else torch.as_tensor(
        np.asarray(weights, np.float32))
    w = w.to(vals.device, torch.float32)
    if tuple(w.shape) != (v.head_num, v.context_len):
        raise CodecError(f"weights must have shape {(v.head_num, v.context_len)}")
    if movement is not None:
        movement.add_read(vals.numel() * 4 + w.numel() * 4)
    return torch.einsum("ht,thd->hd", w, vals)


def multistage_attention(state: LayerCacheState, q,
                         movement: Optional[DataMovement] = None) -> AttentionOutput:
    """attention.py:218-228 — unfused: decode+dequantise, then dense passes."""
    k, v = state.fetch_dequantized()
    scores = reference_scores(k, q, movement=movement)
    weights = softmax_rows(scores)
    out = reference_output(v, weights, movement=movement)
    return AttentionOutput(out=out, scores=scores)


def attention_gqa(states: Sequence[LayerCacheState], q: torch.Tensor, group: int,
                  desc_cache: Optional["_BatchDesc"] = None,
                  workspace: Optional[torch.Tensor] = None, check: bool = True,
                  out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Grouped-query decode attention: q [B, H_kv*group, D], query head
    h*group+j reads KV head h (Llama-3 layout).  The reference has no GQA
    (SPEC non-goal; its oracle runs one attention_step per group member).
    Groups of 2 or 4 with codes <= 6 bits run the decode-once GQA kernel
    (each K/V block decoded once for all members); otherwise one fused
    launch per member.  check=True synchronises and raises the device error
    word (CodecError on a corrupt stream); check=False leaves the launch
    asynchronous (the bench's decode loop)."""
    if not isinstance(group, int) or group < 1:
        raise ConfigError("group must be a positive integer")
    if q.ndim != 3 or q.shape[1] % group != 0:
        raise CodecError("query heads must be a multiple of the group size")
    _check_batch(states, q, group, out)
    B, HQ, D = q.shape
    H = HQ // group
    dev = q.device
    if out is None:
        out = torch.empty((B, HQ, D), dtype=torch.float32, device=dev)
    cache = desc_cache if desc_cache is not None else _BatchDesc()
    if group in (2, 4) and _fused_supported(states) and all(
            max(s.k_codebook.max_code_length, s.v_codebook.max_code_length) <= 6 for s in states):
        lib = _lib.lib()
        ddev, dhost = cache.get(states)
        max_chunks = max(s.n_chunks for s in states)
        need = lib.kvc_attention_workspace_bytes(B, H, group, D, max_chunks)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=dev)
        if check:
            err = torch.zeros(1, dtype=torch.int32, device=dev)
        else:
            # never read on this path: a per-cache scratch word, not zeroed (one
            # fill launch less per decode step)
            if getattr(cache, "scratch_err", None) is None or cache.scratch_err.device != dev:
                cache.scratch_err = torch.zeros(1, dtype=torch.int32, device=dev)
            err = cache.scratch_err
        qc = q.contiguous()
        st = lib.kvc_attention(ddev.data_ptr(), ctypes_addr(dhost), B, H, D,
                               states[0].cfg_k.block_size, group, qc.data_ptr(), out.data_ptr(),
                               None, 0, workspace.data_ptr(), workspace.numel(), err.data_ptr(),
                               _stream(dev))
        if st == _lib.KVC_OK:
            if check:
                _lib.raise_device_error(int(err.item()), "attention_gqa")
            return out
    qv = q.view(B, H, group, D)
    ov = out.view(B, H, group, D)
    for j in range(group):
        o, _, err = attention_batched(states, qv[:, :, j].contiguous(), desc_cache=cache,
                                      workspace=workspace)
        if check:
            _lib.raise_device_error(int(err.item()), "attention_gqa")
        ov[:, :, j] = o
    return out


def dense_attention_f16(k: torch.Tensor, v: torch.Tensor, q: torch.Tensor,
                        out: Optional[torch.Tensor] = None,
                        workspace: Optional[torch.Tensor] = None, group: int = 1) -> torch.Tensor:
    """Uncompressed fp16 decode attention (north-star comparator kernel).
    k, v: [S, H, ctx, D] f16 contiguous on the device; q: [S, H*group, D] f32
    (GQA: K/V rows are read once for all `group` query heads)."""
    S, H, ctx, D = k.shape
    lib = _lib.lib()
    need = lib.kvc_dense_workspace_bytes(S, H, group, D, ctx)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=k.device)
    if out is None:
        out = torch.empty((S, H * group, D), dtype=torch.float32, device=k.device)
    st = lib.kvc_dense_attention_f16(k.data_ptr(), v.data_ptr(), S, H, D, group, ctx,
                                     q.data_ptr(), out.data_ptr(), workspace.data_ptr(),
                                     workspace.numel(), _stream(k.device))
    _lib.check(st, "kvc_dense_attention_f16")
    return out
