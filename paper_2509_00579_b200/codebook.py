"""Shared canonical Huffman codebooks (reference codebook.py:34-230).

Lengths are computed by the C-ABI host builder ``kvc_codebook_lengths``
(heap with (weight, lowest symbol) ties); ``kvc_codebook_build_tables``
derives canonical codewords, the Kraft check and the device decode tables,
which are uploaded once per (sequence, layer, K|V) and reused for every
append (SPEC: codebooks are immutable after prefill).
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Dict

import numpy as np
import torch

from . import _lib
from .errors import CodebookError

ALPHABET = 256
MAX_CODE_LENGTH = 32


def _as_u64(h) -> np.ndarray:
    if isinstance(h, torch.Tensor):
        h = h.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(h).astype(np.uint64))


def build_histogram(codes) -> torch.Tensor:
    """256-bin histogram of uint8 codes (codebook.py:75-80), on the device."""
    t = codes if isinstance(codes, torch.Tensor) else torch.from_numpy(np.asarray(codes, np.uint8))
    if t.numel() == 0:
        raise CodebookError("cannot build a histogram from an empty input")
    if not t.is_cuda:
        t = t.cuda()
    return torch.bincount(t.reshape(-1).to(torch.int64), minlength=ALPHABET)


def smooth_histogram(h, max_code: int) -> np.ndarray:
    """Add-one smoothing over codes [0, max_code] (codebook.py:83-89)."""
    if not 0 <= max_code < ALPHABET:
        raise CodebookError(f"max_code {max_code} outside [0, 255]")
    out = _as_u64(h).copy()
    out[: max_code + 1] += 1
    return out


def histogram_entropy(h) -> float:
    counts = _as_u64(h).astype(np.float64)
    total = counts.sum()
    if total <= 0:
        raise CodebookError("entropy of an empty histogram is undefined")
    p = counts[counts > 0] / total
    return float(-(p * np.log2(p)).sum())


@dataclass(frozen=True, eq=False)
class DecodeTree:
    """Array-form Huffman tree (codebook.py:35-53): node 0 is the root,
    ``children[n] = [child on 0, child on 1]``, leaves carry ``symbols[n]``
    with ``is_symbol[n] == 1``.  Host arrays as in the reference; the device
    copies (``device(dev)``) feed kvc_decode_slices_tree."""

    children: np.ndarray   # (n_nodes, 2) int32
    is_symbol: np.ndarray  # (n_nodes,) int32
    symbols: np.ndarray    # (n_nodes,) uint8
    _dev: Dict[str, tuple] = field(default_factory=dict, repr=False, compare=False)

    @property
    def n_nodes(self) -> int:
        return int(self.children.shape[0])

    def device(self, dev):
        key = str(torch.device(dev))
        t = self._dev.get(key)
        if t is None:
            t = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                      for a in (self.children.astype(np.int32).reshape(-1),
                                self.is_symbol.astype(np.int32), self.symbols.astype(np.uint8)))
            self._dev[key] = t
        return t


def decode_tree_from_words(lengths: np.ndarray, words: np.ndarray) -> DecodeTree:
    """The reference's node numbering (codebook.py:144-176): symbols are
    inserted in increasing symbol order, each walking its codeword MSB-first
    and appending a fresh node wherever a child is missing; a one-symbol
    alphabet gets a root whose two branches both reach the single leaf."""
    present = np.flatnonzero(np.asarray(lengths) > 0)
    n_max = 1 + int(np.asarray(lengths, np.int64)[present].sum()) + 1
    children = np.zeros((n_max, 2), np.int32)
    is_symbol = np.zeros(n_max, np.int32)
    symbols = np.zeros(n_max, np.uint8)
    n = 1
    if present.size == 1:
        children[0] = (1, 1)
        is_symbol[1], symbols[1] = 1, present[0]
        n = 2
    else:
        for sym in present:
            ln, w, node = int(lengths[sym]), int(words[sym]), 0
            for sh in range(ln - 1, -1, -1):
                b = (w >> sh) & 1
                if children[node, b] == 0:
                    children[node, b] = n
                    n += 1
                node = int(children[node, b])
            is_symbol[node], symbols[node] = 1, sym
    return DecodeTree(children=children[:n].copy(), is_symbol=is_symbol[:n].copy(),
                      symbols=symbols[:n].copy())


@dataclass(eq=False)
class HuffmanCodebook:
    """Canonical code + device decode tables; same fields as the reference."""

    code_lengths: np.ndarray   # (256,) uint8
    code_words: np.ndarray     # (256,) uint32
    max_code_length: int
    tables: _lib.CodebookTables = field(repr=False)
    _device: Dict[str, torch.Tensor] = field(default_factory=dict, repr=False)

    @property
    def decode_tree(self) -> DecodeTree:
        """codebook.py:144-176 (built on first use; the device decoders use
        the LUT tables instead)."""
        t = self._device.get("tree")
        if t is None:
            t = self._device["tree"] = decode_tree_from_words(self.code_lengths, self.code_words)
        return t

    @property
    def encode_table(self):
        present = [s for s in range(ALPHABET) if self.code_lengths[s] > 0]
        present.sort(key=lambda s: (int(self.code_lengths[s]), s))
        return [(s, int(self.code_words[s]), int(self.code_lengths[s])) for s in present]

    def device_tables(self, device) -> torch.Tensor:
        """The kvc_codebook_dev blob on `device` (uploaded once, cached)."""
        dev = torch.device(device)
        key = str(dev)
        t = self._device.get(key)
        if t is None:
            t, ext = _upload(self.tables, dev)
            if ext is not None:  # carved from the arena slab pool: freed with the book
                weakref.finalize(self, ext.release)
            self._device[key] = t
        return t


class _PinnedStage:
    """Ring of pinned host buffers for the codebook-table uploads: an upload
    is one memmove plus an asynchronous H2D copy (a pageable copy of the 52 KB
    blob is synchronous, ~50 us).  A slot is rewritten only after the event of
    its previous copy has completed."""

    def __init__(self, nbytes: int, slots: int = 8):
        self.bufs = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(slots)]
        self.events = [None] * slots
        self.i = 0


_STAGE = {}


def _upload(tables, dev: torch.device) -> torch.Tensor:
    n = ctypes.sizeof(tables)
    if dev.type != "cuda":
        return torch.frombuffer(bytearray(bytes(tables)), dtype=torch.uint8).to(dev), None
    stage = _STAGE.get(n)
    if stage is None:
        stage = _STAGE[n] = _PinnedStage(n)
    i = stage.i
    stage.i = (i + 1) % len(stage.bufs)
    if stage.events[i] is not None:
        stage.events[i].synchronize()
    buf = stage.bufs[i]
    ctypes.memmove(buf.data_ptr(), ctypes.addressof(tables), n)
    # long-lived (one per state and tensor): from the slab pool, so building
    # many states does not grow the caching allocator's small pool (each new
    # 2 MB segment was a cudaMalloc, and under load those took milliseconds)
    from .codec import _pool
    raw, ext = _pool(dev).alloc(n)
    out = raw[:n]
    out.copy_(buf, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(dev))
    stage.events[i] = ev
    return out, ext


# Codebooks by code lengths (a canonical code is a function of its lengths):
# the sequences and layers of a batch mostly end up with the same books, so a
# prefill reuses the host tables and their device copy instead of rebuilding
# and uploading ~100 KB per state and tensor.  Shared books are immutable.
_BOOKS: "OrderedDict[bytes, HuffmanCodebook]" = OrderedDict()
_BOOKS_MAX = 64
_BOOKS_LOCK = threading.Lock()


def codebook_from_lengths(lengths) -> HuffmanCodebook:
    """codebook.py:179-208 via kvc_codebook_build_tables."""
    lens = np.ascontiguousarray(np.asarray(lengths).astype(np.uint8))
    if lens.shape != (ALPHABET,):
        raise CodebookError(f"expected {ALPHABET} code lengths, got shape {lens.shape}")
    key = lens.tobytes()
    with _BOOKS_LOCK:
        cb = _BOOKS.get(key)
        if cb is not None:
            _BOOKS.move_to_end(key)
            return cb
    tables = _lib.CodebookTables()
    st = _lib.lib().kvc_codebook_build_tables(lens.ctypes.data_as(ctypes.c_void_p),
                                              ctypes.byref(tables))
    _lib.check(st, "codebook_from_lengths")
    words = np.frombuffer(bytes(tables.words), dtype=np.uint32).copy()
    lens = lens.copy()
    lens.setflags(write=False)
    words.setflags(write=False)
    cb = HuffmanCodebook(code_lengths=lens, code_words=words,
                         max_code_length=int(tables.max_len), tables=tables)
    with _BOOKS_LOCK:
        _BOOKS[key] = cb
        while len(_BOOKS) > _BOOKS_MAX:
            _BOOKS.popitem(last=False)
    return cb


def build_codebook(h) -> HuffmanCodebook:
    """codebook.py:211-218: optimal lengths, then canonical tables."""
    counts = _as_u64(h)
    if counts.shape != (ALPHABET,):
        raise CodebookError(f"expected a 256-bin histogram, got shape {counts.shape}")
    if counts.sum() == 0:
        raise CodebookError("cannot build a codebook from an empty histogram")
    lens = np.zeros(ALPHABET, np.uint8)
    st = _lib.lib().kvc_codebook_lengths(counts.ctypes.data_as(ctypes.c_void_p), -1,
                                         lens.ctypes.data_as(ctypes.c_void_p))
    _lib.check(st, "build_codebook")
    return codebook_from_lengths(lens)


def build_smoothed_codebook(h, max_code: int) -> HuffmanCodebook:
    """smooth_histogram + build_codebook in one host call (kvcache.py:122-123)."""
    counts = _as_u64(h)
    lens = np.zeros(ALPHABET, np.uint8)
    st = _lib.lib().kvc_codebook_lengths(counts.ctypes.data_as(ctypes.c_void_p), int(max_code),
                                         lens.ctypes.data_as(ctypes.c_void_p))
    _lib.check(st, "build_codebook")
    return codebook_from_lengths(lens)


def serialize_codebook(cb: HuffmanCodebook) -> bytes:
    return bytes(cb.code_lengths.astype(np.uint8).tobytes())


def deserialize_codebook(data: bytes) -> HuffmanCodebook:
    if len(data) != ALPHABET:
        raise CodebookError(f"serialized codebook must be {ALPHABET} bytes, got {len(data)}")
    return codebook_from_lengths(np.frombuffer(data, dtype=np.uint8))
