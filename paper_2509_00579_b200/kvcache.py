"""Device-backed LayerCacheState — drop-in for reference kvcache.py:29-268.

Same lifecycle and numbers as the reference: prefill quantises all full
blocks, histograms their codes (all heads together, kvcache.py:116-121),
builds the two shared smoothed Huffman codebooks, appends K blocks then V
blocks in block_index order; the residual stays in f32 buffers
(``buffer_size + 1`` slots); ``append_token`` compresses the largest
block-multiple prefix once ``buffered > buffer_size`` (kvcache.py:168-177).

B200 specifics: arenas, offsets, counters, buffers and codebook tables live
in HBM; Store work is two kernels per tensor (quantise+histogram, encode+
append); the only host round trip at prefill is the 2 x 256-bin histogram
(all-reduced across head shards when a process group is given).
"""

from __future__ import annotations

from typing import Optional, Tuple

import functools
import threading
import weakref

import numpy as np
import torch

from . import _lib
from .codebook import HuffmanCodebook, build_smoothed_codebook
from .codec import DeviceArena, pooled_zeros, readback_extents, worst_block_bytes
from .errors import CodecError, ConfigError
from .quantizer import QuantConfig, QuantMode, as_device_tensor, dtype_code, quantize_tokens
from .tensor_io import CacheTensor

MAX_SLICE_BITS = 0xFFFF


class _HistRing:
    """Pinned host slots for the prefill histogram readback (allocated once:
    a pinned allocation per prefill costs a cudaHostAlloc).  A slot is reused
    only after the event of its previous copy has completed, and callers
    consume a slot (prefill_many: at most two in flight) long before the
    ring wraps."""

    def __init__(self, slots: int = 8):
        self.bufs = [torch.empty(512, dtype=torch.int64, pin_memory=True) for _ in range(slots)]
        self.events = [torch.cuda.Event() for _ in range(slots)]  # re-recorded per use
        self.used = [False] * slots
        self.i = 0


_HIST_RINGS = {}


class _Done:
    """An already-completed event (host data that is ready)."""

    @staticmethod
    def synchronize() -> None:
        return None


_DONE = _Done()

_EMPTY = {}


def _empty_ws(device: torch.device) -> torch.Tensor:
    """A shared zero-size workspace placeholder (replaced, never written,
    when a state first needs scratch)."""
    t = _EMPTY.get(device)
    if t is None:
        t = _EMPTY[device] = torch.empty(0, dtype=torch.uint8, device=device)
    return t


@functools.lru_cache(maxsize=256)
def _store_supported(bs: int, D: int, max_len: int) -> bool:
    return bool(_lib.lib().kvc_store_supported(bs, D, max_len))


@functools.lru_cache(maxsize=256)
def _prefill_supported(bs: int, D: int, rel_k: float, rel_v: float) -> bool:
    return bool(_lib.lib().kvc_store_prefill_supported(bs, D, rel_k, rel_v))


@functools.lru_cache(maxsize=256)
def _store_ws_bytes(n_chunks: int, H: int, D: int, bs: int) -> int:
    return int(_lib.lib().kvc_store_workspace_bytes(n_chunks, H, D, bs))


class _SharedRelease:
    """One slab-pool extent shared by the states of a grouped prefill: given
    back when the last of them is released."""
    __slots__ = ("ext", "n", "lock")

    def __init__(self, ext, n: int):
        self.ext, self.n, self.lock = ext, n, threading.Lock()

    def release(self) -> None:
        with self.lock:
            self.n -= 1
            last = self.n == 0
        if last:
            self.ext.release()


class _GroupRing:
    """Pinned [group, 512] slots for the grouped histogram readback (events
    re-recorded; at most two groups are in flight)."""

    def __init__(self, rows: int, slots: int = 4):
        self.bufs = [torch.empty((rows, 512), dtype=torch.int64, pin_memory=True)
                     for _ in range(slots)]
        self.events = [torch.cuda.Event() for _ in range(slots)]
        self.used = [False] * slots
        self.i = 0


_GROUP_RINGS = {}
PREFILL_GROUP = 8  # items per grouped prefill launch batch


@functools.lru_cache(maxsize=256)
def _prefill_scratch_bytes(n_chunks: int, H: int, D: int, bs: int):
    """(per-block histograms, codes, workspace) bytes, each rounded to 256."""
    lib = _lib.lib()
    r = lambda x: (int(x) + 255) & ~255  # noqa: E731
    codes = lib.kvc_store_codes_bytes(n_chunks, H) if (D == 128 and bs == 64) else 0
    return (r(lib.kvc_store_blk_hist_bytes(n_chunks, H)), r(codes),
            r(lib.kvc_store_workspace_bytes(n_chunks, H, D, bs)))


def _hist_readback(hist: torch.Tensor):
    r = _HIST_RINGS.get(hist.device)  # per device: the slots' events are re-recorded
    if r is None:
        with torch.cuda.device(hist.device):
            r = _HIST_RINGS[hist.device] = _HistRing()
    i = r.i
    r.i = (i + 1) % len(r.bufs)
    ev = r.events[i]
    if r.used[i]:
        ev.synchronize()
    buf = r.bufs[i]
    buf.copy_(hist, non_blocking=True)
    ev.record(torch.cuda.current_stream(hist.device))
    r.used[i] = True
    return buf, ev


class LayerCacheState:
    """Compressed KV cache of a single layer (one sequence), resident in HBM."""

    def __init__(self, head_num: int, head_dim: int, cfg_k: QuantConfig, cfg_v: QuantConfig,
                 k_codebook: HuffmanCodebook, v_codebook: HuffmanCodebook, dtype=np.float32,
                 k_channel_ranges=None, device=None, head_base: int = 0,
                 head_total: Optional[int] = None, capacity: Optional[int] = None,
                 arena_bytes: Optional[Tuple[int, int]] = None, arena_blocks: int = 256,
                 page_pool=None, _pre: Optional[dict] = None):
        if not cfg_k.mode.is_key:
            raise ConfigError("cfg_k must use a K quantization mode")
        if cfg_v.mode is not QuantMode.V_TOKEN:
            raise ConfigError("cfg_v must use the V_TOKEN mode")
        if cfg_k.block_size != cfg_v.block_size or cfg_k.buffer_size != cfg_v.buffer_size:
            raise ConfigError("K and V must share block_size and buffer_size")
        if head_dim * 32 > MAX_SLICE_BITS:
            raise ConfigError("head_dim too large for 16-bit slice counters")
        if cfg_k.mode is QuantMode.K_CHANNEL and k_channel_ranges is None:
            raise ConfigError("K_CHANNEL mode requires whole-context channel ranges")
        self.head_num = head_num
        self.head_dim = head_dim
        self.cfg_k = cfg_k
        self.cfg_v = cfg_v
        self.k_codebook = k_codebook
        self.v_codebook = v_codebook
        self.dtype = np.dtype(dtype)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        # K_CHANNEL whole-context ranges: f32 [2, H, D] on the device (kvcache.py:104-108)
        self._k_ranges = None
        self.k_channel_ranges = None
        if k_channel_ranges is not None:
            mins, maxs = k_channel_ranges
            t = torch.stack([torch.as_tensor(np.asarray(m, np.float32)) if not isinstance(
                m, torch.Tensor) else m.to(torch.float32).cpu() for m in (mins, maxs)])
            self._k_ranges = t.to(self.device).contiguous()
            self.k_channel_ranges = (t[0].numpy(), t[1].numpy())
        self.head_base = head_base
        self.head_total = head_total if head_total is not None else head_num
        # arena_bytes: initial allocations sized by the caller (prefill knows a
        # tight bound), so the prefill does not grow 64 KB arenas by a copy
        ka, va = arena_bytes if arena_bytes is not None else (1 << 16, 1 << 16)
        # the two arenas' counters and the live {n_chunks, buffered} pair share
        # one zeroed pool allocation (one allocation and one fill per state)
        if _pre is not None and "small" in _pre:  # carved by prefill (released with _pre's extents)
            small = _pre["small"]
        elif self.device.type == "cuda":
            small, ext = pooled_zeros((128,), torch.uint8, self.device)
            weakref.finalize(self, ext.release)
        else:
            small = torch.zeros(128, dtype=torch.uint8, device=self.device)
        # page_pool: the arenas map pages of a shared PagePool (paged.py)
        # instead of slab-pool extents
        if page_pool is not None:
            from .paged import PagedArena
            mk = lambda nb, cnt: PagedArena(self.device, capacity, initial_bytes=nb,  # noqa: E731
                                            initial_blocks=arena_blocks, counters=cnt,
                                            pool=page_pool)
        else:
            mk = lambda nb, cnt: DeviceArena(self.device, capacity, initial_bytes=nb,  # noqa: E731
                                             initial_blocks=arena_blocks, counters=cnt)
        self.page_pool = page_pool
        self.k_arena = mk(ka, small[0:40])
        self.v_arena = mk(va, small[48:88])
        cap = cfg_k.buffer_size + 1
        if _pre is not None:  # allocated by prefill while its pass A ran
            self._k_buffer, self._v_buffer = _pre["k_buffer"], _pre["v_buffer"]
            for ext in _pre.get("extents", ()):
                weakref.finalize(self, ext.release)
        else:
            self._k_buffer = torch.zeros((cap, head_num, head_dim), dtype=torch.float32,
                                         device=self.device)
            self._v_buffer = torch.zeros_like(self._k_buffer)
        self._k_tab = k_codebook.device_tables(self.device)
        self._v_tab = v_codebook.device_tables(self.device)
        self._ws = _empty_ws(self.device)
        # live {n_chunks, buffered} on the device (kvc_seq_desc.live): the
        # growing-cache kernels update it, the fetch kernels read it, so the
        # descriptor stays the same across decode steps; the host keeps
        # deterministic mirrors (compressed_tokens, buffered)
        self._live = small[96:104].view(torch.int32)
        self.context_len = 0
        self.compressed_tokens = 0
        self.buffered = 0
        self._desc_dev = None
        self._desc_key = None
        self._fused_store = _store_supported(cfg_k.block_size, head_dim,
                                             max(k_codebook.max_code_length,
                                                 v_codebook.max_code_length))

    # ------------------------------------------------------------------
    @classmethod
    def prefill(cls, k, v, cfg_k: QuantConfig, cfg_v: QuantConfig,
                codebooks: Optional[Tuple[HuffmanCodebook, HuffmanCodebook]] = None,
                k_channel_ranges=None, device=None, process_group=None, head_base: int = 0,
                head_total: Optional[int] = None, capacity: Optional[int] = None,
                check: bool = True, page_pool=None) -> "LayerCacheState":
        """kvcache.py:76-145.  k, v: CacheTensor / ndarray / torch tensor
        [ctx, H, D] f16|f32.  With ``process_group`` this rank holds heads
        [head_base, head_base+H) of head_total, and the code histograms are
        all-reduced so every rank builds the same codebooks.  With
        ``page_pool`` (paged.PagePool) the arenas are paged."""
        return cls._prefill_finish(cls._prefill_begin(
            k, v, cfg_k, cfg_v, codebooks, k_channel_ranges, device, process_group, head_base,
            head_total, capacity, page_pool=page_pool), check)

    @classmethod
    def prefill_many(cls, items, cfg_k: QuantConfig, cfg_v: QuantConfig,
                     check: bool = True, **kw) -> list:
        """prefill() of several (k, v) pairs (the layers or sequences of one
        prompt), pipelined: pass A of item i+1 is launched before the host
        builds item i's codebooks, so the GPU runs it while the host works and
        the per-item host time (histogram readback, Huffman build, table
        upload: ~0.3 ms) hides behind device time.  Results are identical to
        calling prefill() on each item."""
        items = list(items)
        out = []
        group = kw.get("process_group")
        if group is not None and kw.get("codebooks") is None and len(items) > 1:
            # head-sharded prefill: every item's pass A first, then ONE all-reduce
            # of the stacked [n_items, 2 x 256] histograms, then the
            # codebook builds and pass B
            kw1 = dict(kw, process_group=None, _defer_hist=True)
            begun = [cls._prefill_begin(k, v, cfg_k, cfg_v, **kw1) for k, v in items]
            hists = torch.stack([c["hist"] for c in begun])
            torch.distributed.all_reduce(hists, group=group)
            hh = hists.cpu()  # one readback for the whole batch
            for c, h in zip(begun, hh.unbind(0)):
                c["hist_host"], c["ev"] = h, _DONE
            out = [cls._prefill_finish(c, False) for c in begun]
            if check:
                for st in out:
                    st.check()
            return out
        if cls._prefill_group_ok(items, cfg_k, cfg_v, kw):
            # many equal slices (the sequences of a batch): pass A, allocations
            # and the histogram readback per group of PREFILL_GROUP items, the
            # next group's launched before this group's codebooks and pass B
            hk = {k: kw[k] for k in ("head_base", "head_total") if k in kw}
            # at most PREFILL_GROUP items and ~1 GiB of pass-A scratch per group
            ctx, H, D = items[0][0].shape
            one = sum(_prefill_scratch_bytes(ctx // cfg_k.block_size, H, D, cfg_k.block_size))
            G = max(1, min(PREFILL_GROUP, (1 << 30) // max(one, 1)))
            groups = [items[i:i + G] for i in range(0, len(items), G)]
            nxt = cls._prefill_begin_group(groups[0], cfg_k, cfg_v, **hk)
            for gi in range(len(groups)):
                cur = nxt
                nxt = (cls._prefill_begin_group(groups[gi + 1], cfg_k, cfg_v, **hk)
                       if gi + 1 < len(groups) else None)
                out.extend(cls._prefill_finish(c, False) for c in cur)
            if check:
                for st in out:
                    st.check()
            return out
        nxt = cls._prefill_begin(*items[0], cfg_k, cfg_v, **kw) if items else None
        for i in range(len(items)):
            cur = nxt
            nxt = (cls._prefill_begin(*items[i + 1], cfg_k, cfg_v, **kw)
                   if i + 1 < len(items) else None)
            out.append(cls._prefill_finish(cur, False))
        if check:  # one synchronisation for the whole batch, after every launch
            for st in out:
                st.check()
        return out

    @staticmethod
    def _prefill_group_ok(items, cfg_k, cfg_v, kw) -> bool:
        """The grouped prefill covers the common serving case: device fp16/f32
        tensors of one shape, K_BLOCK, codebooks from the data, the fused
        hot-path Store with per-block histograms, default arena placement."""
        if len(items) < 2 or any(kw.get(k) is not None for k in (
                "codebooks", "k_channel_ranges", "process_group", "capacity", "page_pool",
                "device")):
            return False
        if set(kw) - {"head_base", "head_total", "codebooks", "k_channel_ranges",
                      "process_group", "capacity", "page_pool", "device"}:
            return False
        if cfg_k.mode is not QuantMode.K_BLOCK:
            return False
        k0 = items[0][0]
        if not (isinstance(k0, torch.Tensor) and k0.is_cuda and k0.dim() == 3
                and k0.dtype in (torch.float16, torch.float32)):
            return False
        for k, v in items:
            if not (isinstance(k, torch.Tensor) and isinstance(v, torch.Tensor)
                    and k.shape == k0.shape and v.shape == k0.shape and k.dtype == k0.dtype
                    and v.dtype == k0.dtype and k.device == k0.device and v.device == k0.device
                    and k.is_contiguous() and v.is_contiguous()):
                return False
        ctx, H, D = k0.shape
        bs = cfg_k.block_size
        return (ctx >= bs and cfg_k.block_size == cfg_v.block_size
                and cfg_k.buffer_size == cfg_v.buffer_size
                and _store_supported(bs, D, 32)
                and _prefill_supported(bs, D, cfg_k.rel_quant_scale, cfg_v.rel_quant_scale))

    @classmethod
    def _prefill_begin_group(cls, items, cfg_k, cfg_v, head_base: int = 0,
                             head_total: Optional[int] = None) -> list:
        """_prefill_begin for a group of equal slices (see _prefill_group_ok):
        one zeroed slab-pool block [histograms | per state: counters, K and V
        token buffers] shared by the group's states, one scratch allocation,
        pass A per item and ONE histogram readback for the group."""
        k0 = items[0][0]
        dev = k0.device
        ctx, H, D = k0.shape
        bs = cfg_k.block_size
        n_chunks = ctx // bs
        n_full = n_chunks * bs
        G = len(items)
        cap = cfg_k.buffer_size + 1
        nbuf = cap * H * D * 4
        per = 128 + 2 * nbuf
        blk, ext = pooled_zeros((G * 4096 + G * per,), torch.uint8, dev)
        shared = _SharedRelease(ext, G)
        hists = blk[:G * 4096].view(torch.int64).view(G, 512)
        hb, cb_, wb = _prefill_scratch_bytes(n_chunks, H, D, bs)
        one = hb + cb_ + wb
        scratch = torch.empty(G * one, dtype=torch.uint8, device=dev)
        lib = _lib.lib()
        stream = torch.cuda.current_stream(dev).cuda_stream
        src_dtype = np.dtype(np.float16) if k0.dtype == torch.float16 else np.dtype(np.float32)
        code = dtype_code(k0)
        out = []
        for g, (k, v) in enumerate(items):
            b0 = G * 4096 + g * per
            pre = {"small": blk[b0:b0 + 128],
                   "k_buffer": blk[b0 + 128:b0 + 128 + nbuf].view(torch.float32).view(cap, H, D),
                   "v_buffer": blk[b0 + 128 + nbuf:b0 + per].view(torch.float32).view(cap, H, D),
                   "extents": (shared,)}
            s0 = g * one
            blk_hist = scratch[s0:s0 + hb].view(torch.int16)
            blk_codes = scratch[s0 + hb:s0 + hb + cb_] if cb_ else None
            _lib.check(lib.kvc_store_hist_blocks(
                k.data_ptr(), v.data_ptr(), code, H * D, n_chunks, H, D, bs, cfg_k.mode.abi,
                cfg_k.rel_quant_scale, cfg_v.rel_quant_scale, None, hists[g].data_ptr(),
                blk_hist.data_ptr(), blk_codes.data_ptr() if blk_codes is not None else None,
                stream), "kvc_store_hist_blocks")
            out.append(dict(cls=cls, kt=k, vt=v, cfg_k=cfg_k, cfg_v=cfg_v, codebooks=None,
                            page_pool=None, k_channel_ranges=None, head_base=head_base,
                            head_total=head_total, capacity=None, src_dtype=src_dtype, ctx=ctx,
                            H=H, D=D, bs=bs, n_chunks=n_chunks, n_full=n_full, fused=True,
                            hist=hists[g], hist_host=None, ev=None, blk_hist=blk_hist,
                            blk_codes=blk_codes, kcodes=None, kmetas=None, vcodes=None,
                            vmetas=None, pre=pre, pre_ws=scratch[s0 + hb + cb_:s0 + one]))
        ring = _GROUP_RINGS.get(dev)
        if ring is None:
            with torch.cuda.device(dev):
                ring = _GROUP_RINGS[dev] = _GroupRing(PREFILL_GROUP)
        i = ring.i
        ring.i = (i + 1) % len(ring.bufs)
        ev = ring.events[i]
        if ring.used[i]:
            ev.synchronize()
        host = ring.bufs[i]
        host[:G].copy_(hists, non_blocking=True)
        ev.record(torch.cuda.current_stream(dev))
        ring.used[i] = True
        for g, c in enumerate(out):
            c["hist_host"], c["ev"] = host[g], ev
        return out

    @classmethod
    def _prefill_begin(cls, k, v, cfg_k, cfg_v, codebooks=None, k_channel_ranges=None,
                       device=None, process_group=None, head_base: int = 0,
                       head_total: Optional[int] = None, capacity: Optional[int] = None,
                       page_pool=None, _defer_hist: bool = False):
        """Pass A and every allocation that does not depend on the histogram;
        the histogram is copied to pinned host memory behind an event."""
        kv = k.values if isinstance(k, CacheTensor) else k
        vv = v.values if isinstance(v, CacheTensor) else v
        if tuple(kv.shape) != tuple(vv.shape):
            raise ConfigError("K and V tensors must share dimensions")
        if kv.shape[0] < 1:
            raise ConfigError("prefill requires at least one token")
        kt = as_device_tensor(kv, device)
        # state dtype (its itemsize is the "original bytes" of collect_stats,
        # bench.py:77-95): fp16 stays fp16; bf16 (no numpy dtype) is reported
        # as a 2-byte original, everything else as f32 like the reference
        if isinstance(kv, torch.Tensor):
            src_dtype = np.dtype(np.float16) if kv.dtype in (torch.float16, torch.bfloat16) \
                else np.dtype(np.float32)
        else:
            src_dtype = np.dtype(kv.dtype)
        vt = as_device_tensor(vv, kt.device)
        ctx, H, D = kt.shape
        bs = cfg_k.block_size
        n_chunks = ctx // bs
        n_full = n_chunks * bs
        k_is_ch = cfg_k.mode is QuantMode.K_CHANNEL
        if k_is_ch and k_channel_ranges is None:
            kf = kt.to(torch.float32)
            k_channel_ranges = (kf.amin(dim=0), kf.amax(dim=0))
        ranges_dev = None
        if k_is_ch:
            ranges_dev = torch.stack([torch.as_tensor(r, dtype=torch.float32).to(kt.device)
                                      for r in k_channel_ranges]).contiguous()
        if kt.dtype != vt.dtype:
            kt, vt = kt.to(torch.float32), vt.to(torch.float32)
        lib = _lib.lib()
        stream = torch.cuda.current_stream(kt.device).cuda_stream
        fused = _store_supported(bs, D, 32 if codebooks is None else max(
            codebooks[0].max_code_length, codebooks[1].max_code_length))
        # one zeroed slab-pool block per state: [hist 4 KB | counters+live 128 B |
        # K buffer | V buffer] (one allocation and one fill instead of four)
        cap = cfg_k.buffer_size + 1
        pre = None
        if kt.device.type == "cuda":
            nbuf = cap * H * D * 4
            blk, blk_ext = pooled_zeros((4096 + 128 + 2 * nbuf,), torch.uint8, kt.device)
            hist = blk[:4096].view(torch.int64)
            pre = {"small": blk[4096:4224],
                   "k_buffer": blk[4224:4224 + nbuf].view(torch.float32).view(cap, H, D),
                   "v_buffer": blk[4224 + nbuf:].view(torch.float32).view(cap, H, D),
                   "extents": (blk_ext,)}
        else:
            hist = torch.zeros(512, dtype=torch.int64, device=kt.device)
        kcodes = kmetas = vcodes = vmetas = None
        # small alphabets: pass A also records per-block histograms, so pass B takes
        # its arena offsets from one scan instead of the look-back (store_fused.cu)
        blk_hist = blk_codes = pre_ws = None
        if (n_full and codebooks is None and fused
                and _prefill_supported(bs, D, cfg_k.rel_quant_scale, cfg_v.rel_quant_scale)):
            # one scratch allocation: per-block histograms | pass A's codes (hot
            # shape: pass B encodes them, no re-quantisation) | pass B workspace
            hb, cb_, wb = _prefill_scratch_bytes(n_chunks, H, D, bs)
            scratch = torch.empty(hb + cb_ + wb, dtype=torch.uint8, device=kt.device)
            blk_hist = scratch[:hb].view(torch.int16)
            blk_codes = scratch[hb:hb + cb_] if cb_ else None
            pre_ws = scratch[hb + cb_:]
            _lib.check(lib.kvc_store_hist_blocks(kt.data_ptr(), vt.data_ptr(), dtype_code(kt),
                                                 H * D, n_chunks, H, D, bs, cfg_k.mode.abi,
                                                 cfg_k.rel_quant_scale, cfg_v.rel_quant_scale,
                                                 ranges_dev.data_ptr() if ranges_dev is not None
                                                 else None, hist.data_ptr(), blk_hist.data_ptr(),
                                                 blk_codes.data_ptr() if blk_codes is not None
                                                 else None, stream), "kvc_store_hist_blocks")
        elif n_full and codebooks is None and fused:
            # pass A: quantise + histogram only (store_fused.cu)
            _lib.check(lib.kvc_store_hist(kt.data_ptr(), vt.data_ptr(), dtype_code(kt), H * D,
                                          n_chunks, H, D, bs, cfg_k.mode.abi,
                                          cfg_k.rel_quant_scale, cfg_v.rel_quant_scale,
                                          ranges_dev.data_ptr() if ranges_dev is not None
                                          else None, hist.data_ptr(), stream),
                       "kvc_store_hist")
        elif n_full and not fused:
            kcodes, kmetas = quantize_tokens(kt, n_chunks, H, D, bs, cfg_k.mode,
                                             cfg_k.rel_quant_scale,
                                             hist[:256] if codebooks is None else None,
                                             k_ranges=ranges_dev)
            vcodes, vmetas = quantize_tokens(vt, n_chunks, H, D, bs, QuantMode.V_TOKEN,
                                             cfg_v.rel_quant_scale,
                                             hist[256:] if codebooks is None else None)
        # everything that does not depend on the histogram is allocated while
        # pass A runs, so the host work between its completion and pass B is
        # only the codebook build, the table upload and the arena carve-out
        if pre is None:
            pre = {"k_buffer": torch.zeros((cap, H, D), dtype=torch.float32, device=kt.device)}
            pre["v_buffer"] = torch.zeros_like(pre["k_buffer"])
        if pre_ws is None and n_full and fused:
            pre_ws = torch.empty(_store_ws_bytes(n_chunks, H, D, bs), dtype=torch.uint8,
                                 device=kt.device)
        hist_host = ev = None
        if codebooks is None and not _defer_hist:
            if process_group is not None:
                torch.distributed.all_reduce(hist, group=process_group)
            hist_host, ev = _hist_readback(hist)
        return dict(cls=cls, kt=kt, vt=vt, cfg_k=cfg_k, cfg_v=cfg_v, codebooks=codebooks,
                    page_pool=page_pool,
                    k_channel_ranges=k_channel_ranges, head_base=head_base,
                    head_total=head_total, capacity=capacity, src_dtype=src_dtype, ctx=ctx,
                    H=H, D=D, bs=bs, n_chunks=n_chunks, n_full=n_full, fused=fused,
                    hist=hist, hist_host=hist_host, ev=ev, blk_hist=blk_hist, blk_codes=blk_codes,
                    kcodes=kcodes, kmetas=kmetas, vcodes=vcodes, vmetas=vmetas, pre=pre,
                    pre_ws=pre_ws)

    @staticmethod
    def _prefill_finish(c: dict, check: bool) -> "LayerCacheState":
        """Codebooks from the histogram, the state, pass B (prefill's second half)."""
        cls, kt, vt, cfg_k, cfg_v = c["cls"], c["kt"], c["vt"], c["cfg_k"], c["cfg_v"]
        codebooks, k_channel_ranges = c["codebooks"], c["k_channel_ranges"]
        head_base, head_total, capacity = c["head_base"], c["head_total"], c["capacity"]
        src_dtype, ctx, H, D, bs = c["src_dtype"], c["ctx"], c["H"], c["D"], c["bs"]
        n_chunks, n_full = c["n_chunks"], c["n_full"]
        blk_hist, blk_codes, pre, pre_ws = c["blk_hist"], c["blk_codes"], c["pre"], c["pre_ws"]
        kcodes, kmetas, vcodes, vmetas = c["kcodes"], c["kmetas"], c["vcodes"], c["vmetas"]
        if codebooks is None:
            c["ev"].synchronize()  # this item's pass A only, not later launches
            h = c["hist_host"].numpy().astype(np.uint64)  # a copy: the slot may be reused
            k_cb = build_smoothed_codebook(h[:256], cfg_k.max_code)
            v_cb = build_smoothed_codebook(h[256:], cfg_v.max_code)
        else:
            k_cb, v_cb = codebooks
        # Arena sizes: the histogram gives every prefill block's code bits, so
        # sum(count * length) / 8 + (header + 4 B of byte/word padding) per block
        # bounds each arena (codec.py:229-244) far tighter than the max-length
        # worst case; a little headroom covers the first growing-cache appends.
        nb = n_chunks * H
        bounds = None
        if codebooks is None and n_full:
            bounds = []
            for cb, hh, n_units in ((k_cb, h[:256], D), (v_cb, h[256:], bs)):
                bits = int((hh.astype(np.uint64) * cb.code_lengths.astype(np.uint64)).sum())
                tight = nb * (6 + 2 * bs + 8 * n_units + 4) + (bits + 7) // 8
                worst = nb * worst_block_bytes(bs, n_units, D, cb.max_code_length)
                bounds.append(min(tight, worst))
        head = 2 * H * max(worst_block_bytes(bs, D, D, k_cb.max_code_length),
                           worst_block_bytes(bs, bs, D, v_cb.max_code_length))
        arena_bytes = None
        if capacity is None and n_full:
            arena_bytes = ((bounds[0] if bounds else nb * worst_block_bytes(
                bs, D, D, k_cb.max_code_length)) + head,
                (bounds[1] if bounds else nb * worst_block_bytes(
                    bs, bs, D, v_cb.max_code_length)) + head)
        st = cls(H, D, cfg_k, cfg_v, k_cb, v_cb, dtype=src_dtype, device=kt.device,
                 head_base=head_base, head_total=head_total, capacity=capacity,
                 k_channel_ranges=k_channel_ranges, arena_bytes=arena_bytes,
                 arena_blocks=max(nb + 4 * H, 256), page_pool=c.get("page_pool"), _pre=pre)
        if pre_ws is not None:
            st._ws = pre_ws
        if n_full:
            if blk_hist is not None and st._fused_store:
                st._store(kt, vt, n_chunks, blk_hist=blk_hist, blk_codes=blk_codes, bounds=bounds)
            elif st._fused_store:
                st._store(kt, vt, n_chunks, bounds=bounds)
            else:
                if kcodes is None:
                    kcodes, kmetas = quantize_tokens(kt, n_chunks, H, D, bs, cfg_k.mode,
                                                     cfg_k.rel_quant_scale, k_ranges=st._k_ranges)
                    vcodes, vmetas = quantize_tokens(vt, n_chunks, H, D, bs, QuantMode.V_TOKEN,
                                                     cfg_v.rel_quant_scale)
                st._encode(kcodes, kmetas, vcodes, vmetas, n_chunks)
        # the prefill workspace goes back to the allocator's cache for the next
        # prefill; appends size their own
        st._ws = _empty_ws(st.device)
        r = ctx - n_full
        if r:
            st._k_buffer[:r] = kt[n_full:].to(torch.float32)
            st._v_buffer[:r] = vt[n_full:].to(torch.float32)
        st.buffered = r
        st.context_len = ctx
        st._publish_live()
        if check:
            st.check()
        return st

    # ------------------------------------------------------------------
    def _workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 2 * self._ws.numel()), dtype=torch.uint8,
                                   device=self.device)
        return self._ws

    def _encode(self, kcodes, kmetas, vcodes, vmetas, n_chunks: int) -> None:
        bs, H, D = self.cfg_k.block_size, self.head_num, self.head_dim
        lib = _lib.lib()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        nb = n_chunks * H
        ws = self._workspace(lib.kvc_encode_workspace_bytes(nb, bs))
        chunk_base = self.compressed_tokens // bs
        for arena, codes, metas, cb, tab, n_units in (
                (self.k_arena, kcodes, kmetas, self.k_codebook, self._k_tab, D),
                (self.v_arena, vcodes, vmetas, self.v_codebook, self._v_tab, bs)):
            worst = nb * worst_block_bytes(bs, n_units, D, cb.max_code_length)
            arena.reserve(nb, worst)
            st = lib.kvc_encode_append(
                codes.data_ptr(), metas.data_ptr(), n_chunks, H, self.head_total, self.head_base,
                chunk_base, bs, D, n_units, cb.max_code_length, tab.data_ptr(), arena.buf_ptr,
                arena.alloc_capacity, arena.offsets_ptr, arena.counters_ptr, ws.data_ptr(), stream)
            _lib.check(st, "kvc_encode_append")
            if arena.capacity is not None:  # codec.py:313-318: a full arena raises here
                arena.check("arena")
            arena.note_append(nb, worst, worst_block_bytes(bs, n_units, D, cb.max_code_length))
        self.compressed_tokens += n_chunks * bs

    def _store(self, k_src: torch.Tensor, v_src: torch.Tensor, n_chunks: int,
               blk_hist: Optional[torch.Tensor] = None,
               blk_codes: Optional[torch.Tensor] = None,
               bounds: Optional[Tuple[int, int]] = None) -> None:
        """Quantise + encode + append of n_chunks*H blocks per tensor from
        k_src/v_src rows [0, n_chunks*bs) (store_fused.cu): one look-back launch
        (kvc_store_append), or, with the prefill's per-block histograms, the
        offsets scan + encode (kvc_store_prefill)."""
        bs, H, D = self.cfg_k.block_size, self.head_num, self.head_dim
        lib = _lib.lib()
        nb = n_chunks * H
        kw = nb * worst_block_bytes(bs, D, D, self.k_codebook.max_code_length)
        vw = nb * worst_block_bytes(bs, bs, D, self.v_codebook.max_code_length)
        if bounds is not None:  # exact-histogram bounds from the prefill
            kw, vw = min(kw, bounds[0]), min(vw, bounds[1])
        self.k_arena.reserve(nb, kw)
        self.v_arena.reserve(nb, vw)
        ws = self._workspace(lib.kvc_store_workspace_bytes(n_chunks, H, D, bs))
        fn = lib.kvc_store_append if blk_hist is None else functools.partial(
            _prefill_call, lib.kvc_store_prefill, blk_hist.data_ptr(),
            blk_codes.data_ptr() if blk_codes is not None else None)
        st = fn(
            k_src.data_ptr(), v_src.data_ptr(), dtype_code(k_src), H * D, n_chunks, H,
            self.head_total, self.head_base, D, bs, self.cfg_k.mode.abi,
            self.cfg_k.rel_quant_scale, self.cfg_v.rel_quant_scale,
            self._k_ranges.data_ptr() if self._k_ranges is not None else None,
            self.compressed_tokens // bs, self._k_tab.data_ptr(),
            self.k_codebook.max_code_length, self._v_tab.data_ptr(),
            self.v_codebook.max_code_length, self.k_arena.buf_ptr, self.k_arena.alloc_capacity,
            self.k_arena.offsets_ptr, self.k_arena.counters_ptr, self.v_arena.buf_ptr,
            self.v_arena.alloc_capacity, self.v_arena.offsets_ptr, self.v_arena.counters_ptr,
            ws.data_ptr(), ws.numel(), torch.cuda.current_stream(self.device).cuda_stream)
        _lib.check(st, "kvc_store_append" if blk_hist is None else "kvc_store_prefill")
        if self.k_arena.capacity is not None or self.v_arena.capacity is not None:
            # fixed capacity: the device refuses blocks past it (sticky error);
            # raise ArenaFullError now, as CompressedArena.append does
            # (codec.py:313-318), before the host mirrors advance
            self.k_arena.check("K arena")
            self.v_arena.check("V arena")
        self.k_arena.note_append(nb, kw, worst_block_bytes(bs, D, D, self.k_codebook.max_code_length))
        self.v_arena.note_append(nb, vw, worst_block_bytes(bs, bs, D, self.v_codebook.max_code_length))
        self.compressed_tokens += n_chunks * bs

    def _compress_buffer(self, n: int) -> None:
        """Compress buffer rows [0, n) (n a multiple of block_size)."""
        bs = self.cfg_k.block_size
        n_chunks = n // bs
        if self._fused_store:
            self._store(self._k_buffer, self._v_buffer, n_chunks)
            return
        kcodes, kmetas = quantize_tokens(self._k_buffer, n_chunks, self.head_num, self.head_dim,
                                         bs, self.cfg_k.mode, self.cfg_k.rel_quant_scale,
                                         k_ranges=self._k_ranges)
        vcodes, vmetas = quantize_tokens(self._v_buffer, n_chunks, self.head_num, self.head_dim,
                                         bs, QuantMode.V_TOKEN, self.cfg_v.rel_quant_scale)
        self._encode(kcodes, kmetas, vcodes, vmetas, n_chunks)

    def _publish_live(self) -> None:
        """Device live pair <- host mirrors (after prefill / restore)."""
        if self.device.type != "cuda":
            self._live.copy_(torch.tensor([self.n_chunks, self.buffered], dtype=torch.int32))
            return
        _lib.check(_lib.lib().kvc_set_live(self._live.data_ptr(), self.n_chunks, self.buffered,
                                           torch.cuda.current_stream(self.device).cuda_stream),
                   "kvc_set_live")

    def _after_append(self) -> Optional[int]:
        """Host mirrors after one appended token; returns the rows to compress
        when the buffer overflows (kvcache.py:168-177), else None."""
        self.buffered += 1
        self.context_len += 1
        if self.buffered > self.cfg_k.buffer_size:
            bs = self.cfg_k.block_size
            return (self.buffered // bs) * bs
        return None

    def _overflow(self, n: int, desc_dev: Optional[torch.Tensor] = None) -> None:
        """Overflow event: compress buffer rows [0, n), move the remainder to
        the front and publish the new live pair, all on the device."""
        self._compress_buffer(n)
        rem = self.buffered - n
        if desc_dev is None:
            desc_dev = self.desc_device()
        _lib.check(_lib.lib().kvc_buffer_shift(desc_dev.data_ptr(), 1, self.head_num,
                                               self.head_dim, n, rem, self.n_chunks,
                                               torch.cuda.current_stream(self.device).cuda_stream),
                   "kvc_buffer_shift")
        self.buffered = rem

    def append_token(self, k_vec, v_vec, validate: bool = True) -> None:
        """kvcache.py:150-177.  Host arrays are validated on the host; device
        tensors with one device reduction when validate=True (validate=False:
        non-finite values set the state's sticky error, raised by check()).
        The buffer write and the live counts are device work (kvc_buffer_append):
        no synchronisation on the decode path."""
        expected = (self.head_num, self.head_dim)
        if isinstance(k_vec, torch.Tensor) and isinstance(v_vec, torch.Tensor):
            if tuple(k_vec.shape) != expected or tuple(v_vec.shape) != expected:
                raise CodecError(f"token vectors must have shape {expected}")
            kd, vd = k_vec, v_vec
            if kd.dtype not in (torch.float16, torch.float32) or kd.dtype != vd.dtype:
                kd, vd = kd.to(torch.float32), vd.to(torch.float32)
            kd = kd.to(self.device).contiguous()
            vd = vd.to(self.device).contiguous()
            if validate and not bool(torch.isfinite(kd).all() & torch.isfinite(vd).all()):
                raise CodecError("non-finite token vectors rejected")
        else:
            kn = np.asarray(k_vec, dtype=np.float32)
            vn = np.asarray(v_vec, dtype=np.float32)
            if kn.shape != expected or vn.shape != expected:
                raise CodecError(f"token vectors must have shape {expected}")
            if not (np.all(np.isfinite(kn)) and np.all(np.isfinite(vn))):
                raise CodecError("non-finite token vectors rejected")
            kd = torch.from_numpy(kn).to(self.device, non_blocking=False)
            vd = torch.from_numpy(vn).to(self.device, non_blocking=False)
        if self.device.type != "cuda":
            self._k_buffer[self.buffered] = kd
            self._v_buffer[self.buffered] = vd
            n = self._after_append()
            if n is not None:
                self._compress_buffer(n)
                rem = self.buffered - n
                if rem:
                    self._k_buffer[:rem] = self._k_buffer[n: self.buffered].clone()
                    self._v_buffer[:rem] = self._v_buffer[n: self.buffered].clone()
                self.buffered = rem
            self._live.copy_(torch.tensor([self.n_chunks, self.buffered], dtype=torch.int32))
            return
        dd = self.desc_device()
        _lib.check(_lib.lib().kvc_buffer_append(
            dd.data_ptr(), 1, self.head_num, self.head_dim, self.cfg_k.buffer_size + 1,
            kd.data_ptr(), vd.data_ptr(), dtype_code(kd), 0, None,
            torch.cuda.current_stream(self.device).cuda_stream), "kvc_buffer_append")
        n = self._after_append()
        if n is not None:
            self._overflow(n, dd)

    def append_tokens(self, k_tokens: torch.Tensor, v_tokens: torch.Tensor) -> None:
        """Append many tokens (device tensors [n, H, D]); identical arenas to
        n append_token calls (overflow events fire at the same points)."""
        for t in range(k_tokens.shape[0]):
            self.append_token(k_tokens[t], v_tokens[t], validate=False)

    # ------------------------------------------------------------------
    def check(self) -> None:
        """Synchronise and raise any sticky device error (CodecError /
        ArenaFullError) recorded by the Store kernels."""
        self.k_arena.check("K arena")
        self.v_arena.check("V arena")

    def extents_ready(self) -> bool:
        """True when no max-extent readback is pending or in flight
        (non-blocking; starts the readback of stale arenas)."""
        for a in (self.k_arena, self.v_arena):
            a.max_extent_bound()
            if a._ext_pending is not None:
                return False
        return True

    def settle(self) -> None:
        """Wait for the arenas' in-flight max-extent readbacks (after appends)
        so stage_bytes() is exact again; waits on those copies only."""
        for a in (self.k_arena, self.v_arena):
            a.max_extent_bound()
            if a._ext_pending is not None:
                a._ext_pending[1].synchronize()
                a.max_extent_bound()

    def compact(self, headroom: int = 0) -> None:
        """Trim arena allocations to their contents (pointers change)."""
        self.k_arena.compact(headroom)
        self.v_arena.compact(headroom)
        self._desc_key = None

    @property
    def n_chunks(self) -> int:
        return self.compressed_tokens // self.cfg_k.block_size

    def stage_bytes(self) -> Tuple[int, int]:
        """Shared-memory staging size per K / V extent for the fused fetch,
        from the arenas' host max-extent bounds (no synchronisation)."""
        # a block's TMA copy is its 16-B aligned superset: offsets and extents
        # are 4-B aligned, so at most 12 bytes before and 12 after the block.
        # (Tight on purpose: two fetch CTAs per SM need K + V stages <= ~9.8 KB,
        # and config-2 data sits within ~100 B of that.)
        out = []
        for arena in (self.k_arena, self.v_arena):
            ext = arena.max_extent_bound() if arena.n_blocks else 16
            out.append(((ext + 24 + 15) // 16) * 16)
        return out[0], out[1]

    def desc(self) -> _lib.SeqDesc:
        """The kernels' view of this state.  Stable across decode steps: the
        token counts travel through the device live pair, so only an arena
        reallocation or a new stage size makes a new descriptor; the host
        copy's n_chunks / buffered are refreshed on every call."""
        sk, sv = self.stage_bytes()
        key = (self.k_arena.buf_ptr, self.v_arena.buf_ptr, self.k_arena.offsets_ptr,
               self.v_arena.offsets_ptr, self.k_arena.counters_ptr, self.v_arena.counters_ptr,
               sk, sv)
        d = getattr(self, "_desc_host", None)
        if self._desc_key != key or d is None:
            d = _lib.SeqDesc(
                k_arena=self.k_arena.buf_ptr, k_offsets=self.k_arena.offsets_ptr,
                k_counters=self.k_arena.counters_ptr, k_cb=self._k_tab.data_ptr(),
                v_arena=self.v_arena.buf_ptr, v_offsets=self.v_arena.offsets_ptr,
                v_counters=self.v_arena.counters_ptr, v_cb=self._v_tab.data_ptr(),
                k_buffer=self._k_buffer.data_ptr(), v_buffer=self._v_buffer.data_ptr(),
                n_chunks=self.n_chunks, buffered=self.buffered, stage_bytes_k=sk,
                stage_bytes_v=sv, k_max_len=self.k_codebook.max_code_length,
                v_max_len=self.v_codebook.max_code_length, live=self._live.data_ptr())
            self._desc_host = d
            self._desc_key = key
            self._desc_dev = None
        else:
            d.n_chunks = self.n_chunks
            d.buffered = self.buffered
        return d

    def desc_device(self) -> torch.Tensor:
        d = self.desc()
        if self._desc_dev is None:
            self._desc_dev = upload_bytes(bytes(d), self.device)
        return self._desc_dev

    # ------------------------------------------------------------------
    def fetch_dequantized(self) -> Tuple[CacheTensor, CacheTensor]:
        """kvcache.py:182-212: decode + f64 dequantise on the device."""
        outs = []
        err = torch.zeros(1, dtype=torch.int32, device=self.device)
        desc = self.desc_device()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        for which, buf in ((0, self._k_buffer), (1, self._v_buffer)):
            out = torch.empty((self.context_len, self.head_num, self.head_dim),
                              dtype=torch.float32, device=self.device)
            st = _lib.lib().kvc_dequantize(desc.data_ptr(), self.head_num, self.head_dim,
                                           self.cfg_k.block_size, which, self.n_chunks,
                                           out.data_ptr(), err.data_ptr(), stream)
            _lib.check(st, "kvc_dequantize")
            if self.buffered:
                out[self.compressed_tokens:] = buf[: self.buffered]
            outs.append(out)
        _lib.raise_device_error(int(err.item()), "fetch_dequantized")
        return CacheTensor(outs[0]), CacheTensor(outs[1])


def _prefill_call(fn, blk_hist_ptr, codes_ptr, *args):
    """kvc_store_prefill takes kvc_store_append's arguments plus the per-block
    histograms and pass A's codes before the workspace."""
    return fn(*args[:-3], blk_hist_ptr, codes_ptr, *args[-3:])


class _PinnedUpload:
    """Pinned staging ring for small asynchronous H2D uploads (descriptor
    arrays): a pageable .to(device) would synchronise the stream.  A slot is
    rewritten only after the event of its previous copy has completed."""

    def __init__(self, slot_bytes: int = 1 << 16, slots: int = 64):
        self.slot_bytes = slot_bytes
        self.buf = torch.empty((slots, slot_bytes), dtype=torch.uint8, pin_memory=True)
        self.events = [None] * slots
        self.i = 0


_UPLOAD = None


def upload_bytes(raw: bytes, device) -> torch.Tensor:
    """bytes -> a new device uint8 tensor, stream-ordered, without a sync."""
    global _UPLOAD
    dev = torch.device(device)
    n = len(raw)
    if dev.type != "cuda":
        return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
    if _UPLOAD is None:
        _UPLOAD = _PinnedUpload()
    r = _UPLOAD
    if n > r.slot_bytes:
        return torch.from_numpy(np.frombuffer(raw, np.uint8).copy()).pin_memory().to(
            dev, non_blocking=True)
    i = r.i
    r.i = (i + 1) % len(r.events)
    if r.events[i] is not None:
        r.events[i].synchronize()
    slot = r.buf[i, :n]
    slot.numpy()[:] = np.frombuffer(raw, np.uint8)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    out.copy_(slot, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(dev))
    r.events[i] = ev
    return out


class _BatchDesc:
    """Device array of kvc_seq_desc for a fixed list of states, re-uploaded
    only when a state's descriptor changes (arena reallocation, stage size);
    the token counts travel through each state's live pair.  The host copy
    (kvc_attention plans its splits from it) gets the current counts on
    every call."""

    def __init__(self):
        self.key = None
        self.dev = None
        self.host = None
        self.ids = None

    def get(self, states):
        descs = [s.desc() for s in states]
        # desc() returns the same object while a state's descriptor is
        # unchanged: an identity check skips the byte comparison
        ids = tuple(map(id, descs))
        if ids != self.ids or self.dev is None:
            raw = b"".join(bytes(d) for d in descs)
            self.ids = ids
            self.descs = descs  # keep them alive so the ids stay unique
            self.host = (_lib.SeqDesc * len(descs))(*descs)
            if raw != self.key:
                self.dev = upload_bytes(raw, states[0].device)
                self.key = raw
        else:
            h = self.host
            for i, s in enumerate(states):
                h[i].n_chunks = s.n_chunks
                h[i].buffered = s.buffered
        return self.dev, self.host


def append_batched(states, k_rows: torch.Tensor, v_rows: torch.Tensor,
                   desc_cache: Optional[_BatchDesc] = None) -> None:
    """append_token for a batch of same-shape states in one launch
    (kvc_buffer_append): k_rows / v_rows [B, H, D] f16|f32 on the device.
    Overflow events (kvcache.py:168-177) then run per state.  No host sync;
    non-finite values set the states' sticky error (raised by check())."""
    s0 = states[0]
    B, H, D = len(states), s0.head_num, s0.head_dim
    if tuple(k_rows.shape) != (B, H, D) or tuple(v_rows.shape) != (B, H, D):
        raise CodecError(f"token rows must have shape {(B, H, D)}")
    for s in states[1:]:
        if (s.head_num, s.head_dim, s.cfg_k.buffer_size, s.device) != (
                H, D, s0.cfg_k.buffer_size, s0.device):
            raise ConfigError("batched states must share head_num, head_dim, buffer and device")
    if len(set(map(id, states))) != B:  # one CTA per state advances its live count
        raise ConfigError("a state appears twice in the batch")
    kd, vd = k_rows, v_rows
    if kd.dtype not in (torch.float16, torch.float32) or kd.dtype != vd.dtype:
        kd, vd = kd.to(torch.float32), vd.to(torch.float32)
    kd = kd.to(s0.device).contiguous()
    vd = vd.to(s0.device).contiguous()
    cache = desc_cache if desc_cache is not None else _BatchDesc()
    ddev, _ = cache.get(states)
    _lib.check(_lib.lib().kvc_buffer_append(
        ddev.data_ptr(), B, H, D, s0.cfg_k.buffer_size + 1, kd.data_ptr(), vd.data_ptr(),
        dtype_code(kd), H * D, None, torch.cuda.current_stream(s0.device).cuda_stream),
        "kvc_buffer_append")
    over = []
    for s in states:
        n = s._after_append()
        if n is not None:
            over.append((s, n))
    if not over:
        return
    bs = s0.cfg_k.block_size
    if len(over) == B and len({(n, s.buffered - n, s.compressed_tokens + n) for s, n in over}) == 1:
        # the usual decode-loop event: every state overflows at the same
        # point, so one batched shift (through the batch descriptors: only
        # the buffers and live pairs are touched) replaces B per-state
        # descriptor uploads and shifts
        for s, n in over:
            s._compress_buffer(n)
        n = over[0][1]
        rem = s0.buffered - n
        _lib.check(_lib.lib().kvc_buffer_shift(ddev.data_ptr(), B, H, D, n, rem,
                                               s0.compressed_tokens // bs,
                                               torch.cuda.current_stream(s0.device).cuda_stream),
                   "kvc_buffer_shift")
        for s, _ in over:
            s.buffered = rem
    else:
        for s, n in over:
            s._overflow(n)
    readback_extents([a for s, _ in over for a in (s.k_arena, s.v_arena)])


# names the reference's kvcache module also carries (kvcache.py:14-27 imports)
from .codebook import build_codebook, build_histogram, smooth_histogram  # noqa: E402
from .quantizer import quantize_block  # noqa: E402
