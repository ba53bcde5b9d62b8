"""Host logic of the arena slab pool (codec._SlabPool) and of the arena size
bound prefill derives from the histogram.  CPU tensors only: the pool's
bookkeeping is device-independent."""
import numpy as np
import torch

from paper_2509_00579_b200 import codec
from paper_2509_00579_b200.codec import _SlabPool, worst_block_bytes


def pool(slab=1 << 20):
    p = _SlabPool(torch.device("cpu"))
    p.slab_bytes = slab
    return p


def free_bytes(p):
    return sum(sz for fl in p.free for _, sz in fl)


def test_alloc_release_coalesces_back_to_one_extent():
    p = pool()
    exts = [p.alloc(n)[1] for n in (1000, 5000, 300, 70000)]
    assert len(p.slabs) == 1
    used = sum(e.n for e in exts)
    cap = p.slabs[0].numel()
    assert free_bytes(p) == cap - used
    for e in (exts[1], exts[3], exts[0], exts[2]):  # out of order
        e.release()
    assert p.free == [[[0, cap]]]


def test_extents_are_aligned_disjoint_views():
    p = pool()
    views = [p.alloc(n)[0] for n in (1, 255, 256, 257, 4097)]
    spans = sorted((v.data_ptr(), v.data_ptr() + v.numel()) for v in views)
    for (a0, a1), (b0, _) in zip(spans, spans[1:]):
        assert a1 <= b0
    assert all((v.data_ptr() - p.slabs[0].data_ptr()) % _SlabPool.ALIGN == 0 for v in views)


def test_release_is_idempotent_and_reuses_the_hole():
    p = pool()
    a, ea = p.alloc(4096)
    _, eb = p.alloc(4096)
    ea.release()
    ea.release()
    before = free_bytes(p)
    # the slab's tail serves first (prefills carve slabs in order) ...
    p.alloc(free_bytes(p) - 4096)
    # ... then first fit finds the released hole at offset 0
    c, _ = p.alloc(2048)
    assert c.data_ptr() == a.data_ptr()
    assert before == p.slabs[0].numel() - 4096
    eb.release()


def test_large_request_gets_a_dedicated_slab():
    p = pool(slab=1 << 16)
    v, e = p.alloc(3 << 16)
    assert v.numel() == 3 << 16 and len(p.slabs) == 1
    e.release()
    assert free_bytes(p) == p.slabs[0].numel()


def test_reserve_pregrows_the_pool():
    dev = torch.device("cpu")
    key = ("cpu", None)
    codec._POOLS.pop(key, None)
    try:
        pl = codec._pool(dev)
        pl.slab_bytes = 1 << 16
        got = codec.reserve_arena_pool(5 << 16, dev)
        assert got >= 5 << 16 and len(pl.slabs) == 5
        # an allocation after the reservation creates no new slab
        pl.alloc(1 << 15)
        assert len(pl.slabs) == 5
    finally:
        codec._POOLS.pop(key, None)


def test_arena_growth_and_compact_keep_bytes_and_return_extents():
    codec._POOLS.pop(("cpu", None), None)
    try:
        ar = codec.DeviceArena(torch.device("cpu"), initial_bytes=1024)
        pl = codec._pool(torch.device("cpu"))
        ar._buf[:1024] = torch.arange(1024, dtype=torch.int64).to(torch.uint8)
        before = ar._buf[:1024].clone()
        ar.reserve(4, 10000)  # grows: copy + release of the old extent
        assert torch.equal(ar._buf[:1024], before)
        n_ext = sum(len(fl) for fl in pl.free)
        del ar
        import gc
        gc.collect()
        # everything back: one free extent per slab
        assert sum(len(fl) for fl in pl.free) <= max(n_ext, len(pl.slabs))
        assert free_bytes(pl) == sum(s.numel() for s in pl.slabs)
    finally:
        codec._POOLS.pop(("cpu", None), None)


def test_histogram_bound_covers_every_block_layout():
    """prefill's arena bound: sum(count*len)/8 + (header + 4) per block is >= the
    serialised size sum over blocks of (header + ceil(bits_b/8) padded to 4)
    (codec.py:229-244), for random per-block bit counts."""
    rng = np.random.default_rng(0)
    bs, D = 64, 128
    for n_units in (D, bs):
        hdr = 6 + 2 * bs + 8 * n_units
        for _ in range(50):
            nb = int(rng.integers(1, 400))
            bits = rng.integers(0, bs * D * 6, size=nb)
            actual = int(sum((hdr + (int(b) + 7) // 8 + 3) & ~3 for b in bits))
            bound = nb * (hdr + 4) + (int(bits.sum()) + 7) // 8
            assert actual <= bound <= nb * worst_block_bytes(bs, n_units, D, 6) + 4 * nb


def test_release_inside_alloc_is_deferred_not_lost():
    """A release arriving while the pool lock is held (an arena finalizer run
    by a GC pass inside alloc, or another thread) is queued and applied by the
    next pool operation."""
    p = pool()
    _, e1 = p.alloc(4096)
    with p.lock:
        e1.release()  # cannot take the lock: queued
        assert p.pending
    _, e2 = p.alloc(1024)  # drains the queue first
    assert not p.pending
    e2.release()
    assert p.free == [[[0, p.slabs[0].numel()]]]


def test_shrink_returns_the_tail_in_place():
    p = pool()
    a, ea = p.alloc(100000)
    b, eb = p.alloc(5000)
    ea.shrink(30000)
    assert ea.n == 30208  # aligned up to 256
    # the returned tail is a hole between a and b: first fit reuses it
    p.alloc(free_bytes(p) - (100000 // 256 * 256 + 256 - 30208))  # drain the slab tail
    c, _ = p.alloc(60000)
    assert c.data_ptr() == a.data_ptr() + 30208
    ea.release()
    eb.release()


def test_arena_compact_shrinks_without_moving():
    codec._POOLS.pop(("cpu", None), None)
    try:
        ar = codec.DeviceArena(torch.device("cpu"), initial_bytes=1 << 16)
        ptr = ar.buf_ptr
        ar._counters.zero_()  # cursor 0: compact to the slack
        ar.compact(headroom=1000)
        assert ar.buf_ptr == ptr and ar._buf.numel() == 1000 + codec.TMA_SLACK
        assert ar._extent.n < (1 << 16)
    finally:
        codec._POOLS.pop(("cpu", None), None)
