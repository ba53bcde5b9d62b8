"""Paged arenas (paged.py; the paper's paged-cache integration, PAPER.md:276,
:490): states whose arenas map pages of a shared PagePool must store and fetch
exactly like slab-backed states (bit-exact arenas, identical attention),
grow without moving, and hand their pages back to the pool for reuse."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kv():
    import paper_2509_00579_b200 as kv
    return kv


def _data(ctx, H, seed):
    k = oracle.generate_synthetic(ctx, H, 128, seed=seed).astype(np.float16)
    v = oracle.generate_synthetic(ctx, H, 128, seed=seed + 1).astype(np.float16)
    return k, v


def test_paged_states_match_slab_states(kv):
    import torch
    pool = kv.PagePool(page_bytes=2 << 20)
    ck, cv = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    H, ctx, extra = 4, 64 * 40 + 9, 400
    datas = [_data(ctx + extra, H, 90 + 2 * b) for b in range(3)]
    items = [(torch.from_numpy(k[:ctx]).cuda(), torch.from_numpy(v[:ctx]).cuda())
             for k, v in datas]
    paged = kv.LayerCacheState.prefill_many(items, ck, cv, page_pool=pool)
    slab = kv.LayerCacheState.prefill_many(items, ck, cv)
    assert all(isinstance(s.k_arena, kv.PagedArena) for s in paged)
    ptrs = [(s.k_arena.buf_ptr, s.v_arena.buf_ptr) for s in paged]
    kd = torch.from_numpy(np.stack([k for k, _ in datas])).cuda()
    vd = torch.from_numpy(np.stack([v for _, v in datas])).cuda()
    cp, cs = kv.kvcache._BatchDesc(), kv.kvcache._BatchDesc()
    for t in range(ctx, ctx + extra):  # three overflow events: the arenas grow
        kv.append_batched(paged, kd[:, t], vd[:, t], desc_cache=cp)
        kv.append_batched(slab, kd[:, t], vd[:, t], desc_cache=cs)
    for p, s in zip(paged, slab):
        p.check()
        assert p.k_arena.snapshot() == s.k_arena.snapshot()
        assert p.v_arena.snapshot() == s.v_arena.snapshot()
        assert np.array_equal(p.k_arena.block_offsets, s.k_arena.block_offsets)
    # growth mapped pages in place: the arenas never moved
    assert [(s.k_arena.buf_ptr, s.v_arena.buf_ptr) for s in paged] == ptrs
    q = torch.randn((3, H, 128), device="cuda")
    op, _, ep = kv.attention_batched(paged, q)
    os_, _, es = kv.attention_batched(slab, q)
    assert int(ep.item()) == 0 and int(es.item()) == 0
    assert torch.equal(op, os_)
    # a single-state fetch and the dequantised view agree too
    assert torch.equal(kv.attention_step(paged[1], q[1]).out, kv.attention_step(slab[1], q[1]).out)


def test_paged_pages_return_to_the_pool(kv):
    import gc
    import torch
    pool = kv.PagePool(page_bytes=2 << 20)
    ck, cv = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    k, v = _data(64 * 200, 8, 7)
    st = kv.LayerCacheState.prefill(kv.CacheTensor(k), kv.CacheTensor(v), ck, cv, page_pool=pool)
    in_use = pool.pages_in_use
    assert in_use >= 2
    ref = kv.attention_step(st, np.ones((8, 128), np.float32)).out.clone()
    st.compact()                      # unused tail pages go back
    assert pool.pages_in_use <= in_use
    assert torch.equal(kv.attention_step(st, np.ones((8, 128), np.float32)).out, ref)
    del st
    gc.collect()
    assert pool.pages_in_use == 0 and len(pool.free) == pool.created
    created = pool.created
    st2 = kv.LayerCacheState.prefill(kv.CacheTensor(k), kv.CacheTensor(v), ck, cv, page_pool=pool)
    assert pool.created == created   # the freed pages were reused
    assert torch.equal(kv.attention_step(st2, np.ones((8, 128), np.float32)).out, ref)
    del st2
    gc.collect()
    assert pool.trim() == created


def test_paged_pool_limit_raises_arena_full(kv):
    pool = kv.PagePool(page_bytes=2 << 20, max_pages=1)
    ck, cv = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    k, v = _data(64 * 100, 8, 3)
    with pytest.raises(kv.ArenaFullError):
        kv.LayerCacheState.prefill(kv.CacheTensor(k), kv.CacheTensor(v), ck, cv, page_pool=pool)
