"""Streaming decode on the device (reference kvcache.py:150-177 growing cache,
bench.py:207-330 decode loop): the sync-free append path (kvc_buffer_append /
kvc_buffer_shift, live counts in kvc_seq_desc.live), the batched append and
the CUDA-graph DecodeLoop must give the same arenas and attention outputs as
the per-token reference-shaped path and the CPU oracle."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kv():
    import paper_2509_00579_b200 as kv
    return kv


def _data(ctx, extra, H, seed):
    k = oracle.generate_synthetic(ctx + extra, H, 128, seed=seed).astype(np.float16)
    v = oracle.generate_synthetic(ctx + extra, H, 128, seed=seed + 100).astype(np.float16)
    return k, v


def _prefill(kv, k, v, ctx, rels=(None, None)):
    return kv.LayerCacheState.prefill(kv.CacheTensor(k[:ctx]), kv.CacheTensor(v[:ctx]),
                                      kv.QuantConfig(kv.QuantMode.K_BLOCK, rel_quant_scale=rels[0]),
                                      kv.QuantConfig(kv.QuantMode.V_TOKEN, rel_quant_scale=rels[1]))


def test_append_batched_matches_append_token_and_oracle(kv):
    import torch
    H, ctx, extra, B = 4, 64 * 5 + 17, 300, 3   # crosses two overflow events
    data = [_data(ctx, extra, H, 10 + b) for b in range(B)]
    a = [_prefill(kv, k, v, ctx) for k, v in data]
    b_ = [_prefill(kv, k, v, ctx) for k, v in data]
    cache = kv.kvcache._BatchDesc()
    kd = torch.from_numpy(np.stack([k for k, _ in data])).cuda()
    vd = torch.from_numpy(np.stack([v for _, v in data])).cuda()
    for t in range(ctx, ctx + extra):
        kv.append_batched(a, kd[:, t], vd[:, t], desc_cache=cache)
        for i, st in enumerate(b_):
            st.append_token(data[i][0][t].astype(np.float32), data[i][1][t].astype(np.float32))
    for i in range(B):
        a[i].check()
        o = oracle.OracleState.prefill(data[i][0][:ctx], data[i][1][:ctx])
        for t in range(ctx, ctx + extra):
            o.append_token(data[i][0][t].astype(np.float32), data[i][1][t].astype(np.float32))
        for w in ("k", "v"):
            ar_a = a[i].k_arena if w == "k" else a[i].v_arena
            ar_b = b_[i].k_arena if w == "k" else b_[i].v_arena
            assert ar_a.snapshot() == ar_b.snapshot() == o.arena_bytes(w)
            assert np.array_equal(ar_a.block_offsets, o.block_offsets(w))
        assert (a[i].buffered, a[i].context_len, a[i].compressed_tokens) == (
            b_[i].buffered, b_[i].context_len, b_[i].compressed_tokens)
        assert torch.equal(a[i]._k_buffer[: a[i].buffered], b_[i]._k_buffer[: b_[i].buffered])
        assert a[i]._live.tolist() == [a[i].n_chunks, a[i].buffered]
    q = torch.randn((B, H, 128), device="cuda")
    out_a, _, err = kv.attention_batched(a, q, desc_cache=cache)
    assert int(err.item()) == 0
    for i in range(B):
        ref = kv.attention_step(b_[i], q[i]).out
        assert torch.equal(out_a[i], ref)


def test_attention_right_after_an_event_is_exact(kv):
    """The stage sizes after an overflow event come from the worst-case bound
    until the asynchronous max-extent readback lands; results must not
    depend on which one the launch used."""
    import torch
    H, ctx = 3, 64 * 6
    k, v = _data(ctx, 200, H, 33)
    st = _prefill(kv, k, v, ctx)
    st.check()
    cache = kv.kvcache._BatchDesc()
    q = torch.randn((1, H, 128), device="cuda")
    kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
    outs = []
    for t in range(ctx, ctx + 200):
        kv.append_batched([st], kd[t:t + 1], vd[t:t + 1], desc_cache=cache)
        o, _, _ = kv.attention_batched([st], q, desc_cache=cache, want_err=False)
        outs.append(o.clone())
    st.check()
    o = oracle.OracleState.prefill(k[:ctx], v[:ctx])
    for t in range(ctx, ctx + 200):
        o.append_token(k[t].astype(np.float32), v[t].astype(np.float32))
    ref, _ = o.attention_step(q[0].cpu().numpy())
    got = outs[-1][0].cpu().numpy()
    assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-5


@pytest.mark.parametrize("group,rels", [(1, (None, None)), (4, (None, None)), (1, (0.02, 0.05)),
                                        (1, (0.01, 0.02))])
def test_decode_loop_graph_matches_eager(kv, group, rels):
    """Default scales (pair decoders; G = 4 on the GQA kernel) and fine scales
    (lane-copied single-symbol decoders, 7-10-bit codes)."""
    import torch
    L, B, H, ctx, steps = 3, 2, 2, 64 * 4 + 60, 140   # one overflow event inside
    mk = lambda: [[_prefill(kv, *_data(ctx, 0, H, 50 + 7 * l + b), ctx, rels) for b in range(B)]
                  for l in range(L)]
    sa, sb = mk(), mk()
    ga = kv.DecodeLoop(sa, group=group, use_graph=True)
    gb = kv.DecodeLoop(sb, group=group, use_graph=False)
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.empty((L, B, H * group, 128), device="cuda")
    oa, ob = torch.empty_like(q), torch.empty_like(q)
    kn = torch.empty((L, B, H, 128), device="cuda", dtype=torch.float16)
    vn = torch.empty_like(kn)
    for i in range(steps):
        q.normal_(generator=g)
        kn.normal_(generator=g)
        vn.normal_(generator=g)
        ga.step(kn, vn, q, oa)
        gb.step(kn, vn, q, ob)
        assert torch.equal(oa, ob), f"step {i}"
    assert ga.events == gb.events == 1 and ga.captures >= 2
    if rels[0] is not None:
        assert all(max(x.k_codebook.max_code_length, x.v_codebook.max_code_length) >= 7
                   for r in sa for x in r)
    for ra, rb in zip(sa, sb):
        for x, y in zip(ra, rb):
            x.check()
            assert x.k_arena.snapshot() == y.k_arena.snapshot()
            assert x.v_arena.snapshot() == y.v_arena.snapshot()
            assert (x.buffered, x.context_len) == (y.buffered, y.context_len)
    # and the graph's outputs are the fused attention of the final states
    if group == 1:
        ref, _, _ = kv.attention_batched(sa[0], q[0].contiguous())
        assert torch.equal(ref, oa[0]) or float((ref - oa[0]).abs().max()) == 0.0


@pytest.mark.parametrize("ctxs", [(64 * 5 + 17, 64 * 7 + 17, 64 * 2 + 17),   # same step, unequal n_chunks
                                  (64 * 5 + 17, 64 * 5 + 40, 64 * 3 + 90)])  # events at different steps
def test_append_batched_ragged_events(kv, ctxs):
    """Batches whose overflow events differ per state take the per-state
    shift; the arenas, counts and live pairs equal append_token's."""
    import torch
    H, extra = 2, 240
    data = [_data(c, extra, H, 40 + i) for i, c in enumerate(ctxs)]
    a = [_prefill(kv, k, v, c) for (k, v), c in zip(data, ctxs)]
    b_ = [_prefill(kv, k, v, c) for (k, v), c in zip(data, ctxs)]
    cache = kv.kvcache._BatchDesc()
    for j in range(extra):
        kd = torch.from_numpy(np.stack([d[0][c + j] for d, c in zip(data, ctxs)])).cuda()
        vd = torch.from_numpy(np.stack([d[1][c + j] for d, c in zip(data, ctxs)])).cuda()
        kv.append_batched(a, kd, vd, desc_cache=cache)
        for i, st in enumerate(b_):
            st.append_token(data[i][0][ctxs[i] + j].astype(np.float32),
                            data[i][1][ctxs[i] + j].astype(np.float32))
    for i in range(len(ctxs)):
        a[i].check()
        assert a[i].k_arena.snapshot() == b_[i].k_arena.snapshot()
        assert a[i].v_arena.snapshot() == b_[i].v_arena.snapshot()
        assert (a[i].buffered, a[i].compressed_tokens) == (b_[i].buffered, b_[i].compressed_tokens)
        assert a[i]._live.tolist() == [a[i].n_chunks, a[i].buffered]
        a[i].settle()
        b_[i].settle()
        assert a[i].stage_bytes() == b_[i].stage_bytes()
