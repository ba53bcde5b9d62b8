"""Head-sharded Store/Fetch through the product path on the GPU,
two ranks on one B200 over gloo (CUDA tensors): LayerCacheState.prefill_many
with a process group (one histogram all-reduce per call), growing-cache
appends (no collective), the fused fetch on each rank's heads and
gather_head_outputs.  The reassembled arenas must equal the single-process
state's byte for byte and the gathered outputs its attention."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, D, CTX, B, EXTRA = 4, 128, 64 * 5 + 19, 3, 150


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    import oracle
    ks = [oracle.generate_synthetic(CTX + EXTRA, H, D, seed=70 + b).astype(np.float16)
          for b in range(B)]
    vs = [oracle.generate_synthetic(CTX + EXTRA, H, D, seed=80 + b).astype(np.float16)
          for b in range(B)]
    q = np.random.default_rng(9).standard_normal((B, H, D), dtype=np.float32)
    return np.stack(ks), np.stack(vs), q


def _build(kv, torch, ks, vs, head_base, heads, group=None):
    ck, cv = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    sl = slice(head_base, head_base + heads)
    items = [(torch.from_numpy(np.ascontiguousarray(ks[b, :CTX, sl])).cuda(),
              torch.from_numpy(np.ascontiguousarray(vs[b, :CTX, sl])).cuda()) for b in range(B)]
    states = kv.LayerCacheState.prefill_many(items, ck, cv, head_base=head_base, head_total=H,
                                             process_group=group)
    kd = torch.from_numpy(np.ascontiguousarray(ks[:, :, sl])).cuda()
    vd = torch.from_numpy(np.ascontiguousarray(vs[:, :, sl])).cuda()
    cache = kv.kvcache._BatchDesc()
    for t in range(CTX, CTX + EXTRA):  # crosses an overflow event: no collective
        kv.append_batched(states, kd[:, t], vd[:, t], desc_cache=cache)
    for s in states:
        s.check()
    return states


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2509_00579_b200 as kv
        from paper_2509_00579_b200.sharded import HeadShard, gather_head_outputs
        ks, vs, q = _data()
        sh = HeadShard(rank, world, H)
        states = _build(kv, torch, ks, vs, sh.head_base, sh.heads_local, group=dist.group.WORLD)
        ql = torch.from_numpy(np.ascontiguousarray(q[:, sh.head_base: sh.head_base +
                                                     sh.heads_local])).cuda()
        out_l, _, err = kv.attention_batched(states, ql)
        assert int(err.item()) == 0
        out = gather_head_outputs(out_l)
        parts = [None] * world
        dist.all_gather_object(parts, [(s.k_arena.snapshot(), s.k_arena.block_offsets.tolist(),
                                        s.v_arena.snapshot(), s.v_arena.block_offsets.tolist(),
                                        s.k_codebook.code_lengths.tolist())
                                       for s in states])
        if rank == 0:
            from paper_2509_00579_b200.sharded import interleave_shard_arenas
            full = _build(kv, torch, ks, vs, 0, H)
            ref, _, _ = kv.attention_batched(full, torch.from_numpy(q).cuda())
            res = {"arenas": True, "books": True}
            for b in range(B):
                gk = interleave_shard_arenas([(p[b][0], p[b][1]) for p in parts])
                gv = interleave_shard_arenas([(p[b][2], p[b][3]) for p in parts])
                res["arenas"] &= (gk[0] == full[b].k_arena.snapshot()
                                  and np.array_equal(gk[1], full[b].k_arena.block_offsets)
                                  and gv[0] == full[b].v_arena.snapshot()
                                  and np.array_equal(gv[1], full[b].v_arena.block_offsets))
                res["books"] &= all(p[b][4] == full[b].k_codebook.code_lengths.tolist()
                                    for p in parts)
            res["out_err"] = float((out - ref).abs().max() / ref.abs().max())
            out_q.put(res)
    finally:
        dist.destroy_process_group()


def test_two_rank_head_sharded_product_path():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    res = q.get()
    assert res["books"] and res["arenas"]
    assert res["out_err"] <= 1e-6
