"""World-size-2 CPU (gloo) test of the multi-GPU host logic:
histogram all-reduce -> identical codebooks on every rank, per-rank head-shard
arenas that reassemble byte-for-byte into the single-process arena, and the
all-gather of per-head attention outputs.  The per-rank compressor here is the
CPU oracle standing in for the device (this is a test of the exchange steps and
the global block numbering, not of the kernels)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

H, D, CTX, BS = 4, 128, 64 * 4 + 19, 64


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2509_00579_b200.codebook import build_smoothed_codebook
        from paper_2509_00579_b200.sharded import (HeadShard, allreduce_histograms,
                                                   gather_head_outputs, interleave_shard_arenas)
        sh = HeadShard(rank, world, H)
        k = oracle.generate_synthetic(CTX, H, D, seed=21).astype(np.float16)
        v = oracle.generate_synthetic(CTX, H, D, seed=22).astype(np.float16)
        kl, vl = sh.slice(k).astype(np.float32), sh.slice(v).astype(np.float32)
        hist = torch.zeros(512, dtype=torch.int64)
        hist[:256] = torch.from_numpy(oracle.tokens_histogram(kl, BS, "kblock", 0.05).astype(np.int64))
        hist[256:] = torch.from_numpy(oracle.tokens_histogram(vl, BS, "vtoken", 0.15).astype(np.int64))
        allreduce_histograms(hist)
        h = hist.numpy().astype(np.uint64)
        kcb = build_smoothed_codebook(h[:256], 20)
        vcb = build_smoothed_codebook(h[256:], 7)
        n_full = (CTX // BS) * BS
        ka, ko = oracle.compress_shard(kl[:n_full], BS, "kblock", 0.05, kcb.code_lengths, H,
                                       sh.head_base)
        va, vo = oracle.compress_shard(vl[:n_full], BS, "vtoken", 0.15, vcb.code_lengths, H,
                                       sh.head_base)
        shards = [None] * world
        dist.all_gather_object(shards, (ka, ko.tolist(), va, vo.tolist(),
                                        kcb.code_lengths.tolist()))
        # attention for this rank's heads, then gather across ranks
        st = oracle.OracleState.prefill(sh.slice(k), sh.slice(v),
                                        codebooks=(kcb.code_lengths, vcb.code_lengths))
        q = np.random.default_rng(7).standard_normal((H, D), dtype=np.float32)
        out_l, _ = st.attention_step(q[sh.head_base: sh.head_base + sh.heads_local])
        out = gather_head_outputs(torch.from_numpy(out_l).unsqueeze(0))
        if rank == 0:
            full = oracle.OracleState.prefill(k, v)
            gk = interleave_shard_arenas([(s[0], s[1]) for s in shards])
            gv = interleave_shard_arenas([(s[2], s[3]) for s in shards])
            ref_out, _ = full.attention_step(q)
            out_q.put({
                "same_codebooks": all(s[4] == shards[0][4] for s in shards),
                "k_equal": gk[0] == full.arena_bytes("k")
                and np.array_equal(gk[1], full.block_offsets("k")),
                "v_equal": gv[0] == full.arena_bytes("v")
                and np.array_equal(gv[1], full.block_offsets("v")),
                "lengths_equal": list(full.k_lengths) == list(kcb.code_lengths),
                "out_err": float(np.abs(out[0].numpy() - ref_out).max() / np.abs(ref_out).max()),
            })
    finally:
        dist.destroy_process_group()


def test_two_rank_head_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = q.get()
    assert res["same_codebooks"] and res["lengths_equal"]
    assert res["k_equal"] and res["v_equal"]
    assert res["out_err"] <= 1e-5


def test_head_shard_math():
    from paper_2509_00579_b200.sharded import HeadShard
    s = HeadShard(3, 8, 40)
    assert (s.heads_local, s.head_base) == (5, 15)
    with pytest.raises(ValueError):
        HeadShard(0, 3, 40)
