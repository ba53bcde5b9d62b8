"""Where the time of a streaming-decode overflow event goes (host phases,
synchronised brackets).  Not a bench: a diagnostic for DecodeLoop.

  python tools/stream_prof.py --layers 8 --batch 8 --ctx 32768 --heads 40
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=40)
    a = ap.parse_args()
    import torch
    import paper_2509_00579_b200 as kv
    from paper_2509_00579_b200 import kvcache
    dev = torch.device("cuda", 0)
    L, B, T, H = a.layers, a.batch, a.ctx, a.heads
    kv.reserve_arena_pool(int(1.1 * 0.3 * 2 * L * B * T * H * 128 * 2), dev)
    cfg_k, cfg_v = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    states = []
    for l in range(L):
        items = []
        for b in range(B):
            k = kv.generate_synthetic_device(kv.SyntheticSpec(T, H, 128, seed=l * 8 + b), dev)
            v = kv.generate_synthetic_device(kv.SyntheticSpec(T, H, 128, seed=l * 8 + b + 99), dev)
            items.append((k, v))
        row = kv.LayerCacheState.prefill_many(items, cfg_k, cfg_v)
        for st in row:
            st.compact(headroom=16 * 2 * H * 8192)
        states.append(row)
        del items
    torch.cuda.synchronize()
    kn = torch.randn((L, B, H, 128), device=dev, dtype=torch.float16)
    vn = torch.randn_like(kn)
    q = torch.randn((L, B, H, 128), device=dev)
    out = torch.empty_like(q)

    def sync_t(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3, r

    loop = kv.DecodeLoop(states, use_graph=False)
    # advance to one step before the overflow
    while states[0][0].buffered + 1 <= 128:
        loop.step(kn, vn, q, out)
    torch.cuda.synchronize()
    # instrumented event step
    ms_total, _ = sync_t(lambda: loop.step(kn, vn, q, out))
    print(f"event step total (synced): {ms_total:.1f} ms")
    # break the event work down on a fresh overflow: time the pieces directly
    while states[0][0].buffered + 1 <= 128:
        loop.step(kn, vn, q, out)
    torch.cuda.synchronize()
    caches = loop.caches
    tt = {"append_batched_host": 0.0, "store": 0.0, "shift": 0.0, "attention": 0.0}
    for layer, row in enumerate(states):
        t0 = time.perf_counter()
        kvcache._BatchDesc.get(caches[layer], row)
        kernel_rows = (kn[layer], vn[layer])
        import paper_2509_00579_b200._lib as _lib
        ddev, _ = caches[layer].get(row)
        _lib.check(_lib.lib().kvc_buffer_append(ddev.data_ptr(), B, H, 128, 129,
                                                kernel_rows[0].data_ptr(), kernel_rows[1].data_ptr(),
                                                _lib.KVC_F16, H * 128, None,
                                                torch.cuda.current_stream().cuda_stream))
        tt["append_batched_host"] += time.perf_counter() - t0
        for s in row:
            n = s._after_append()
            t1, _ = sync_t(lambda: s._compress_buffer(n))
            tt["store"] += t1 / 1e3
            rem = s.buffered - n
            t2, _ = sync_t(lambda: _lib.check(_lib.lib().kvc_buffer_shift(
                s.desc_device().data_ptr(), 1, H, 128, n, rem, s.n_chunks,
                torch.cuda.current_stream().cuda_stream)))
            s.buffered = rem
            tt["shift"] += t2 / 1e3
        t3, _ = sync_t(lambda: loop._attend(layer, q[layer], out[layer]))
        tt["attention"] += t3 / 1e3
    print({k: round(v * 1e3, 2) for k, v in tt.items()}, "ms over", L, "layers")
    # graph capture cost
    gl = kv.DecodeLoop(states, use_graph=True)
    t, _ = sync_t(lambda: gl.step(kn, vn, q, out))
    print(f"first graph step (settle + capture + replay): {t:.1f} ms")
    t, _ = sync_t(lambda: gl.step(kn, vn, q, out))
    print(f"graph replay step: {t:.1f} ms")
    for i in range(3):
        t, _ = sync_t(lambda: loop.step(kn, vn, q, out))
        print(f"eager step {i}: {t:.1f} ms")
    for i in range(3):
        t, _ = sync_t(lambda: gl.step(kn, vn, q, out))
        print(f"graph step {i}: {t:.1f} ms")
    for layer in range(L):
        t1, _ = sync_t(lambda: kv.append_batched(states[layer], kn[layer], vn[layer],
                                                 desc_cache=loop.caches[layer]))
        t2, _ = sync_t(lambda: loop._attend(layer, q[layer], out[layer]))
        print(f"layer {layer}: append {t1:.2f} ms, attention {t2:.2f} ms")


if __name__ == "__main__":
    main()
