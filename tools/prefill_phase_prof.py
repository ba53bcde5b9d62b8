"""Wall time of prefill_many's host phases on config-5 slices (64 items of
8K x 32 heads x 128 fp16): _prefill_begin (allocations + pass A launch),
_prefill_finish (codebooks + state + pass B), with the device idle or not.
  python tools/prefill_phase_prof.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2509_00579_b200 as kv
    from paper_2509_00579_b200.kvcache import LayerCacheState as S
    dev = torch.device("cuda", 0)
    B, T, H = 64, 8192, 32
    kv.reserve_arena_pool(int(1.2 * 0.3 * 2 * 2 * B * T * H * 128 * 2), dev)
    kb = torch.empty((B, T, H, 128), dtype=torch.float16, device=dev)
    vb = torch.empty_like(kb)
    for b in range(B):
        kv.generate_synthetic_device(kv.SyntheticSpec(T, H, 128, seed=b), dev, out=kb[b])
        kv.generate_synthetic_device(kv.SyntheticSpec(T, H, 128, seed=b + 99), dev, out=vb[b])
    ck, cv = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    items = [(kb[b], vb[b]) for b in range(B)]
    kv.LayerCacheState.prefill_many(items[:4], ck, cv)
    torch.cuda.synchronize()
    tb, tf = [], []
    ob = S.__dict__["_prefill_begin"].__func__
    of = S.__dict__["_prefill_finish"].__func__

    def pb(cls, *a, **k):
        t = time.perf_counter()
        r = ob(cls, *a, **k)
        tb.append(time.perf_counter() - t)
        return r

    def pf(*a, **k):
        t = time.perf_counter()
        r = of(*a, **k)
        tf.append(time.perf_counter() - t)
        return r

    S._prefill_begin, S._prefill_finish = classmethod(pb), staticmethod(pf)
    t0 = time.perf_counter()
    st = kv.LayerCacheState.prefill_many(items, ck, cv, check=False)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    n = len(items)
    print(f"host {1e3 * (t1 - t0) / n:.3f} ms/item, +sync {1e3 * (t2 - t0) / n:.3f}; begin "
          f"{1e3 * sum(tb) / n:.3f}, finish {1e3 * sum(tf) / n:.3f} ms/item")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    st = kv.LayerCacheState.prefill_many(items, ck, cv, check=False)
    ev1.record()
    torch.cuda.synchronize()
    print(f"device span {ev0.elapsed_time(ev1) / n:.3f} ms/item")


if __name__ == "__main__":
    main()
