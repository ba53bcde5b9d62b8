"""Host-side profile of LayerCacheState.prefill_many on config-5 slices
(8K x 32 heads x 128 fp16 per item, 64 items): wall time per item vs device
time, and the cProfile of the Python side.
  python tools/prefill_host_prof.py
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2509_00579_b200 as kv
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
    kv.LayerCacheState.prefill_many(items[:4], ck, cv)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = kv.LayerCacheState.prefill_many(items, ck, cv)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"prefill_many {B} items: {dt * 1e3:.1f} ms, {dt / B * 1e3:.3f} ms/item, "
          f"{2 * T * H * 128 * 2 * B / dt / 1e9:.1f} GB/s fp16 in")
    pr = cProfile.Profile()
    pr.enable()
    st = kv.LayerCacheState.prefill_many(items, ck, cv)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
    pstats.Stats(pr).sort_stats("cumtime").print_stats(40)


if __name__ == "__main__":
    main()
