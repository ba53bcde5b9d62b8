"""Host-side profile of LayerCacheState.prefill (cProfile, sorted by cumulative time)."""
import cProfile, pstats, time, sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_00579_b200 as kv
dev = torch.device('cuda', 0)
for (T, H) in ((32768, 40), (131072, 8)):
    k = torch.empty((T, H, 128), dtype=torch.float16, device=dev)
    v = torch.empty_like(k)
    kv.generate_synthetic_device(kv.SyntheticSpec(T, H, 128, seed=1), dev, out=k)
    kv.generate_synthetic_device(kv.SyntheticSpec(T, H, 128, seed=2), dev, out=v)
    ck, cv = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    keep = []
    kv.reserve_arena_pool(8 << 30, dev)
    for _ in range(3):
        keep.append(kv.LayerCacheState.prefill(k, v, ck, cv, check=False))
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        t0 = time.perf_counter(); st = kv.LayerCacheState.prefill(k, v, ck, cv, check=False); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0); keep.append(st)
    print(T, H, 'prefill ms', [round(t * 1e3, 3) for t in ts])
    pr = cProfile.Profile(); pr.enable()
    for _ in range(10):
        keep.append(kv.LayerCacheState.prefill(k, v, ck, cv, check=False))
        torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats('tottime').print_stats(18)
    break
