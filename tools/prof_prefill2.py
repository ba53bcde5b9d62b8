"""Prefill/append wall time with many compressed states alive (bench-like)."""
import cProfile, pstats, time, sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_00579_b200 as kv
import bench
dev = torch.device('cuda', 0)
T, H, L, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
states, st_times, nbytes = bench.build_cache(kv, torch, L, B, T, H, 0, H, dev)
print('build prefill ms', [round(t * 1e3, 2) for t in st_times[-8:]], 'median GB/s', nbytes / sorted(st_times)[len(st_times)//2] / 1e9)
sys.path.insert(0, 'tools')
import store_bench
pr = cProfile.Profile(); pr.enable()
d = store_bench.main(ctx=T, H=H, D=128, reps=5)
pr.disable()
print(d['append_event'], d['prefill_slice']['prefill_gbs'])
pstats.Stats(pr).sort_stats('tottime').print_stats(12)
