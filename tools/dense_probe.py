"""One call of the fp16 dense comparator at a BASELINE config's shape (for ncu):
  python tools/dense_probe.py --config 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2509_00579_b200 as kv
    p = bench.PRESETS[a.config]
    B, T, H, G = p["batch"], p["ctx"], p["heads"], p["group"]
    k = torch.randn((B, H, T, 128), device="cuda", dtype=torch.float16)
    v = torch.randn_like(k)
    q = torch.randn((B, H * G, 128), device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kv.dense_attention_f16(k, v, q, group=G)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        kv.dense_attention_f16(k, v, q, group=G)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    print(f"dense fp16 G={G}: {ms:.4f} ms/layer, {2 * B * H * T * 128 * 2 / ms / 1e9:.3f} TB/s")


if __name__ == "__main__":
    main()
