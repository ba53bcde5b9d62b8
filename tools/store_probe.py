"""One prefill of a config-2 (seq, layer) slice (32K x 40 heads x 128 fp16) through
LayerCacheState.prefill, for ncu captures of the Store passes.
  python tools/store_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2509_00579_b200 as kv
    dev = torch.device("cuda", 0)
    k = kv.generate_synthetic_device(kv.SyntheticSpec(32768, 40, 128, seed=0), dev)
    v = kv.generate_synthetic_device(kv.SyntheticSpec(32768, 40, 128, seed=1), dev)
    ck, cv = kv.QuantConfig(kv.QuantMode.K_BLOCK), kv.QuantConfig(kv.QuantMode.V_TOKEN)
    for _ in range(3):
        st = kv.LayerCacheState.prefill(k, v, ck, cv)
    torch.cuda.synchronize()
    print("ratio", kv.collect_stats(st).compression_ratio)


if __name__ == "__main__":
    main()
