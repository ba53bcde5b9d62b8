"""Time the fused fetch-attention launch on one layer of a BASELINE config under
several decoder variants (selected through the KVC_FUSED_* environment
variables that kvc_attention reads at launch time).

  python tools/fetch_variants.py --config 2 --variants "base;KVC_FUSED_VMODE=0"
  python tools/fetch_variants.py --config 3 --iters 1     # single launch (for ncu)

Prints one line per variant: ms per layer launch (CUDA events, after warm-up),
equivalent-fp16 TB/s and compressed TB/s.  Never a bench number: bench.py is.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_00579_b200 as kv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 5])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--heads", type=int, default=None)
    ap.add_argument("--variants", default="base")
    ap.add_argument("--rel-k", type=str, default=None, help="float, or 1/255")
    ap.add_argument("--rel-v", type=str, default=None)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--check", action="store_true", help="compare every variant's output with base")
    a = ap.parse_args()
    frac = lambda x: None if x is None else (1.0 / 255.0 if x == "1/255" else float(x))
    a.rel_k, a.rel_v = frac(a.rel_k), frac(a.rel_v)
    p = dict(bench.PRESETS[a.config])
    B = a.batch or p["batch"]
    T = a.ctx or p["ctx"]
    H, G = a.heads or p["heads"], p["group"]
    dev = torch.device("cuda", 0)
    states, _, _ = bench.build_cache(kv, torch, 1, B, T, H, 0, H, dev, rel_k=a.rel_k,
                                     rel_v=a.rel_v)
    s0 = states[0][0]
    print(f"k max len {s0.k_codebook.max_code_length}, v max len {s0.v_codebook.max_code_length}, "
          f"stage bytes {s0.stage_bytes()}", flush=True)
    row = states[0]
    comp = sum(s.k_arena.size_bytes + s.v_arena.size_bytes for s in row)
    eq = 2 * T * H * 128 * 2 * B
    q = torch.randn((B, H * G, 128), device=dev)
    out = torch.empty_like(q)
    cache = kv.attention._BatchDesc()
    ws = torch.empty(bench._lib_ws(kv, B, H * G, max(s.n_chunks for s in row)), dtype=torch.uint8,
                     device=dev)

    def call():
        if G == 1:
            kv.attention_batched(row, q, desc_cache=cache, workspace=ws, out=out)
            return out
        return kv.attention_gqa(row, q, G, desc_cache=cache, workspace=ws, check=False)

    ref = None
    for var in a.variants.split(";"):
        env = {}
        if var != "base":
            for kvp in var.split(","):
                k, v = kvp.split("=")
                env[k] = v
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            o = call().clone()
            torch.cuda.synchronize()
            if a.iters > 1:
                for _ in range(3):
                    call()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.iters):
                call()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            err = ""
            if ref is None:
                ref = o
            elif a.check:
                d = float((o - ref).abs().max() / ref.abs().max())
                err = f" rel-diff-vs-first {d:.2e}"
            print(f"{var:40s} {ms:8.4f} ms/layer  eq {eq / ms / 1e9:6.3f} TB/s  "
                  f"comp {comp / ms / 1e9:6.3f} TB/s{err}", flush=True)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


if __name__ == "__main__":
    main()
