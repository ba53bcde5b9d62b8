"""Graph-vs-eager decode steps on bench-built states (config-2 shape, few
layers): device ms per step of each mode in steady state, and the host time
of the overflow step's phases.  A diagnostic, not a bench.
  python tools/graph_diag.py --layers 8
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
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--heads", type=int, default=40)
    ap.add_argument("--side-stream", action="store_true",
                    help="run both loops on a created (non-default) stream")
    ap.add_argument("--profile-capture", action="store_true",
                    help="cProfile each re-capture (top functions by cumulative time)")
    a = ap.parse_args()
    import torch
    import bench
    import paper_2509_00579_b200 as kv
    from paper_2509_00579_b200 import decode_loop
    dev = torch.device("cuda", 0)
    L, B, T, H = a.layers, a.batch, a.ctx, a.heads
    kv.reserve_arena_pool(int(1.1 * 0.3 * 2 * L * B * T * H * 128 * 2), dev)
    states, _, _ = bench.build_cache(kv, torch, L, B, T, H, 0, H, dev)
    q = torch.randn((L, B, H, 128), device=dev)
    out = torch.empty_like(q)
    kn = (torch.randn((L, B, H, 128), device=dev) * 0.5).half()
    vn = (torch.randn((L, B, H, 128), device=dev) * 0.5).half()
    if a.side_stream:
        torch.cuda.set_stream(torch.cuda.Stream(dev))
    stream = torch.cuda.current_stream(dev)
    orig = decode_loop.DecodeLoop._capture
    cap_t = []

    def cap(self, *args):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if a.profile_capture:
            import cProfile
            import pstats
            pr = cProfile.Profile()
            pr.enable()
            orig(self, *args)
            pr.disable()
            pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
        else:
            orig(self, *args)
        torch.cuda.synchronize()
        cap_t.append(time.perf_counter() - t)
    decode_loop.DecodeLoop._capture = cap
    if os.environ.get("DIAG_BENCH"):
        no_app = 0.947 * L
        def layer_stages():
            out = []
            for r in states:
                sk = max(st.stage_bytes()[0] for st in r)
                sv = max(st.stage_bytes()[1] for st in r)
                out.append(sk + sv)
            return sorted(out)
        sb0 = layer_stages()
        res = bench.streaming_block(kv, torch, None, states, 1, q, out, stream, a.steps, 1, dev,
                                    no_app)
        sb1 = layer_stages()
        print("layer sk+sv before", sb0[-4:], "after", sb1[-4:], "(2-CTA limit ~9822)")
        print({k: res[k] for k in ("eager", "graph")})
        return
    for name, g in (("eager", False), ("graph", True)):
        loop = kv.DecodeLoop(states, use_graph=g)
        for _ in range(3):
            loop.step(kn, vn, q, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        per = []
        for i in range(a.steps):
            e0.record(stream)
            loop.step(kn, vn, q, out)
            e1.record(stream)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1))
        per.sort()
        print(f"{name}: median {per[len(per) // 2]:.3f} ms/step, min {per[0]:.3f}, max {per[-1]:.3f}, "
              f"events {loop.events}, captures {loop.captures}")
    print("capture host s:", [round(x, 3) for x in cap_t])


if __name__ == "__main__":
    main()
