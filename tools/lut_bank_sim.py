"""Replay the fused fetch's shared-memory access pattern on real arenas and
count bank-conflict ways (wavefronts per warp instruction) for candidate
LUT layouts and for the window reloads.

The arena comes from the product Store (LayerCacheState.prefill on the GPU,
synthetic KV of the reference generator's distribution); the replay is host
numpy.  Each warp instruction = 32 lanes, lane l decoding slice l (cursor A)
or slice l + 32 (cursor B) of one block, in lockstep over the 64 pair steps,
with a 3-word window reload every 5 steps.  Wavefronts of an instruction =
the largest number of distinct 32-bit words any bank is asked for.

  python tools/lut_bank_sim.py --ctx 2048 --heads 8

This is what chose the swizzled V table (DESIGN.md §4.2 v8): plain index
4.4-way for V, index ^ ((index >> 7) & 31) 3.1-way.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LAYOUTS = {
    "plain": lambda i: i,
    "xor_top5": lambda i: i ^ ((i >> 7) & 31),   # fetch_lut_x
    "xor_mid5": lambda i: i ^ ((i >> 5) & 31),
    "bank_top5": lambda i: ((i & 127) << 5) | (i >> 7),
    "random": (lambda p: (lambda i: p[i]))(np.random.default_rng(0).permutation(4096)),
}


def pair_lengths(lengths):
    """Consumed bits of the 12-bit pair LUT for every window (codes <= 6 bits)."""
    lens = np.asarray(lengths, np.int64)
    words = {}
    code, prev = 0, 0
    for s in sorted((s for s in range(256) if lens[s]), key=lambda s: (lens[s], s)):
        code <<= int(lens[s]) - prev
        prev = int(lens[s])
        words[(prev, code)] = s
        code += 1

    def first(w):
        for L in range(1, 13):
            if (L, w >> (12 - L)) in words:
                return L
        return 12
    tab = np.zeros(4096, np.int64)
    for w in range(4096):
        l0 = first(w)
        tab[w] = l0 + first((w << l0) & 0xFFF)
    return tab


def ways(addrs):
    banks = {}
    for a in set(int(x) for x in addrs):
        banks[a % 32] = banks.get(a % 32, 0) + 1
    return max(banks.values())


def replay(arena, offsets, lengths, n_units, bs=64, max_blocks=64):
    tab = pair_lengths(lengths)
    hdr = 6 + 2 * bs + 8 * n_units
    ends = list(offsets[1:]) + [len(arena)]
    lut = {k: 0 for k in LAYOUTS}
    n_lut = reload = n_reload = 0
    for b in range(min(len(offsets), max_blocks)):
        o, e = int(offsets[b]), int(ends[b])
        counts = np.frombuffer(arena[o + 6:o + 6 + 2 * bs].tobytes(), "<u2").astype(np.int64)
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
        bits = np.concatenate([np.unpackbits(arena[o + hdr:e]), np.zeros(64, np.uint8)])
        weights = 1 << np.arange(11, -1, -1)
        base_bit = ((o & 15) + hdr) * 8
        for half in (0, 1):
            cur = starts[half * 32: half * 32 + 32].copy()
            for step in range(64):
                if step % 5 == 0:
                    for d in range(3):
                        reload += ways((base_bit + cur) // 32 + d)
                        n_reload += 1
                idx = np.array([int((bits[c:c + 12] * weights).sum()) for c in cur])
                for k, fn in LAYOUTS.items():
                    lut[k] += ways(fn(idx))
                n_lut += 1
                cur = cur + tab[idx]
    return {k: v / n_lut for k, v in lut.items()}, reload / max(n_reload, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--blocks", type=int, default=64)
    a = ap.parse_args()
    import torch
    import paper_2509_00579_b200 as kv
    dev = torch.device("cuda", 0)
    k = kv.generate_synthetic_device(kv.SyntheticSpec(a.ctx, a.heads, 128, seed=1), dev)
    v = kv.generate_synthetic_device(kv.SyntheticSpec(a.ctx, a.heads, 128, seed=2), dev)
    st = kv.LayerCacheState.prefill(k, v, kv.QuantConfig(kv.QuantMode.K_BLOCK),
                                    kv.QuantConfig(kv.QuantMode.V_TOKEN))
    for name, arena, cb, n_units in (("K", st.k_arena, st.k_codebook, 128),
                                     ("V", st.v_arena, st.v_codebook, 64)):
        raw = np.frombuffer(arena.snapshot(), np.uint8)
        lut, rel = replay(raw, arena.block_offsets, cb.code_lengths, n_units, max_blocks=a.blocks)
        print(name, "LUT ways:", {k: round(x, 3) for k, x in lut.items()},
              "reload ways:", round(rel, 3))


if __name__ == "__main__":
    main()
