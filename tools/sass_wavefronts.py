"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
shared-memory wavefronts, executed instructions and stall samples per SASS
opcode class, so decoder variants can be compared per instruction kind.

  python tools/sass_wavefronts.py gpurun_out/x_src.csv [--top 40]
"""
import argparse
import collections
import csv
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=0, help="also list the N hottest instructions")
    a = ap.parse_args()
    with open(a.csv) as fh:
        rows = list(csv.reader(fh))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {h: i for i, h in enumerate(hdr)}

    def num(r, k):
        try:
            return float(r[col[k]].replace(",", ""))
        except (KeyError, ValueError, IndexError):
            return 0.0

    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
    insts = []
    tot = [0.0, 0.0, 0.0]
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        src = r[col["Source"]]
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
        if not m:
            continue
        op = m.group(2) + (m.group(3) or "")
        op = re.sub(r"\.(reuse)", "", op)
        ex = num(r, "Instructions Executed")
        wf = num(r, "L1 Wavefronts Shared")
        ideal = num(r, "L1 Wavefronts Shared Ideal")
        smp = num(r, "Warp Stall Sampling (All Samples)")
        g = agg[op.split(".")[0] if not op.startswith("LDS") else op]
        g[0] += ex
        g[1] += wf
        g[2] += ideal
        g[3] += smp
        tot[0] += ex
        tot[1] += wf
        tot[2] += smp
        insts.append((smp, ex, wf, r[col["Address"]], src.strip()))
    print(f"total: {tot[0] / 1e6:.1f} M warp instr, {tot[1] / 1e6:.1f} M shared wavefronts, "
          f"{tot[2]:.0f} stall samples")
    print(f"{'op':22s} {'M instr':>9s} {'M wavefr':>9s} {'wf/instr':>8s} {'ideal':>6s} {'samples%':>8s}")
    for op, (ex, wf, ideal, smp) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if ex < tot[0] * 0.002 and wf < tot[1] * 0.002:
            continue
        print(f"{op:22s} {ex / 1e6:9.2f} {wf / 1e6:9.2f} {wf / ex if ex else 0:8.2f} "
              f"{ideal / ex if ex else 0:6.2f} {100 * smp / max(tot[2], 1):8.1f}")
    if a.top:
        for smp, ex, wf, addr, src in sorted(insts, reverse=True)[: a.top]:
            print(f"{addr:>8s} {smp:8.0f} {ex / 1e6:7.2f}M {wf / max(ex, 1):5.2f}wf  {src[:70]}")


if __name__ == "__main__":
    main()
