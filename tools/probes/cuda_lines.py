"""Stall samples per CUDA source line from `ncu -i rep --page source --csv --print-source cuda,sass`.

usage: python tools/probes/cuda_lines.py <src.csv> [top]
Prints the top lines by warp-stall samples with their two largest stall reasons and executed instructions."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
    cur, hdr = None, None
    agg, inst, src = collections.Counter(), collections.Counter(), {}
    reasons = collections.defaultdict(collections.Counter)
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or r[2] != "-":
            continue
        d = dict(zip(hdr, r))
        key = (cur, int(r[0]))
        src[key] = r[1]
        agg[key] += float(d["Warp Stall Sampling (All Samples)"] or 0)
        inst[key] += float(d["Instructions Executed"] or 0)
        for k in hdr:
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    reasons[key][k[6:]] += float(d[k] or 0)
                except ValueError:
                    pass
    tot = sum(agg.values()) or 1
    ti = sum(inst.values()) or 1
    print(f"samples {tot:.0f} warp-instructions {ti:.3g}")
    for key, v in agg.most_common(top):
        rs = ", ".join(f"{k} {x / v * 100:.0f}%" for k, x in reasons[key].most_common(2) if v)
        print(f"{v / tot * 100:5.1f}% inst {inst[key] / ti * 100:5.1f}% {key[0]}:{key[1]:<4} {src[key].strip()[:70]:70} | {rs}")


if __name__ == "__main__":
    main()
