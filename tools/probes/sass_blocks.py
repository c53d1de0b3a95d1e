"""Per-block share of executed warp-instructions of k_improve<1,false> from an ncu SourceCounters capture.

usage: python tools/probes/sass_blocks.py <ncu source csv (--page source --csv --print-source sass)> <kernel.cubin>
The cubin must be compiled from the same sources with -lineinfo (nvcc -cubin ... csrc/improve.cu); SASS
offsets of the capture are mapped to source lines through `nvdisasm -g` of that cubin.
"""
import collections
import csv
import re
import subprocess
import sys

KERNEL = "_ZN8plse_dev9k_improveILi1ELb0EEEvNS_11ImproveArgsE"
CSRC = __import__("os").environ.get("CSRC_DIR") or __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)),
                                  "..", "..", "paper_2103_10453_b200", "csrc")
_FUNCS = {}


def enclosing_function(f, l):
    """name of the __device__ helper of csrc/<f> whose definition precedes line l"""
    if f not in _FUNCS:
        starts = []
        try:
            for i, t in enumerate(open(__import__("os").path.join(CSRC, f)), 1):
                m = re.search(r"__device__.*?(\w+)\(", t)
                if m:
                    starts.append((i, m.group(1)))
        except OSError:
            pass
        _FUNCS[f] = starts
    name = None
    for i, n in _FUNCS[f]:
        if i <= l:
            name = n
    return name


def line_map(cubin):
    sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True, check=True).stdout
    out, cur, on = {}, None, False
    for l in sass.splitlines():
        if ".text." in l and ":" in l:
            on = KERNEL in l
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+", l)
        if m and cur:
            out[int(m.group(1), 16)] = cur
    return out


_SECTIONS = {}


def section(f, l):
    """the last `// ----` / `// ====` section comment of csrc/<f> at or before line l"""
    if f not in _SECTIONS:
        marks = []
        for i, t in enumerate(open(__import__("os").path.join(CSRC, f)), 1):
            m = re.match(r"\s*// [-=]{4,}\s*(.*)", t)
            if m:
                marks.append((i, m.group(1).strip()[:60]))
        _SECTIONS[f] = marks
    name = None
    for i, n in _SECTIONS[f]:
        if i <= l:
            name = n
    return name


def block(f, l):
    if f == "improve.cu":
        return "improve.cu: " + (section(f, l) or "other")
    fn = enclosing_function(f, l) if f.endswith((".cuh", ".h")) else None
    return f + ":" + fn if fn else "other (" + f + ")"


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, data = rows[1], rows[2:]
    ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
    base = int(data[0][ia], 16)
    lm = line_map(sys.argv[2])
    per = collections.Counter()
    for r in data:
        f, l = lm.get(int(r[ia], 16) - base, ("?", -1))
        per[block(f, l)] += int(r[iex] or 0)
    tot = sum(per.values())
    print(f"total warp-instructions {tot:.4g}")
    for k, v in per.most_common():
        print(f"{100 * v / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
