"""Summarise one ncu --set full capture of an improve kernel into profiles/<kernel>_ncu_summary.json,
the file bench.py's roofline reads (matched on the kernel's source hash and the config key).

usage: python tools/probes/ncu_summary.py <raw.csv from `ncu -i rep --page raw --csv`> <probe log> <kernel>
       <config_key> <out.json>
The probe log is improve_probe.py's output of the same run; the launch's move count is taken from the
generation line of the profiled launch (GEN env var, default 2).
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    raw, log, kernel, key, out = sys.argv[1:6]
    gen = int(os.environ.get("GEN", "2"))
    with open(raw) as f:
        rows = list(csv.reader(f))
    hdr, units = rows[0], rows[1]
    data = [r for r in rows[2:] if any(kernel in c for c in r)]
    if not data:
        raise SystemExit(f"no {kernel} launch in {raw}")
    r = dict(zip(hdr, data[0]))
    u = dict(zip(hdr, units))

    def metric(name, scale_to=None):
        v = num(r.get(name))
        if v is None:
            return None
        unit = u.get(name, "")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9,
                "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                "s": 1.0}.get(unit, 1.0)
        return v * mult

    moves = None
    with open(log) as f:
        for line in f:
            m = re.match(rf"gen {gen} moves (\d+)", line)
            if m:
                moves = int(m.group(1))
    import bench
    dur = metric("gpu__time_duration.sum")
    rd = metric("dram__bytes_read.sum")
    wr = metric("dram__bytes_write.sum")
    inst = num(r.get("smsp__inst_executed.sum"))
    summary = {
        "kernel": kernel, "src_hash": bench.kernel_src_hash(kernel), "config_key": key,
        "launch_ms": dur * 1e3 if dur else None,
        "dram_bytes_per_launch": (rd or 0) + (wr or 0) if rd is not None else None,
        "dram_read": rd, "dram_write": wr,
        "warp_inst_per_launch": inst, "moves_per_launch": moves,
        "inst_per_move": inst / moves if inst and moves else None,
        "issue_active_pct": num(r.get("sm__inst_issued.avg.pct_of_peak_sustained_active")),
        "warps_active_pct": num(r.get("sm__warps_active.avg.pct_of_peak_sustained_active")),
        "sm_ghz": num(r.get("sm__cycles_elapsed.avg.per_second")),  # ncu reports it in GHz
        "source": os.path.relpath(raw, ROOT), "generation": gen,
        "note": os.environ.get("NOTE", "ncu --clock-control none (sections SpeedOfLight/LaunchStats/Occupancy/"
                "WarpStateStats/SchedulerStats plus instruction and DRAM metrics) of one launch (the generation "
                "above) of improve_probe.py; dram bytes = dram__bytes_read.sum + dram__bytes_write.sum"),
    }
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
