"""Time-to-target where the generational loop matters.

For each instance: the reference's own run() (oracle/_ref = the unmodified headers, Partial-MPMA,
p = 1024 -- the CLI default, plse.cpp:29 -- on every host thread, time limit T) gives the target: its best
score and the wall time at which it first reached it.  The device run() then chases that score on the same
instance (master seed 1 for both), with the reference's semantics (parity mode: every individual runs its
whole budget) and in race mode (the improve phase stops once any individual reaches the target).

usage (GPU box): python tools/ttb_hard.py [--configs hard,c4] [--limit 600] > profiles/ttb_hard.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {
    "hard": (60, 0.7, 12345, "n=60 r=0.7 (SURVEY 6: reference best 3591 at 401 s on 8 cores, still improving)"),
    "c4": (70, 0.6, 12345, "BASELINE C4 instance (reference optimum 4900 in generation 13, 210 s on 8 cores)"),
    "c2": (50, 0.4, 12345, "BASELINE C2 instance"),
    "c3": (60, 0.5, 12345, "BASELINE C3 instance"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="hard,c4")
    ap.add_argument("--limit", type=float, default=600.0)
    ap.add_argument("--ref-pop", type=int, default=1024)
    ap.add_argument("--pops", default="16384,4096")
    ap.add_argument("--reference-from", default="",
                    help="reuse the reference runs of an earlier output (same host) instead of re-running them")
    ap.add_argument("--race-only", action="store_true")
    a = ap.parse_args()
    import oracle
    import paper_2103_10453_b200 as P
    threads = len(os.sched_getaffinity(0))
    out = {"host_threads": threads, "limit_s": a.limit, "runs": []}
    for name in a.configs.split(","):
        n, r, s, what = CONFIGS[name]
        grid = P.generate_instance(n, r, s)
        rec = {"config": name, "instance": f"generate_instance({n},{r},{s})", "what": what}
        prev = None
        if a.reference_from:
            with open(a.reference_from) as fh:
                prev = next((x for x in json.load(fh)["runs"] if x["config"] == name), None)
        if prev is not None:
            rec["reference"] = dict(prev["reference"], reused_from=a.reference_from)
            target = prev["target_score"]
        elif oracle.Reference.available():
            ref = oracle.Reference()
            t0 = time.time()
            rr = ref.run(grid, p=a.ref_pop, seed=1, workers=threads, time_limit=a.limit, variant=1, log_cap=4096)
            rec["reference"] = {"pop": a.ref_pop, "best_score": rr["best_score"], "best_f": rr["best_f"],
                                "seconds_to_best": rr["first_best_seconds"], "seconds_total": rr["elapsed_seconds"],
                                "generations": rr["generations"], "stop": rr["stop_reason"],
                                "moves": rr["total_iterations"], "cores": threads,
                                "best_f_by_generation": [g["best_f"] for g in rr["log"]],
                                "wall_s": time.time() - t0}
            target = rr["best_score"]
        else:
            rec["reference"] = "oracle/_ref not built"
            target = None
        rec["target_score"] = target
        for pop in (int(x) for x in a.pops.split(",")):
            for race in ((True,) if a.race_only else (True, False)):
                traj = []
                t0 = time.time()
                cfg = P.SolverConfig(p=pop, master_seed=1, time_limit=a.limit, target_score=float(target or 0),
                                     race=race and target is not None)
                res = P.run(grid, cfg, on_generation=lambda st: traj.append((st.generation, st.best_f,
                                                                            round(st.elapsed_seconds, 3))))
                rec[f"ours_p{pop}_{'race' if race else 'parity'}"] = {
                    "pop": pop, "best_score": res.best_score, "seconds_to_best": res.time_to_best_seconds,
                    "seconds_total": res.elapsed_seconds, "generations": res.generations, "stop": res.stop_reason,
                    "moves": res.total_iterations, "reached_target": target is not None and res.best_score >= target,
                    "trajectory": traj, "wall_s": time.time() - t0,
                    "mode": "race (device-global early exit at the target)" if race else
                            "parity (every individual runs its full budget)"}
        ref_t = rec["reference"]["seconds_to_best"] if isinstance(rec["reference"], dict) else None
        for k, v in list(rec.items()):
            if k.startswith("ours_") and ref_t and v["reached_target"] and v["seconds_to_best"] > 0:
                v["speedup_vs_reference"] = ref_t / v["seconds_to_best"]
        out["runs"].append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
