#!/usr/bin/env python
"""Headline bench over the workload seeds {0, 1, 2} (SURVEY.md §8(d) "Seeds and runs": report mean ± std of
3 runs, paper P:513; weight seed 1234).  Each seed is one `bench.py --seed s` run (device value and e2e);
writes profiles/<round>/seeds.json.

    python scripts/seed_runs.py r02 [extra bench.py args]
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
    extra = sys.argv[2:]
    runs = []
    for seed in (0, 1, 2):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--seed", str(seed),
                              "--no-cpu-baseline", *extra], capture_output=True, text=True, cwd=ROOT)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        if out.returncode != 0 or not line:
            sys.exit(f"seed {seed}: bench.py failed\n{out.stderr[-2000:]}")
        d = json.loads(line[-1])
        runs.append({"seed": seed, "value": d["value"], "e2e": d.get("e2e", {}).get("value"),
                     "ttfo_s": d.get("e2e", {}).get("ttfo_s"), "sm_mhz": d["clocks"]["sm_mhz"],
                     "superbatches": d["config"].get("superbatches_per_step"),
                     "safety_flushes": d.get("e2e", {}).get("safety_flushes"),
                     "peak_buffered_texts": d.get("e2e", {}).get("peak_buffered_texts"),
                     "lemma_bound_texts": d.get("e2e", {}).get("lemma_bound_texts")})
        print(json.dumps(runs[-1]), flush=True)
    vals = [r["value"] for r in runs]
    e2e = [r["e2e"] for r in runs if r["e2e"]]
    summary = {"metric": d["metric"], "unit": d["unit"], "runs": runs,
               "value_mean": statistics.mean(vals), "value_std": statistics.stdev(vals),
               "e2e_mean": statistics.mean(e2e) if e2e else None,
               "e2e_std": statistics.stdev(e2e) if len(e2e) > 1 else None}
    os.makedirs(os.path.join(ROOT, "profiles", rnd), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", rnd, "seeds.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: summary[k] for k in ("value_mean", "value_std", "e2e_mean", "e2e_std")}))


if __name__ == "__main__":
    main()
