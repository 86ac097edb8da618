"""The paper's Table 2 protocol on one B200 (context numbers).

Two moons / three circles at n = 15k, 30k, 45k (the reference's own
generators, noise 0.05 = the reference CLI default), cosine similarity,
maxiterations = 3 (the CLI --bench-preset, cli.py:105-108), precision
1e-5/n, averaged over 10 runs as in the paper. Each run
is the public `report.benchmark` path: host X in, labels + v out, per-phase
CUDA-event times. Prints one JSON document; the paper's K40m GPIC seconds
are quoted beside each row for context (different hardware and code).

    python scripts/paper_table2.py [--reps 10] [--out profiles/r1_paper_table2.json]
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

PAPER_K40M_S = {  # PAPER.md:342-347 (European decimal commas)
    ("two-moons", 15000): 3.99, ("three-circles", 15000): 4.03,
    ("two-moons", 30000): 18.00, ("three-circles", 30000): 18.03,
    ("two-moons", 45000): 45.07, ("three-circles", 45000): 45.90,
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--storage", default="packed", choices=["packed", "dense"])
    args = ap.parse_args()

    import torch

    from paper_1604_02700_b200 import Cosine, KernelConfig, PicParams
    from paper_1604_02700_b200 import report as R
    from paper_1604_02700_b200.datasets import three_circles, two_moons

    make = {"two-moons": (two_moons, 2), "three-circles": (three_circles, 3)}
    cfg = KernelConfig(storage=args.storage)
    rows = []
    for n in (15000, 30000, 45000):
        for shape, (gen, k) in make.items():
            d = gen(n, 0.05, 0)
            params = PicParams(k=k, max_iterations=3)
            R.run_timed(d, Cosine(), params, config=cfg)  # warm-up (module load, graph build)
            torch.cuda.synchronize()
            rep, last = R.benchmark(d, Cosine(), params, config=cfg, repetitions=args.reps)
            doc = rep.to_dict()
            rows.append({
                "dataset": shape, "n": n, "k": k, "A_fp32_gb": 4.0 * n * n / 1e9,
                "mean_s": doc["mean_seconds"], "stddev_s": doc["stddev_seconds"],
                "phases_ms": {p: 1e3 * sum(r["phases"][p] for r in doc["runs"]) / len(doc["runs"])
                              for p in R.PHASES},
                "iterations": last.trace.iterations_run, "ari_vs_truth": doc["ari"],
                "paper_gpic_k40m_s": PAPER_K40M_S[(shape, n)],
                "ratio_vs_paper": PAPER_K40M_S[(shape, n)] / doc["mean_seconds"],
            })
            print(json.dumps(rows[-1]), flush=True)
    out = {"protocol": "cosine, maxiterations=3, epsilon=1e-5/n, noise 0.05, seed 0, "
                       f"{args.reps} reps, storage={args.storage}, 1x B200",
           "device": torch.cuda.get_device_name(0), "rows": rows}
    if args.out:
        pathlib.Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
