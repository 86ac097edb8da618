"""Experiment II: the subsampling sweep on the batched GPU engine.

`run_experiment2` returns the rows the reference's `run_experiment2`
(cli.py:230-256) returns — one dict per fraction with the mean / standard
deviation of ARI and Jaccard over `reps` balanced subsamples — with every
one of the fractions x reps PIC runs done in ONE batched launch
(`gpu.cluster_batch`, csrc/batch.cu) instead of one run after another.
Subsample r of a fraction uses seed + 7919 r for both the sampler and the
k-means, as the reference does (cli.py:240-246).
"""

from __future__ import annotations

import math

from .datasets import subsample_balanced
from .errors import MissingLabels
from .params import KernelConfig
from .validation import adjusted_rand_index, contingency, jaccard_index

# cli.py:40 — 0.01% .. 0.09% and 0.1% .. 0.9%
DEFAULT_FRACTIONS = [i * 0.0001 for i in range(1, 10)] + [i * 0.001 for i in range(1, 10)]


def subsamples(d, fraction_list, reps, seed=0):
    """(fraction, rep seed, subsample) of the sweep, in the reference's order."""
    if d.labels is None:
        raise MissingLabels()
    out = []
    for fraction in fraction_list:
        for rep in range(reps):
            rep_seed = seed + 7919 * rep
            out.append((fraction, rep_seed, subsample_balanced(d, fraction, rep_seed)))
    return out


def _mean_std(xs):
    m = sum(xs) / len(xs)
    return m, math.sqrt(sum((x - m) ** 2 for x in xs) / len(xs))


def run_experiment2(d, kind, params, fraction_list=None, reps=10, backend="gpu",
                    config: KernelConfig | None = None, seed: int = 0) -> list[dict]:
    """Subsample, cluster (batched on the GPU) and score each fraction."""
    from . import gpu
    from .errors import InvalidSpec

    if backend != "gpu":
        raise InvalidSpec(f"unknown backend {backend!r}: this build provides only 'gpu'")
    fraction_list = DEFAULT_FRACTIONS if fraction_list is None else list(fraction_list)
    runs = subsamples(d, fraction_list, reps, seed)
    results = gpu.cluster_batch([s for _, _, s in runs], kind, params,
                                [rs for _, rs, _ in runs], config)
    rows = []
    for i, fraction in enumerate(fraction_list):
        aris, jacs = [], []
        for r in range(reps):
            _, _, sub = runs[i * reps + r]
            table = contingency(sub.labels, results[i * reps + r][0])
            aris.append(adjusted_rand_index(table))
            jacs.append(jaccard_index(table))
        am, asd = _mean_std(aris)
        jm, jsd = _mean_std(jacs)
        rows.append({"fraction": fraction, "ari_mean": am, "ari_std": asd,
                     "jaccard_mean": jm, "jaccard_std": jsd})
    return rows
