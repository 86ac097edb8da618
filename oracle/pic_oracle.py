"""CPU oracle for the GPIC hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `picluster` package's
Gaussian-RBF PIC pipeline (affinity -> degree -> D^-1 -> power iteration ->
1-D k-means). It is the checker the parity tests, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` legs compare against.
The product path (`paper_1604_02700_b200`) never imports it.

Pinning: every function here is validated against golden vectors produced by
running the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`,
checked by `tests/test_oracle_golden.py`). Parity is therefore pinned to the
reference, not to this restatement.

All arithmetic is float64 like the reference. Each function cites the
reference file:line it restates (paths relative to
`/root/reference/pkg/src/picluster/`).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


class OracleError(ValueError):
    """Raised where the reference raises one of its typed errors.

    ``kind`` names the reference exception class (errors.py), ``index`` the
    first offending position where the reference carries one.
    """

    def __init__(self, kind: str, index=None, detail: str = ""):
        self.kind = kind
        self.index = index
        super().__init__(f"{kind}({index}) {detail}".strip())


# --------------------------------------------------------------------------
# Affinity (affinity.py:74-127)
# --------------------------------------------------------------------------

def rbf_rows(points: np.ndarray, lo: int, hi: int, sigma: float) -> np.ndarray:
    """Rows [lo, hi) of A with A_ij = exp(-|x_i - x_j|^2 / (2 sigma^2)), A_ii = 0.

    Restates affinity.py:96-103: the squared distance is accumulated one
    feature at a time (same operation order as the reference, so values are
    bitwise identical to it), then scaled by -1/(2 sigma^2) and exponentiated.
    """
    x = np.asarray(points, dtype=np.float64)
    n, m = x.shape
    acc = np.zeros((hi - lo, n))
    for f in range(m):
        col = x[:, f]
        step = col[lo:hi, None] - col[None, :]
        acc += step * step
    out = np.exp(acc * (-1.0 / (2.0 * sigma * sigma)))
    rows = np.arange(lo, hi)
    out[rows - lo, rows] = 0.0
    return out


def cosine_rows(points: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Rows [lo, hi) of A_ij = max(0, x_i.x_j / (|x_i||x_j|)), A_ii = 0.

    Restates affinity.py:41-53 (norms accumulated feature by feature,
    ZeroVector(first i) for a zero row) and :88-95,102-103.
    """
    x = np.asarray(points, dtype=np.float64)
    n, m = x.shape
    sq = np.zeros(n)
    for f in range(m):
        sq += x[:, f] * x[:, f]
    zero = np.flatnonzero(sq == 0.0)
    if zero.size:
        raise OracleError("ZeroVector", int(zero[0]))
    norms = np.sqrt(sq)
    dots = np.zeros((hi - lo, n))
    for f in range(m):
        dots += x[lo:hi, f, None] * x[None, :, f]
    out = dots / (norms[lo:hi, None] * norms[None, :])
    np.maximum(out, 0.0, out=out)
    rows = np.arange(lo, hi)
    out[rows - lo, rows] = 0.0
    return out


def affinity(points: np.ndarray, sigma: float | None) -> np.ndarray:
    """Full A (affinity.py:107-110 build_affinity): RBF, or cosine when sigma is None."""
    x = np.asarray(points, dtype=np.float64)
    bad = ~np.isfinite(x)
    if bad.any():  # data.py:69-72 NonFiniteEntry(row, col) of the first bad entry
        r, c = np.argwhere(bad)[0]
        raise OracleError("NonFiniteEntry", (int(r), int(c)))
    if sigma is None:
        return cosine_rows(x, 0, x.shape[0])
    return rbf_rows(x, 0, x.shape[0], sigma)


def degree(a: np.ndarray) -> np.ndarray:
    """Row sums; ZeroDegree(first i) when d_i <= 0 (affinity.py:113-119)."""
    d = a.sum(axis=1)
    nz = np.flatnonzero(d <= 0.0)
    if nz.size:
        raise OracleError("ZeroDegree", int(nz[0]))
    return d


def normalize(a: np.ndarray, d: np.ndarray) -> np.ndarray:
    """W = A / d[:, None] (affinity.py:122-127)."""
    nz = np.flatnonzero(d <= 0.0)
    if nz.size:
        raise OracleError("ZeroDegree", int(nz[0]))
    return a / d[:, None]


# --------------------------------------------------------------------------
# Reductions and the power iteration (serial.py:77-128, parallel.py:161-233)
# --------------------------------------------------------------------------

def tree_sum(v: np.ndarray) -> float:
    """Fixed-shape sum: zero-pad to 2^ceil(log2 n), halve the stride each round.

    Restates parallel.py:161-178 (k_reduce). Raises EmptyVector for n == 0.
    """
    v = np.asarray(v, dtype=np.float64).ravel()
    if v.size == 0:
        raise OracleError("EmptyVector")
    width = 1
    while width < v.size:
        width <<= 1
    buf = np.zeros(width)
    buf[: v.size] = v
    half = width // 2
    while half:
        buf[:half] = buf[:half] + buf[half: 2 * half]
        half //= 2
    return float(buf[0])


def start_vector(deg: np.ndarray, choice="degree") -> np.ndarray:
    """v0 (serial.py:77-101): "degree" -> d / sum(d), "uniform" -> 1/n, or explicit."""
    deg = np.asarray(deg, dtype=np.float64)
    n = deg.size
    if isinstance(choice, str):
        if choice == "degree":
            nz = np.flatnonzero(deg <= 0.0)
            if nz.size:
                raise OracleError("ZeroDegree", int(nz[0]))
            return deg / deg.sum()
        if choice == "uniform":
            return np.full(n, 1.0 / n)
        raise OracleError("InvalidSpec", detail=f"v0 kind {choice!r}")
    v0 = np.array(choice, dtype=np.float64)
    if v0.shape != (n,) or v0.min() < 0.0 or abs(v0.sum() - 1.0) > 1e-12:
        raise OracleError("InvalidSpec", detail="explicit v0")
    return v0


def resolved_epsilon(epsilon, n: int) -> float:
    """serial.py:46-47: a user epsilon is used as given; None -> 1e-5 / n."""
    return float(epsilon) if epsilon is not None else 1e-5 / n


ROW_SUM_TOL = 1e-9  # serial.py:20


def row_stochastic_violation(w: np.ndarray):
    """check_row_stochastic (serial.py:63-74) as a verdict, not an exception.

    Returns None when every row sums to 1 within 1e-9 and entries lie in
    [0, 1] (1e-12 slack); else ("row", i, sum_i) for the worst row, or
    ("range", None, None).
    """
    w = np.asarray(w, dtype=np.float64)
    sums = w.sum(axis=1)
    if np.max(np.abs(sums - 1.0)) > ROW_SUM_TOL:
        bad = int(np.argmax(np.abs(sums - 1.0)))
        return ("row", bad, float(sums[bad]))
    if w.min() < -1e-12 or w.max() > 1.0 + 1e-12:
        return ("range", None, None)
    return None


def power_iteration(w: np.ndarray, v0: np.ndarray, eps: float, max_iterations: int):
    """v <- W v / |W v|_1 with the acceleration stop (serial.py:104-128).

    delta_t = max|v_t - v_(t-1)|; stop after iteration t >= 2 when
    |delta_t - delta_(t-1)| <= eps. Returns (v, deltas, converged).
    """
    v = np.asarray(v0, dtype=np.float64)
    deltas = []
    for _ in range(max_iterations):
        y = w @ v
        nxt = y / np.abs(y).sum()
        deltas.append(float(np.abs(nxt - v).max()))
        v = nxt
        if len(deltas) > 1 and abs(deltas[-1] - deltas[-2]) <= eps:
            return v, np.array(deltas), True
    return v, np.array(deltas), False


# --------------------------------------------------------------------------
# 1-D k-means (kmeans.py:39-196)
# --------------------------------------------------------------------------

POLISH_LIMIT = 4096  # kmeans.py:22


def kmeanspp_seeds(values: np.ndarray, k: int, rng) -> np.ndarray:
    """D^2 seeding (kmeans.py:39-55). rng is np.random.default_rng(seed)."""
    n = values.size
    c = np.empty(k)
    c[0] = values[int(rng.integers(n))]
    dist2 = (values - c[0]) ** 2
    for j in range(1, k):
        mass = dist2.sum()
        if mass <= 0.0:
            c[j:] = c[0]
            break
        r = rng.random() * mass
        pick = int(np.searchsorted(np.cumsum(dist2), r, side="right"))
        c[j] = values[min(pick, n - 1)]
        dist2 = np.minimum(dist2, (values - c[j]) ** 2)
    return c


def nearest(values: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """Index of the closest centre, lowest index on ties (kmeans.py:58-60)."""
    return np.argmin(np.abs(values[:, None] - centers[None, :]), axis=1)


def wcss(values: np.ndarray, labels: np.ndarray, k: int) -> float:
    """Within-cluster sum of squares (kmeans.py:63-69)."""
    s = 0.0
    for j in range(k):
        part = values[labels == j]
        if part.size:
            s += float(((part - part.mean()) ** 2).sum())
    return s


def lloyd(values: np.ndarray, k: int, seed: int, max_rounds: int = 100, tol: float = 1e-12):
    """Seeded Lloyd iterations with empty-cluster reseeding (kmeans.py:72-94)."""
    rng = np.random.default_rng(seed)
    centers = kmeanspp_seeds(values, k, rng)
    labels = nearest(values, centers)
    for _ in range(max_rounds):
        for j in range(k):
            if not (labels == j).any():
                far = int(np.argmax(np.abs(values - centers[labels])))
                centers[j] = values[far]
                labels = nearest(values, centers)
        shift = 0.0
        for j in range(k):
            part = values[labels == j]
            if part.size:
                mu = float(part.mean())
                shift = max(shift, abs(mu - centers[j]))
                centers[j] = mu
        labels = nearest(values, centers)
        if shift < tol:
            break
    return labels


def optimal_contiguous(values: np.ndarray, k: int) -> np.ndarray:
    """Exact 1-D k-means by DP over sorted order, earliest split on ties (kmeans.py:97-130)."""
    order = np.argsort(values, kind="stable")
    xs = values[order]
    n = xs.size
    s1 = np.concatenate([[0.0], np.cumsum(xs)])
    s2 = np.concatenate([[0.0], np.cumsum(xs * xs)])
    cost = np.full((k + 1, n + 1), np.inf)
    back = np.zeros((k + 1, n + 1), dtype=np.int64)
    cost[0, 0] = 0.0
    for q in range(1, k + 1):
        for j in range(q, n + 1):
            i = np.arange(q - 1, j)
            seg = s1[j] - s1[i]
            c = cost[q - 1, q - 1: j] + (s2[j] - s2[i]) - seg * seg / (j - i)
            b = int(np.argmin(c))
            cost[q, j] = c[b]
            back[q, j] = q - 1 + b
    lab_sorted = np.zeros(n, dtype=np.int64)
    j = n
    for q in range(k, 0, -1):
        i = int(back[q, j])
        lab_sorted[i:j] = q - 1
        j = i
    out = np.empty(n, dtype=np.int64)
    out[order] = lab_sorted
    return out


def is_contiguous(values: np.ndarray, labels: np.ndarray) -> bool:
    """Every label occupies one run of the stable sorted order (kmeans.py:149-160)."""
    seq = labels[np.argsort(values, kind="stable")]
    if seq.size == 0:
        return True
    starts = np.concatenate([[True], seq[1:] != seq[:-1]])
    run_labels = seq[starts]
    return np.unique(run_labels).size == run_labels.size


def split_largest_gaps(values: np.ndarray, k: int) -> np.ndarray:
    """Cut sorted values at the k-1 widest gaps (kmeans.py:133-146)."""
    order = np.argsort(values, kind="stable")
    xs = values[order]
    n = xs.size
    lab_sorted = np.zeros(n, dtype=np.int64)
    if n > 1 and k > 1:
        gaps = np.diff(xs)
        cuts = np.sort(np.argsort(gaps, kind="stable")[::-1][: k - 1])
        for c in cuts:
            lab_sorted[c + 1:] += 1
    out = np.empty(n, dtype=np.int64)
    out[order] = lab_sorted
    return out


def canonical(values: np.ndarray, labels: np.ndarray, k: int) -> np.ndarray:
    """Renumber clusters by ascending centroid; empty ids compact (kmeans.py:163-175)."""
    cent = np.full(k, np.inf)
    for j in range(k):
        part = values[labels == j]
        if part.size:
            cent[j] = part.mean()
    used = np.flatnonzero(np.isfinite(cent))
    rank = used[np.argsort(cent[used], kind="stable")]
    remap = np.zeros(k, dtype=np.int64)
    remap[rank] = np.arange(rank.size)
    return remap[labels]


def kmeans_1d(values, k: int, seed: int = 0, max_rounds: int = 100, tol: float = 1e-12):
    """Full kmeans_1d pipeline (kmeans.py:178-196)."""
    values = np.asarray(values, dtype=np.float64).ravel()
    n = values.size
    if k > n:
        raise OracleError("KTooLarge", detail=f"k={k} n={n}")
    labels = lloyd(values, k, seed, max_rounds, tol)
    if n <= POLISH_LIMIT:
        exact = optimal_contiguous(values, k)
        if wcss(values, exact, k) < wcss(values, labels, k):
            labels = exact
    if not is_contiguous(values, labels):
        labels = split_largest_gaps(values, k)
    return canonical(values, labels, k)


# --------------------------------------------------------------------------
# End to end (serial.py:131-150 / parallel.py:386-405)
# --------------------------------------------------------------------------

def pic_cluster(points, sigma: float, k: int, epsilon=None, max_iterations: int = 50,
                seed: int = 0, v0="degree"):
    """Returns (labels int64[n], v float64[n], deltas float64[T], converged)."""
    a = affinity(points, sigma)
    d = degree(a)
    w = normalize(a, d)
    del a
    v_init = start_vector(d, v0)
    eps = resolved_epsilon(epsilon, w.shape[0])
    v, deltas, conv = power_iteration(w, v_init, eps, max_iterations)
    labels = kmeans_1d(v, k, seed)
    return labels, v, deltas, conv


# --------------------------------------------------------------------------
# Threaded port of the reference's parallel backend, used as the CPU
# baseline (parallel.py:90-128, 196-207). Work is split into <= p contiguous
# row ranges of ceil(n/p) rows, executed on a thread pool; numpy releases
# the GIL inside the array operations exactly as in the reference.
# --------------------------------------------------------------------------

def row_ranges(n: int, p: int):
    """plan_rows (parallel.py:90-98)."""
    step = -(-n // p)
    return [(lo, min(lo + step, n)) for lo in range(0, n, step)]


def _fan_out(fn, ranges, p):
    if len(ranges) == 1:
        fn(*ranges[0])
        return
    with ThreadPoolExecutor(max_workers=min(p, len(ranges))) as ex:
        for fut in [ex.submit(fn, lo, hi) for lo, hi in ranges]:
            fut.result()


def chunk_rows(n: int, budget: int = 256 * 1024 * 1024) -> int:
    """KernelConfig.resolved_chunk_rows default (parallel.py:68-77)."""
    return max(1, min(n, budget // (8 * n)))


def affinity_rows_threaded(points, lo: int, hi: int, sigma: float, p: int | None = None):
    """Rows [lo, hi) of A built like k_affinity (parallel.py:113-128)."""
    p = p or os.cpu_count() or 1
    x = np.asarray(points, dtype=np.float64)
    n = x.shape[0]
    chunk = chunk_rows(n)
    out = np.empty((hi - lo, n))

    def work(a, b):
        for s in range(a, b, chunk):
            e = min(s + chunk, b)
            out[s - lo: e - lo] = rbf_rows(x, s, e, sigma)

    _fan_out(work, [(a + lo, b + lo) for a, b in row_ranges(hi - lo, p)], p)
    return out


def matvec_threaded(w: np.ndarray, v: np.ndarray, p: int | None = None) -> np.ndarray:
    """k_multiply (parallel.py:196-207): einsum ij,j->i per row range."""
    p = p or os.cpu_count() or 1
    out = np.empty(w.shape[0])

    def work(a, b):
        out[a:b] = np.einsum("ij,j->i", w[a:b], v)

    _fan_out(work, row_ranges(w.shape[0], p), p)
    return out


# --------------------------------------------------------------------------
# Device App-B generator restated (csrc/generate.cu). The
# reference has no such generator (its datasets.py:147-172 is 2-D only); this
# pins the CUDA kernel's stream: Philox4x32-10 keyed by the seed, counter =
# element-pair index, Box-Muller on two 53-bit uniforms.
# --------------------------------------------------------------------------

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, seed: int) -> np.ndarray:
    """ctr: (m, 4) uint64 words < 2^32 -> (m, 4) output words."""
    c0, c1, c2, c3 = (ctr[:, j].astype(np.uint64) for j in range(4))
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return np.stack([c0, c1, c2, c3], axis=1)


def device_blobs(centers: np.ndarray, counts, seed: int, noise: float, offset: float):
    """X (n x d) and labels exactly as gpic_generate_blobs lays them out."""
    k, d = centers.shape
    counts = np.asarray(counts, dtype=np.int64)
    n = int(counts.sum())
    total = n * d
    pairs = (total + 1) // 2
    p = np.arange(pairs, dtype=np.uint64)
    ctr = np.zeros((pairs, 4), dtype=np.uint64)
    ctr[:, 0] = p & _MASK
    ctr[:, 1] = p >> np.uint64(32)
    w = philox4x32_10(ctr, seed)
    a = (w[:, 0] << np.uint64(21)) | (w[:, 1] >> np.uint64(11))
    b = (w[:, 2] << np.uint64(21)) | (w[:, 3] >> np.uint64(11))
    u1 = 1.0 - a.astype(np.float64) * 2.0 ** -53
    u2 = b.astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty(2 * pairs)
    z[0::2] = r * np.cos(2.0 * np.pi * u2)
    z[1::2] = r * np.sin(2.0 * np.pi * u2)
    labels = np.repeat(np.arange(k, dtype=np.int64), counts)
    x = centers[labels] + noise * z[:total].reshape(n, d) + offset
    return x, labels
