"""fp64 matrix-free CPU oracle (ctypes over oracle/pic_mf.c) — TEST INFRASTRUCTURE ONLY.

The reference stores A and W as dense fp64 n x n matrices
(`/root/reference/pkg/src/picluster/affinity.py:107-127`), which does not fit
any host at the benchmark configs (80 GB at n = 100k, 8 TB at n = 1M). This
module runs the same pipeline with every affinity row recomputed on the fly
in fp64 by `pic_mf.c` (its header lists the reference lines it restates), and
the O(n) steps in numpy exactly as `serial.py:77-128` writes them.

Used by tests/, `tests/golden/make_config_fixtures.py` and bench.py's CPU
legs, never by the product path. Pinned against the reference itself on
configs 1-2 (`tests/test_oracle_mf.py` against `tests/golden/*.npz`, which
`tests/golden/make_golden.py` made by running the reference).
"""

from __future__ import annotations

import ctypes
import pathlib
import subprocess

import numpy as np

from . import pic_oracle as po

_HERE = pathlib.Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libpicmf.so"
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def lib():
    """Load (building on first use when the source tree allows it) libpicmf.so."""
    global _lib
    if _lib is None:
        if not _SO.exists():
            subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
        L = ctypes.CDLL(str(_SO))
        sig = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
               ctypes.c_int64, ctypes.c_int64]
        L.picmf_degree.argtypes = sig + [ctypes.c_void_p]
        L.picmf_matvec.argtypes = sig + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.picmf_rows.argtypes = sig + [ctypes.c_void_p]
        for f in (L.picmf_degree, L.picmf_matvec, L.picmf_rows):
            f.restype = None
        L.picmf_exp.argtypes = [ctypes.c_double]
        L.picmf_exp.restype = ctypes.c_double
        L.picmf_set_skip.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.picmf_set_skip.restype = None
        L.picmf_block.restype = ctypes.c_int64
        _lib = L
    return _lib


def _x(points):
    x = np.ascontiguousarray(points, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError("points must be (n, m)")
    return x


def _sig(sigma):
    # sigma None selects the cosine kind (affinity.py:22-24), encoded as 0
    return 0.0 if sigma is None else float(sigma)


def rows(points, lo: int, hi: int, sigma) -> np.ndarray:
    """Rows [lo, hi) of A (affinity.py:74-103), fp64."""
    x = _x(points)
    out = np.empty((hi - lo, x.shape[0]))
    lib().picmf_rows(x.ctypes.data, x.shape[0], x.shape[1], _sig(sigma), lo, hi, out.ctypes.data)
    return out


def degree(points, sigma, lo: int = 0, hi: int | None = None) -> np.ndarray:
    """deg_i = sum_j a_ij for rows [lo, hi) (affinity.py:113-115), no ZeroDegree check."""
    x = _x(points)
    hi = x.shape[0] if hi is None else hi
    out = np.empty(hi - lo)
    lib().picmf_degree(x.ctypes.data, x.shape[0], x.shape[1], _sig(sigma), lo, hi, out.ctypes.data)
    return out


def matvec(points, sigma, deg, v, lo: int = 0, hi: int | None = None) -> np.ndarray:
    """(W v)[lo:hi] with W = A / deg[:, None] (affinity.py:126, serial.py:121)."""
    x = _x(points)
    hi = x.shape[0] if hi is None else hi
    deg = np.ascontiguousarray(deg, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty(hi - lo)
    lib().picmf_matvec(x.ctypes.data, x.shape[0], x.shape[1], _sig(sigma), lo, hi,
                       deg.ctypes.data, v.ctypes.data, out.ctypes.data)
    return out


class negligible_blocks:
    """Context manager: skip BLK x BLK block pairs (pic_mf.c picmf_set_skip)
    whose every entry is proved below e^-``exponent`` (RBF only).

    The proof is the projection on the line joining the two block centroids,
    in fp64: for i in S, j in T, |x_i - x_j| >= (min_T u.x_j - max_S u.x_i) /
    |u|, u = c_T - c_S, less a generous rounding allowance. Skipping leaves
    every fp64 row sum bit-identical (see pic_mf.c), which
    tests/test_oracle_mf.py checks against the unskipped pass.
    """

    def __init__(self, points, sigma, exponent: float = 70.0):
        x = _x(points)
        n = x.shape[0]
        B = int(lib().picmf_block())
        nb = -(-n // B)
        cent = np.stack([x[S * B:(S + 1) * B].mean(axis=0) for S in range(nb)])
        M = np.empty((nb, nb))  # M[S][T] = max_{i in S} x_i.(c_T - c_S)
        for S in range(nb):
            P = x[S * B:(S + 1) * B] @ cent.T
            M[S] = (P - P[:, S:S + 1]).max(axis=0)
        gap = -(M + M.T)
        u = np.sqrt(((cent[:, None, :] - cent[None, :, :]) ** 2).sum(-1))
        xm = float(np.sqrt((x * x).sum(1)).max())
        cm = float(np.sqrt((cent * cent).sum(1)).max())
        err = 8.0 * (x.shape[1] + 2) * 2.0 ** -53 * xm * cm
        with np.errstate(divide="ignore", invalid="ignore"):
            lb = (gap - err) / u * (1 - 1e-9)
        skip = (u > 0) & (lb > 0) & (lb * lb / (2.0 * sigma * sigma) >= exponent)
        np.fill_diagonal(skip, False)
        self.skip = np.ascontiguousarray(skip, dtype=np.uint8)
        self.nb = nb
        self.fraction = float(skip.mean())

    def __enter__(self):
        lib().picmf_set_skip(self.skip.ctypes.data, self.nb)
        return self

    def __exit__(self, *exc):
        lib().picmf_set_skip(None, 0)


def power_trajectory(points, sigma, epsilon=None, max_iterations: int = 50, v0="degree",
                     keep=(), log=None):
    """The reference's serial pipeline up to the embedding, matrix-free.

    Restates serial.py:77-128 (initial_vector, then v <- Wv/|Wv|_1 with
    delta = max|v' - v| and the stop |delta_t - delta_(t-1)| <= eps for t >= 2),
    recording v after the iterations listed in ``keep`` — a run with the
    native rule passes through exactly the states a forced-T run
    (epsilon=5e-324, max_iterations=T) ends in.

    Returns dict(v, deltas, converged, deg, kept={T: v_T}).
    """
    x = _x(points)
    n = x.shape[0]
    deg = degree(x, sigma)
    bad = np.flatnonzero(deg <= 0.0)
    if bad.size:
        raise po.OracleError("ZeroDegree", int(bad[0]))
    v = po.start_vector(deg, v0)
    eps = po.resolved_epsilon(epsilon, n)
    deltas, kept, converged = [], {}, False
    for t in range(1, max_iterations + 1):
        wv = matvec(x, sigma, deg, v)
        nxt = wv / np.abs(wv).sum()
        deltas.append(float(np.abs(nxt - v).max()))
        v = nxt
        if log:
            log(f"iteration {t}: delta {deltas[-1]:.6e}")
        if t in keep:
            kept[t] = v.copy()
        if len(deltas) >= 2 and abs(deltas[-1] - deltas[-2]) <= eps:
            converged = True
            break
    return dict(v=v, deltas=np.array(deltas), converged=converged, deg=deg, kept=kept)


def pic_cluster(points, sigma, k: int, epsilon=None, max_iterations: int = 50, seed: int = 0,
                v0="degree"):
    """(labels, v, deltas, converged) like pic_oracle.pic_cluster, matrix-free."""
    tr = power_trajectory(points, sigma, epsilon, max_iterations, v0)
    labels = po.kmeans_1d(tr["v"], k, seed)
    return labels, tr["v"], tr["deltas"], tr["converged"]
