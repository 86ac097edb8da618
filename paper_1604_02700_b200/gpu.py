"""The B200 backend: the reference's backend-module protocol on libgpic.

Same stage names and argument meanings as `picluster/parallel.py`
(k_affinity :113, k_rowsum :131, k_normalize :146, k_reduce :161, k_norm :181,
k_multiply :196, initial_embedding :210, iterate :217, cluster :236) plus
`kmeans_1d` (kmeans.py:178), so `report.run_timed`-style drivers and the
reference's per-kernel tests read the same against this module.

Data stays on the device between stages: `k_affinity` returns a
`DeviceAffinity` (fp32 A row block + fused degrees), `k_normalize` returns a
`NormalizedAffinity` view (W = D^-1 A is never materialised; the GEMV applies
1/deg), vectors are CUDA tensors. Functions also accept numpy inputs and then
return numpy outputs (uploaded in fp32 / fp64 as the engine computes), which
is how the reference-style unit tests drive them.

Tensors are PyTorch CUDA tensors (memory + streams only); every computation
is a libgpic kernel. No CPU fallback: without a CUDA device or libgpic.so
every entry point raises.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .data import DataSet, check_labels, check_shape
from .errors import (
    DeviceError,
    DimensionMismatch,
    EmptyVector,
    InvalidSpec,
    KTooLarge,
    NonPositiveTau,
    ZeroDegree,
)
from .params import (
    Cosine,
    GaussianRbf,
    KernelConfig,
    KMeansParams,
    PicParams,
    PicTrace,
)

KMEANS_MAX_K = 4096      # single problems (k > 64: the sorted-domain variant, kmeans_big.cu)
BATCH_MAX_K = 64         # the batched Experiment-II engine


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("the GPIC backend needs a CUDA device (B200 / sm_100a); none is visible")
    return torch


def _device(config: KernelConfig | None):
    torch = _torch()
    if config is not None and config.device is not None:
        return torch.device("cuda", config.device)
    return torch.device("cuda", torch.cuda.current_device())


def _stream(dev):
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _check_kind(kind) -> tuple[int, float]:
    """(GPIC_KIND_*, sigma) of a similarity kind (affinity.py:22-35)."""
    if isinstance(kind, Cosine):
        return _lib.KIND_COSINE, 1.0
    if not isinstance(kind, GaussianRbf):
        raise InvalidSpec(f"unknown similarity kind {kind!r}")
    return _lib.KIND_RBF, float(kind.sigma)


def _read_ctl(ctl_t, dev) -> _lib.Ctl:
    h = _lib.Ctl()
    rc = _lib.lib().gpic_ctl_read(_ptr(ctl_t), C.byref(h), _stream(dev))
    _lib.check(rc)
    return h


def _raise_ctl(h: _lib.Ctl, d: int = 1) -> None:
    if h.status != _lib.GPIC_OK:
        _lib.raise_for(h.status, h, d)


def _new_ctl(dev, eps: float = 0.0, max_iter: int = 1):
    torch = _torch()
    ctl = torch.empty(256, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().gpic_ctl_init(_ptr(ctl), eps, max_iter, _stream(dev)))
    return ctl


def kmeans_draws(n: int, k: int, seed: int):
    """The PCG64 numbers kmeans.py draws: integers(n) then k-1 x random() (kmeans.py:43,51,73)."""
    rng = np.random.default_rng(seed)
    first = int(rng.integers(n))
    u = np.ascontiguousarray(rng.random(max(k - 1, 1)), dtype=np.float64)
    return first, u


# ------------------------------------------------------------ containers
@dataclass
class DeviceAffinity:
    """Rows [row_lo, row_hi) of A (fp32, row pitch `lda`) with fused degrees."""

    a: object          # torch.float32 [rows, lda]
    deg: object        # torch.float64 [rows]
    n: int
    lda: int
    row_lo: int
    row_hi: int
    ctl: object        # torch.uint8[256] device control block
    d: int = 1

    @property
    def shape(self):
        return (self.row_hi - self.row_lo, self.n)

    def numpy(self) -> np.ndarray:
        return self.a[:, : self.n].double().cpu().numpy()


@dataclass
class NormalizedAffinity:
    """W = D^-1 A without the second n^2 pass (k_normalize, folded into the GEMV)."""

    a: object          # torch.float32 [rows, lda]
    deg: object        # torch.float64 [rows] or None (already stochastic)
    n: int
    lda: int

    @property
    def shape(self):
        return (self.a.shape[0], self.n)

    def numpy(self) -> np.ndarray:
        w = self.a[:, : self.n].double()
        if self.deg is not None:
            w = w / self.deg[:, None]
        return w.cpu().numpy()


def _as_device_matrix(w, dev):
    """numpy (rows, n) -> fp32 device matrix with a 32-float pitch."""
    torch = _torch()
    w = np.asarray(w, dtype=np.float64)
    if w.ndim != 2:
        raise InvalidSpec(f"expected a matrix, got shape {w.shape}")
    rows, n = w.shape
    lda = int(_lib.lib().gpic_affinity_pitch(n))
    t = torch.zeros((rows, lda), dtype=torch.float32, device=dev)
    t[:, :n] = torch.from_numpy(w.astype(np.float32))
    return t, rows, n, lda


def _vec64(v, dev):
    torch = _torch()
    if isinstance(v, np.ndarray) or not hasattr(v, "is_cuda"):
        arr = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
        return torch.from_numpy(arr).to(dev), True
    return v.to(device=dev, dtype=torch.float64).contiguous().reshape(-1), False


def _vec32_padded(v64, n, dev):
    torch = _torch()
    lda = int(_lib.lib().gpic_affinity_pitch(n))
    out = torch.zeros(lda, dtype=torch.float32, device=dev)
    out[:n] = v64.to(torch.float32)
    return out


# ----------------------------------------------------------------- stages
def k_affinity(d: DataSet, kind, config: KernelConfig | None = None,
               rows: tuple[int, int] | None = None) -> DeviceAffinity:
    """Affinity row block on the device (parallel.py:113-128, affinity.py:74-110).

    Runs the fp64 centring/validation prepass, the selected Gram engine with
    the fused exp/diagonal/row-sum epilogue, and the fixed-order degree
    combine. Raises NonFiniteEntry like validate_dataset (data.py:69-72).
    """
    config = config or KernelConfig()
    code, sigma = _check_kind(kind)
    check_shape(d)
    check_labels(d)
    dev = _device(config)
    n = d.points.shape[0]
    lo, hi = rows if rows is not None else (0, n)
    prep = prepare_points(d, dev, code)
    return affinity_rows(prep, lo, hi, sigma, config.affinity_impl)


@dataclass
class PreparedPoints:
    """fp32 operands of the Gram engines (gpic_prepare_points): centred rows
    (RBF) or unit rows (cosine), TF32 hi + fp32 lo split."""

    xhi: object
    xlo: object
    sqn: object
    n: int
    d: int
    device: object
    kind: int = _lib.KIND_RBF
    x: object = None  # the fp64 points on the device (isolated-row fix, lowdeg.cu)
    spread2: float = 0.0  # R^2 = max_i |x_i - mean|^2 (RBF): engine routing
    work: object = None  # gpic_prepare_points' column sums + mean (tile pruning)

    def engine(self, sigma: float, engine: str, storage: int) -> str:
        """The engine gpic_cluster would run (gpic_engine_for): SIMT difference
        form for RBF at d <= 8 or a spread too large for the tensor Gram."""
        impl = _lib.AFFINITY_TC if engine == "tc" else _lib.AFFINITY_SIMT
        got = _lib.lib().gpic_engine_for(self.kind, self.d, float(sigma), float(self.spread2), impl,
                                         storage)
        return "tc" if got == _lib.AFFINITY_TC else "simt"


def prepare_points(d, dev, kind: int = _lib.KIND_RBF) -> PreparedPoints:
    """Upload X (fp64), scan for non-finite entries, centre (RBF) or
    normalise (cosine, ZeroVector for a zero row), cast and split.

    ``d`` is a DataSet (host points, uploaded here) or an (n, m) float64
    CUDA tensor already resident on ``dev``.
    """
    torch = _torch()
    L = _lib.lib()
    if isinstance(d, DataSet):
        x = torch.from_numpy(d.points).to(dev, non_blocking=True)
    else:
        x = d.to(device=dev, dtype=torch.float64).contiguous()
    n, m = x.shape
    st = _stream(dev)
    dp = int(L.gpic_feature_pitch(m))
    npad = int(L.gpic_row_pad(n))
    xhi = torch.empty(int(L.gpic_operand_floats(n, m)), dtype=torch.float32, device=dev)
    xlo = torch.empty((npad, dp), dtype=torch.float32, device=dev)
    sqn = torch.empty(npad, dtype=torch.float32, device=dev)
    ctl = _new_ctl(dev)
    ncol = ((n + 255) // 256) * m
    work = torch.empty(ncol + m + 2, dtype=torch.float64, device=dev)
    _lib.check(L.gpic_prepare_points(_ptr(x), n, m, kind, _ptr(xhi), _ptr(xlo), _ptr(sqn),
                                     _ptr(work), _ptr(ctl), st))
    _raise_ctl(_read_ctl(ctl, dev), m)
    spread2 = float(work[ncol + m + 1].item()) if kind == _lib.KIND_RBF else 0.0
    return PreparedPoints(xhi=xhi, xlo=xlo, sqn=sqn, n=n, d=m, device=dev, kind=kind, x=x,
                          spread2=spread2, work=work)


def affinity_rows(prep: PreparedPoints, lo: int, hi: int, sigma: float, engine: str = "tc"):
    """Rows [lo, hi) of A plus their degrees (fused epilogue + fixed-order combine)."""
    torch = _torch()
    L = _lib.lib()
    dev, n, m = prep.device, prep.n, prep.d
    lda = int(L.gpic_affinity_pitch(n))
    nrows = hi - lo
    a = torch.empty((nrows, lda), dtype=torch.float32, device=dev)
    deg = torch.empty(nrows, dtype=torch.float64, device=dev)
    rows_pad = -(-nrows // 128) * 128
    rowpart = torch.empty(((n + 127) // 128) * rows_pad, dtype=torch.float32, device=dev)
    ctl = _new_ctl(dev)
    engine = prep.engine(sigma, engine, _lib.STORAGE_DENSE)
    impl = _lib.AFFINITY_TC if engine == "tc" else _lib.AFFINITY_SIMT
    if prep.kind == _lib.KIND_COSINE:
        rc = L.gpic_affinity_cosine(_ptr(prep.xhi), _ptr(prep.xlo), _ptr(prep.sqn), n, m, lo, hi,
                                    impl, _ptr(a), lda, _ptr(deg), _ptr(rowpart), _ptr(ctl),
                                    _stream(dev))
    else:
        rc = L.gpic_affinity_rbf(_ptr(prep.xhi), _ptr(prep.xlo), _ptr(prep.sqn), n, m, lo, hi,
                                 sigma, impl, _ptr(a), lda, _ptr(deg), _ptr(rowpart), _ptr(ctl),
                                 _stream(dev))
    _lib.check(rc)
    return DeviceAffinity(a=a, deg=deg, n=n, lda=lda, row_lo=lo, row_hi=hi, ctl=ctl, d=m)


def k_rowsum(a, config: KernelConfig | None = None):
    """Row sums = degrees (parallel.py:131-143). ZeroDegree(first row) if any <= 0.

    A device block returns its fused degrees; a host fp64 matrix is summed in
    fp64 on the device (gpic_row_stats), as the reference sums it.
    """
    torch = _torch()
    if isinstance(a, DeviceAffinity):
        h = _read_ctl(a.ctl, a.a.device)
        _raise_ctl(h, a.d)
        return a.deg
    wn = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if wn.ndim != 2 or wn.size == 0:
        raise InvalidSpec(f"expected a non-empty matrix, got shape {wn.shape}")
    rows, n = wn.shape
    dev = _device(config)
    t = torch.from_numpy(wn).to(dev)
    stats = torch.empty((3, rows), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().gpic_row_stats(_ptr(t), rows, n, n, _ptr(stats[0]), _ptr(stats[1]),
                                         _ptr(stats[2]), _stream(dev)))
    res = stats[0].cpu().numpy()
    bad = np.flatnonzero(res <= 0.0)
    if bad.size:
        raise ZeroDegree(int(bad[0]))
    return res


def k_normalize(a, deg, config: KernelConfig | None = None):
    """W = A / deg (parallel.py:146-158), folded: returns a lazy NormalizedAffinity."""
    torch = _torch()
    if isinstance(a, DeviceAffinity):
        if deg is not a.deg:
            deg_t, _ = _vec64(deg, a.a.device)
        else:
            deg_t = a.deg
        return NormalizedAffinity(a=a.a, deg=deg_t, n=a.n, lda=a.lda)
    deg_np = np.asarray(deg, dtype=np.float64)
    bad = np.flatnonzero(deg_np <= 0.0)
    if bad.size:
        raise ZeroDegree(int(bad[0]))
    dev = _device(config)
    t, rows, n, lda = _as_device_matrix(a, dev)
    return NormalizedAffinity(a=t, deg=torch.from_numpy(deg_np).to(dev), n=n, lda=lda)


def k_reduce(v, config: KernelConfig | None = None) -> float:
    """Fixed-shape fp64 tree sum (parallel.py:161-178)."""
    torch = _torch()
    dev = _device(config) if not hasattr(v, "is_cuda") else v.device
    t, _ = _vec64(v, dev)
    n = t.numel()
    if n == 0:
        raise EmptyVector()
    work = torch.empty(256 + 8 * ((n + 2047) // 2048 + 1), dtype=torch.uint8, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().gpic_reduce_sum(_ptr(t), n, _ptr(out), _ptr(work), _stream(dev)))
    return float(out.item())


def k_norm(v, tau: float, config: KernelConfig | None = None):
    """v / tau (parallel.py:181-193); NonPositiveTau when tau <= 0 or NaN."""
    torch = _torch()
    if not (tau > 0.0):
        raise NonPositiveTau(tau)
    dev = _device(config) if not hasattr(v, "is_cuda") else v.device
    t, was_np = _vec64(v, dev)
    out = torch.empty_like(t)
    _lib.check(_lib.lib().gpic_scale(_ptr(t), t.numel(), float(tau), _ptr(out), None, 0,
                                     _stream(dev)))
    return out.cpu().numpy() if was_np else out


def k_multiply(w, v, config: KernelConfig | None = None):
    """W @ v (parallel.py:196-207): fp32 W / v streamed, fp64 row results."""
    torch = _torch()
    was_np = not isinstance(w, (NormalizedAffinity, DeviceAffinity))
    if was_np:
        wn = np.asarray(w)
        if wn.ndim != 2 or wn.shape[1] != np.asarray(v).reshape(-1).shape[0]:
            raise DimensionMismatch(wn.shape, np.asarray(v).shape)
        dev = _device(config)
        a, rows, n, lda = _as_device_matrix(wn, dev)
        scale = None
    else:
        a, n, lda, rows = w.a, w.n, w.lda, w.a.shape[0]
        dev = a.device
        scale = getattr(w, "deg", None) if isinstance(w, NormalizedAffinity) else None
        if isinstance(w, DeviceAffinity):
            scale = None
    v64, v_np = _vec64(v, dev)
    if v64.numel() != n:
        raise DimensionMismatch((rows, n), tuple(v64.shape))
    v32 = _vec32_padded(v64, n, dev)
    out = torch.empty(rows, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().gpic_matvec(_ptr(a), lda, rows, n, _ptr(v32), _ptr(scale), _ptr(out),
                                      _stream(dev)))
    return out.cpu().numpy() if (was_np or v_np) else out


def initial_embedding(deg, params: PicParams, config: KernelConfig | None = None):
    """Start vector (parallel.py:210-214 / serial.py:77-101)."""
    torch = _torch()
    was_np = not hasattr(deg, "is_cuda")
    dev = _device(config) if was_np else deg.device
    d64, _ = _vec64(deg, dev)
    n = d64.numel()
    choice = params.v0
    if isinstance(choice, str) and choice == "degree":
        v64 = torch.empty(n, dtype=torch.float64, device=dev)
        v32 = torch.empty(int(_lib.lib().gpic_affinity_pitch(n)), dtype=torch.float32, device=dev)
        ctl = _new_ctl(dev)
        work = torch.empty(((n + 2047) // 2048 + 2), dtype=torch.float64, device=dev)
        if was_np and np.any(np.asarray(deg) <= 0.0):
            raise ZeroDegree(int(np.flatnonzero(np.asarray(deg) <= 0.0)[0]))
        _lib.check(_lib.lib().gpic_initial_vector(_ptr(d64), n, _ptr(v64), _ptr(v32), _ptr(work),
                                                  _ptr(ctl), _stream(dev)))
        return v64.cpu().numpy() if was_np else v64
    if isinstance(choice, str):
        if choice != "uniform":
            raise InvalidSpec(f"unknown initial vector kind {choice!r}")
        v = np.full(n, 1.0 / n)
    else:
        v = np.asarray(choice, dtype=np.float64).copy()
        if v.shape != (n,):
            raise InvalidSpec(f"explicit v0 has length {v.size}, expected {n}")
        if v.min() < 0.0:
            raise InvalidSpec("explicit v0 must be nonnegative")
        if abs(v.sum() - 1.0) > 1e-12:
            raise InvalidSpec("explicit v0 must have unit L1 norm within 1e-12")
    return v if was_np else torch.from_numpy(v).to(dev)


def iterate(w, v, params: PicParams, config: KernelConfig | None = None):
    """Device-resident power iteration (parallel.py:217-233, serial.py:104-128)."""
    torch = _torch()
    if isinstance(w, DeviceAffinity):
        w = NormalizedAffinity(a=w.a, deg=None, n=w.n, lda=w.lda)
    was_np = not isinstance(w, NormalizedAffinity)
    if was_np:
        wn = np.asarray(w, dtype=np.float64)
        if wn.ndim != 2 or wn.shape[0] != wn.shape[1]:
            raise InvalidSpec(f"expected a square matrix, got shape {wn.shape}")
        dev = _device(config)
        a, rows, n, lda = _as_device_matrix(wn, dev)
        w = NormalizedAffinity(a=a, deg=None, n=n, lda=lda)
    dev = w.a.device
    n = w.n
    if w.a.shape[0] != n:
        raise InvalidSpec("iterate on one device needs the whole matrix (use cluster(p>1) for shards)")
    v64_in, v_np = _vec64(v, dev)
    if v64_in.numel() != n:
        raise DimensionMismatch((n, n), tuple(v64_in.shape))
    eps = params.resolved_epsilon(n)
    T = params.max_iterations
    v64 = torch.empty(2 * n, dtype=torch.float64, device=dev)
    v64[:n] = v64_in
    v32 = _vec32_padded(v64_in, n, dev)
    hist = torch.zeros(T, dtype=torch.float64, device=dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    ctl = _new_ctl(dev, eps, T)
    work = torch.empty(n + (n + 2047) // 2048 + 2, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().gpic_power_iterate(_ptr(w.a), w.lda, _ptr(w.deg), n, _ptr(v64),
                                             _ptr(v32), eps, T, _ptr(hist), _ptr(out), _ptr(work),
                                             _ptr(ctl), _stream(dev)))
    h = _read_ctl(ctl, dev)
    _raise_ctl(h)
    trace = PicTrace(int(h.iter), hist[: h.iter].cpu().numpy(), bool(h.converged))
    return (out.cpu().numpy() if (was_np or v_np) else out), trace


ROW_SUM_TOL = 1e-9  # serial.py:20


def generate_blobs(n: int, d: int, k: int, seed: int = 0, noise: float = 1.0,
                   radius: float = 40.0, offset: float = 8.0, sizes: str = "graded",
                   config: KernelConfig | None = None):
    """App-B Gaussian blobs generated in HBM (gpic_generate_blobs; §8f-4).

    Centres and blob sizes are exactly those of `datasets.gaussian_blobs`
    for the same arguments (the first k*d draws of the seeded numpy
    generator); the per-point noise comes from the device Philox stream, so
    X follows the same distribution but not the same draws. Returns
    (X float64 CUDA tensor (n, d), labels int64 CUDA tensor (n,)).
    """
    from .datasets import _even_split, graded_sizes

    torch = _torch()
    if k < 1 or n < k or d < 1:
        raise InvalidSpec("generate_blobs needs k >= 1, n >= k, d >= 1")
    if sizes == "graded":
        counts = graded_sizes(n, k)
    elif sizes == "balanced":
        counts = np.asarray(_even_split(n, k), dtype=np.int64)
    else:
        raise InvalidSpec(f"sizes must be 'graded' or 'balanced', got {sizes!r}")
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((k, d))
    centers /= np.linalg.norm(centers, axis=1, keepdims=True)
    centers *= radius
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    dev = _device(config)
    c_t = torch.from_numpy(np.ascontiguousarray(centers)).to(dev)
    o_t = torch.from_numpy(offsets).to(dev)
    x = torch.empty((n, d), dtype=torch.float64, device=dev)
    labels = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib().gpic_generate_blobs(_ptr(c_t), _ptr(o_t), n, d, k, seed & (2**64 - 1),
                                              float(noise), float(offset), _ptr(x), _ptr(labels),
                                              _stream(dev)))
    return x, labels


def check_row_stochastic(w, config: KernelConfig | None = None):
    """serial.py:63-74: every row of w sums to 1 within 1e-9, entries in [0, 1].

    The fp64 matrix is scanned on the device (gpic_row_stats: per-row sum,
    min, max); the verdict and the InvalidSpec messages follow the
    reference (the worst row is named). Returns w as float64.
    """
    torch = _torch()
    wn = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
    if wn.ndim != 2 or wn.shape[0] != wn.shape[1]:
        raise InvalidSpec(f"expected a square matrix, got shape {wn.shape}")
    n = wn.shape[0]
    if n == 0:
        raise InvalidSpec("expected a non-empty matrix")
    dev = _device(config)
    t = torch.from_numpy(wn).to(dev)
    stats = torch.empty((3, n), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().gpic_row_stats(_ptr(t), n, n, n, _ptr(stats[0]), _ptr(stats[1]),
                                         _ptr(stats[2]), _stream(dev)))
    sums, lo, hi = stats.cpu().numpy()
    if np.max(np.abs(sums - 1.0)) > ROW_SUM_TOL:
        bad = int(np.argmax(np.abs(sums - 1.0)))
        raise InvalidSpec(f"row {bad} sums to {sums[bad]!r}, not 1")
    if lo.min() < -1e-12 or hi.max() > 1.0 + 1e-12:
        raise InvalidSpec("entries must lie in [0, 1]")
    return wn


def power_iterate(w, params: PicParams, v0, config: KernelConfig | None = None):
    """serial.py:104-128: validate W row-stochastic, then the device power loop.

    Same contract as the serial entry point: (v, PicTrace), v float64 of
    length n. W is streamed in fp32 by the GEMV (DESIGN.md §2 tolerance).
    A `NormalizedAffinity` (from `normalize`/`k_normalize`) is row-stochastic
    by construction (D^-1 A with the degrees of the same A) and is not
    re-scanned.
    """
    if not isinstance(w, (NormalizedAffinity, DeviceAffinity)):
        w = check_row_stochastic(w, config)
    return iterate(w, v0, params, config)


# ---- serial-module names (affinity.py:107-127, serial.py:77-101) --------
def build_affinity(d: DataSet, kind, config: KernelConfig | None = None) -> np.ndarray:
    """affinity.py:107-110: the dense A (zero diagonal) as a host float64 array.

    Computed by the same device engine as `k_affinity` (fp32 storage) and
    copied out; use `k_affinity` to keep A on the device.
    """
    a = k_affinity(d, kind, config)
    _raise_ctl(_read_ctl(a.ctl, a.a.device), a.d)
    return a.a[:, : a.n].cpu().numpy().astype(np.float64)


def degree(a, config: KernelConfig | None = None):
    """affinity.py:113-119: row sums, ZeroDegree(first row) if any <= 0."""
    return k_rowsum(a, config)


def normalize(a, deg, config: KernelConfig | None = None):
    """affinity.py:122-127: W = A / deg, as the folded `NormalizedAffinity`
    view (no second n x n; `.numpy()` materialises it)."""
    return k_normalize(a, deg, config)


def initial_vector(deg, choice, config: KernelConfig | None = None):
    """serial.py:77-101: "degree" -> deg / sum(deg) (device tree sum),
    "uniform" -> 1/n, or a validated explicit vector."""
    return initial_embedding(deg, PicParams(k=2, v0=choice), config)


def kmeans_1d(values, params: KMeansParams, config: KernelConfig | None = None):
    """GPU 1-D k-means with the reference's seeding, ties and canonical labels."""
    torch = _torch()
    was_np = not hasattr(values, "is_cuda")
    dev = _device(config) if was_np else values.device
    v, _ = _vec64(values, dev)
    n = v.numel()
    k = params.k
    if k > n:
        raise KTooLarge(k, n)
    if k > KMEANS_MAX_K:
        raise InvalidSpec(f"the device k-means holds at most {KMEANS_MAX_K} centres")
    first, u = kmeans_draws(n, k, params.seed)
    L = _lib.lib()
    scratch = torch.empty(int(L.gpic_kmeans_scratch_bytes(n, k)), dtype=torch.uint8, device=dev)
    labels = torch.empty(n, dtype=torch.int64, device=dev)
    ctl = _new_ctl(dev)
    _lib.check(L.gpic_kmeans1d(_ptr(v), n, k, first, u.ctypes.data_as(C.c_void_p),
                               params.max_rounds, params.tol, _ptr(labels), _ptr(scratch),
                               _ptr(ctl), _stream(dev)))
    h = _read_ctl(ctl, dev)
    _raise_ctl(h)
    return labels.cpu().numpy() if was_np else labels


# ------------------------------------------------------------- pipeline
def workspace_bytes(n: int, d: int, k: int, max_iter: int, storage: int = 1) -> int:
    """Device bytes one cluster() call needs: scratch + the fp32 affinity storage."""
    return int(_lib.lib().gpic_cluster_workspace_bytes(n, d, k, max_iter, storage))


def cluster(d: DataSet, kind, params: PicParams, config: KernelConfig | None = None, seed: int = 0):
    """End-to-end PIC on the GPU: (labels int64[n], v float64[n], PicTrace).

    Same contract as parallel.cluster (parallel.py:236-255). One libgpic call
    runs centring, affinity + degree, the start vector, the device-resident
    power iteration and the k-means; the host syncs twice (after the loop and
    at the end).
    """
    _torch()
    config = config or KernelConfig()
    _check_kind(kind)
    check_shape(d)
    check_labels(d)
    n, m = d.points.shape
    k = params.k
    if k > n:
        raise KTooLarge(k, n)
    if k > KMEANS_MAX_K:
        raise InvalidSpec(f"the device k-means holds at most {KMEANS_MAX_K} centres")
    v0 = start_vector(params.v0, n)
    if config.p > 1:
        from . import sharded

        return sharded.cluster(d, kind, params, config, seed, v0=v0)
    labels, v, trace, _ = cluster_fused(d, kind, params, config, seed, v0=v0)
    return labels, v, trace


def start_vector(choice, n: int):
    """The host side of initial_vector (serial.py:77-101): None for "degree"
    (the device computes d / sum(d)), the 1/n vector for "uniform", or a
    validated copy of an explicit vector (length n, nonnegative, unit L1
    norm within 1e-12); InvalidSpec otherwise."""
    if isinstance(choice, str):
        if choice == "degree":
            return None
        if choice == "uniform":
            return np.full(n, 1.0 / n)
        raise InvalidSpec(f"unknown initial vector kind {choice!r}")
    v = np.asarray(choice, dtype=np.float64).copy()
    if v.shape != (n,):
        raise InvalidSpec(f"explicit v0 has length {v.size}, expected {n}")
    if v.min() < 0.0:
        raise InvalidSpec("explicit v0 must be nonnegative")
    if abs(v.sum() - 1.0) > 1e-12:
        raise InvalidSpec("explicit v0 must have unit L1 norm within 1e-12")
    return v


def cluster_fused(d: DataSet, kind, params: PicParams, config: KernelConfig, seed: int = 0,
                  timed: bool = False, v0=None):
    """One gpic_cluster call (p == 1). ``v0``: None (degree start) or an
    explicit start vector (see start_vector). With ``timed`` the per-phase
    device milliseconds come back as a dict (report.py:28 PHASES)."""
    torch = _torch()
    dev = _device(config)
    x = torch.from_numpy(d.points).to(dev, non_blocking=True)
    if v0 is None:
        v0 = start_vector(params.v0, d.points.shape[0])
    return _cluster_x(x, kind, params, config, seed, timed, v0)


def cluster_points(x, kind, params: PicParams, config: KernelConfig | None = None, seed: int = 0,
                   timed: bool = False):
    """`cluster` on a device-resident fp64 (n, d) tensor (e.g. from
    `generate_blobs`): no host copy of X. Returns numpy labels / embedding
    and the PicTrace (+ phase ms when ``timed``), like `cluster_fused`."""
    torch = _torch()
    if not (hasattr(x, "is_cuda") and x.is_cuda and x.dtype == torch.float64 and x.dim() == 2):
        raise InvalidSpec("cluster_points needs a CUDA float64 (n, d) tensor")
    if x.shape[0] < params.k:
        raise KTooLarge(params.k, x.shape[0])
    return _cluster_x(x.contiguous(), kind, params, config or KernelConfig(), seed, timed,
                      start_vector(params.v0, x.shape[0]))


def _cluster_x(x, kind, params, config, seed, timed, v0=None):
    torch = _torch()
    code, sigma = _check_kind(kind)
    n, m = x.shape
    k = params.k
    dev = x.device
    L = _lib.lib()
    eps = params.resolved_epsilon(n)
    T = params.max_iterations
    impl = _lib.AFFINITY_TC if config.affinity_impl == "tc" else _lib.AFFINITY_SIMT
    storage = config.storage_code()
    nbytes = workspace_bytes(n, m, k, T, storage)
    work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    # labels, v and the delta history side by side: one device->host copy
    # (every entry read back is written by the run: labels and v in full,
    # the history up to the iteration count)
    out = torch.empty(2 * n + T, dtype=torch.int64, device=dev)
    labels = out[:n]
    v = out[n:2 * n].view(torch.float64)
    hist = out[2 * n:].view(torch.float64)
    first, u = kmeans_draws(n, k, seed)
    iters = C.c_int32(0)
    conv = C.c_int32(0)
    v0_t = None if v0 is None else torch.from_numpy(np.ascontiguousarray(v0)).to(dev)
    args = (_ptr(x), n, m, sigma, code, k, eps, T, first, u.ctypes.data_as(C.c_void_p), impl,
            storage, _ptr(v0_t), _ptr(labels), _ptr(v), _ptr(hist), C.byref(iters), C.byref(conv),
            _ptr(work), nbytes, _stream(dev))
    ms = (C.c_float * 5)()
    rc = L.gpic_cluster_timed(*args, ms) if timed else L.gpic_cluster(*args)
    if rc != _lib.GPIC_OK:
        h = _lib.Ctl()
        if L.gpic_ctl_read(_ptr(work), C.byref(h), _stream(dev)) == 0 and h.status == rc:
            _lib.raise_for(rc, h, m)
        _lib.raise_for(rc, None, m)
    it = int(iters.value)
    phases = dict(zip(("affinity", "rowsum", "normalize", "iterate", "kmeans"),
                      (t / 1e3 for t in ms))) if timed else None
    # into page-locked memory from torch's caching host allocator (a
    # pageable destination halves the copy rate); the returned arrays are
    # views that keep that block alive
    host_t = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    host_t.copy_(out, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    host = host_t.numpy()
    return (host[:n], host[n:2 * n].view(np.float64),
            PicTrace(it, host[2 * n:2 * n + it].view(np.float64).copy(), bool(conv.value)), phases)


# ------------------------------------------------- batched small problems
BATCH_MAX_N = 4096


def cluster_batch(datasets, kind, params: PicParams, seeds, config: KernelConfig | None = None):
    """Many small independent PIC runs in one launch (Experiment II engine).

    ``datasets``: DataSets with the same feature count and 1..4096 points;
    ``seeds``: the k-means seed of each run. Returns one (labels, v, PicTrace)
    per dataset — what ``cluster(d, kind, params, seed=s)`` returns for it.
    Errors raise the reference's exception of the first failing problem, in
    input order (cli.py:240-246 runs them one after another).
    """
    torch = _torch()
    config = config or KernelConfig()
    code, sigma = _check_kind(kind)
    datasets = list(datasets)
    seeds = list(seeds)
    if not datasets or len(seeds) != len(datasets):
        raise InvalidSpec("cluster_batch needs one seed per dataset and at least one dataset")
    if not (isinstance(params.v0, str) and params.v0 == "degree"):
        raise InvalidSpec("the batched engine starts from the degree vector (v0='degree')")
    for d in datasets:
        check_shape(d)
        check_labels(d)
    m = datasets[0].points.shape[1]
    if any(d.points.shape[1] != m for d in datasets):
        raise DimensionMismatch((datasets[0].n, m), next(d.points.shape for d in datasets
                                                          if d.points.shape[1] != m))
    k = params.k
    for d in datasets:
        if k > d.n:
            raise KTooLarge(k, d.n)
    if k > BATCH_MAX_K:
        raise InvalidSpec(f"the batched k-means holds at most {BATCH_MAX_K} centres")
    if max(d.n for d in datasets) > BATCH_MAX_N:
        raise InvalidSpec(f"batched problems hold at most {BATCH_MAX_N} points; use cluster()")
    B = len(datasets)
    T = params.max_iterations
    offsets = np.zeros(B + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([d.n for d in datasets])
    eps = np.array([params.resolved_epsilon(d.n) for d in datasets], dtype=np.float64)
    first = np.zeros(B, dtype=np.int64)
    unif = np.zeros(B * max(k - 1, 1), dtype=np.float64)
    for b, (d, s) in enumerate(zip(datasets, seeds)):
        f, u = kmeans_draws(d.n, k, s)
        first[b] = f
        unif[b * (k - 1):(b + 1) * (k - 1)] = u[: k - 1]
    dev = _device(config)
    L = _lib.lib()
    x = torch.from_numpy(np.ascontiguousarray(np.concatenate([d.points for d in datasets]))).to(dev)
    N = int(offsets[-1])
    labels = torch.empty(N, dtype=torch.int64, device=dev)
    v = torch.empty(N, dtype=torch.float64, device=dev)
    hist = torch.zeros(B * T, dtype=torch.float64, device=dev)
    cptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    nbytes = int(L.gpic_batch_workspace_bytes(cptr(offsets), B, m, k, T))
    if nbytes < 0:
        raise InvalidSpec("invalid batch shape")
    work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ctls = (_lib.Ctl * B)()
    rc = L.gpic_cluster_batch(_ptr(x), cptr(offsets), B, m, sigma, code, k, cptr(eps), T,
                              cptr(first), cptr(unif), _ptr(labels), _ptr(v), _ptr(hist), ctls,
                              _ptr(work), nbytes, _stream(dev))
    _lib.check(rc)
    for c in ctls:
        if c.status != _lib.GPIC_OK:
            _lib.raise_for(c.status, c, m)
    lab_np, v_np, h_np = labels.cpu().numpy(), v.cpu().numpy(), hist.cpu().numpy()
    out = []
    for b in range(B):
        lo, hi = int(offsets[b]), int(offsets[b + 1])
        it = int(ctls[b].iter)
        out.append((lab_np[lo:hi].copy(), v_np[lo:hi].copy(),
                    PicTrace(it, h_np[b * T: b * T + it].copy(), bool(ctls[b].converged))))
    return out
