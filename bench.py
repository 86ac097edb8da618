"""GPIC benchmark: PIC end to end on BASELINE.json config 3 (n=100k, d=64, k=10).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

A step is one whole PIC run (centre -> affinity+degree -> start vector ->
device-resident power iteration -> k-means) over the config's synthetic
Gaussian blobs (SURVEY.md App. B generator, seed 0). Prints ONE JSON line
(rank 0). Key fields:

  value      seconds per PIC run with X already resident in HBM (CUDA events,
             max over ranks), the BASELINE metric ("PIC end-to-end s")
  e2e        the same through the public API cluster(DataSet(host X)) with
             the H2D of X and the D2H of labels + embedding inside the timing
  roofline   the dominant kernel (the power-iteration GEMV): algorithmic
             bytes (rows * n * 4 per launch) / its CUDA-event duration vs the
             measured HBM peak
  cpu_baseline  the reference algorithm (oracle/ numpy port of the
             reference's threaded backend) on a bounded row sample, scaled to
             the full job
  power_iter_hbm_gbs  the second half of the BASELINE metric

--impl reference times only the CPU reference port (rank 0) on the same
config and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1604_02700_b200.datasets import CONFIGS, config_dataset  # noqa: E402

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def f16_peak():
    """Dense fp16 tensor rate (kind::f16, fp32 accumulate) = the measured
    cuBLAS bf16 burst rate (same pipe, same rate)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["bf16_tflops"]), "measured (bf16 cuBLAS burst)"
    return 1590.0, "fallback"


CONFIGS_SIGMA = {c["n"]: c["sigma"] for c in CONFIGS.values()}


# ------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        import threading

        self.lines = []
        self._live = True
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
        except OSError:
            self.proc = None
            return self
        first = threading.Event()

        def pump():
            for ln in self.proc.stdout:
                if ln.strip():
                    if self._live:
                        self.lines.append(ln.strip())
                    first.set()

        self._thread = threading.Thread(target=pump, daemon=True)
        self._thread.start()
        first.wait(timeout=5.0)  # sampling is live before the timed region starts
        self.lines.clear()
        return self

    def __exit__(self, *exc):
        self._live = False
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------- CPU reference
REF_DIR = ROOT / "baseline" / "_ref"


def reference_package():
    """The unmodified reference package installed into baseline/_ref (see
    DESIGN.md §9), or None when it is not installed on this host."""
    if not (REF_DIR / "picluster" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import picluster

    return picluster


def host_info(threads):
    mem = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal:"):
                mem = round(int(ln.split()[1]) / 2**20, 1)
    except OSError:
        pass
    return {"cores": threads, "os_cpu_count": os.cpu_count(), "host_ram_gib": mem,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset"),
            "numpy": np.__version__}


def fixture(cfg):
    """CPU-reference fixture of a benchmark config (tests/golden/config<c>.npz)."""
    p = ROOT / "tests" / "golden" / f"config{cfg}.npz"
    return dict(np.load(p)) if p.exists() else None


def cpu_reference_sample(points, sigma, k, iters, threads, v_real=None, offset=0, block=None):
    """One bounded sample of the CPU reference's own pipeline, scaled to the job.

    With the reference installed (baseline/_ref) it runs the reference's own
    code exactly as parallel.cluster composes it (parallel.py:113-255): its
    `similarity_rows` per `resolved_chunk_rows(n)`-row block (335 rows at
    n = 100k, 256 MiB per block) with one block per worker of a
    `_run_workers` pool of `threads` workers — the memory footprint of every
    worker of the full run — then `k_rowsum`, `k_normalize` and `iters` x
    `k_multiply` on those rows, `k_reduce` / `k_norm` / the delta on full
    n-vectors, and `kmeans_1d` on the real embedding (the committed CPU
    fixture's v). Row-proportional phases are scaled by n / rows.
    Without it, the oracle's port of the same steps (kind "port").

    Returns (seconds_full_job, phases, measured_wall_seconds, kind, sample).
    """
    n = points.shape[0]
    ref = reference_package()
    if ref is not None:
        from picluster import parallel as P
        from picluster.affinity import GaussianRbf as RefRbf
        from picluster.affinity import similarity_rows
        from picluster.kmeans import KMeansParams as RefKM
        from picluster.kmeans import kmeans_1d

        cfgk = P.KernelConfig(p=threads)
        chunk = cfgk.resolved_chunk_rows(n)
        if block is not None:  # shorter blocks (still far beyond the LLC) for many-step runs
            chunk = min(chunk, block)
        kind = RefRbf(sigma)
        step = max(1, n // threads)
        starts = [((offset + w) * step) % max(1, n - chunk + 1) for w in range(threads)]
        rows = chunk * threads
        t0 = time.perf_counter()
        a = np.empty((rows, n))

        def worker(lo, hi):  # one 256 MiB block per worker, as k_affinity's workers do
            w = lo // chunk
            a[lo:hi] = similarity_rows(points, starts[w], starts[w] + (hi - lo), kind)

        P._run_workers(worker, P.PartitionPlan(tuple((w * chunk, (w + 1) * chunk)
                                                     for w in range(threads))), threads)
        t1 = time.perf_counter()
        deg = P.k_rowsum(a, cfgk)
        w_ = P.k_normalize(a, deg, cfgk)
        del a
        t2 = time.perf_counter()
        v = np.full(n, 1.0 / n)
        t_mul = t_vec = 0.0
        for _ in range(iters):
            s0 = time.perf_counter()
            P.k_multiply(w_, v, cfgk)
            s1 = time.perf_counter()
            tau = P.k_reduce(v, cfgk)
            v_next = P.k_norm(v, tau, cfgk)
            float(np.max(np.abs(v_next - v)))
            s2 = time.perf_counter()
            t_mul += s1 - s0
            t_vec += s2 - s1
        del w_
        vk = v_real if v_real is not None else v
        t4 = time.perf_counter()
        kmeans_1d(np.asarray(vk, dtype=np.float64), RefKM(k=k, seed=0))
        t5 = time.perf_counter()
        kind_s = "reference"
        sample = (f"the reference's own parallel-backend code (baseline/_ref picluster): "
                  f"{threads} workers x one {chunk}-row block (resolved_chunk_rows(n) = "
                  f"{cfgk.resolved_chunk_rows(n)}) = {rows} of {n} "
                  f"affinity rows + k_rowsum/k_normalize + {iters} k_multiply on them, scaled "
                  f"x{n / rows:.1f}; k_reduce/k_norm on full vectors; kmeans_1d on the "
                  f"{'CPU-reference embedding' if v_real is not None else 'uniform vector'} (n={n})")
    else:
        from oracle import pic_oracle as po

        chunk = po.chunk_rows(n)
        rows = chunk * threads
        t0 = time.perf_counter()
        a = po.affinity_rows_threaded(points, 0, rows, sigma, p=threads)
        t1 = time.perf_counter()
        deg = np.einsum("ij->i", a)
        w_ = a / deg[:, None]
        del a
        t2 = time.perf_counter()
        v = np.full(n, 1.0 / n)
        t_mul = t_vec = 0.0
        for _ in range(iters):
            s0 = time.perf_counter()
            po.matvec_threaded(w_, v, threads)
            s1 = time.perf_counter()
            v_next = v / po.tree_sum(v)
            float(np.max(np.abs(v_next - v)))
            s2 = time.perf_counter()
            t_mul += s1 - s0
            t_vec += s2 - s1
        del w_
        vk = v_real if v_real is not None else v
        t4 = time.perf_counter()
        po.kmeans_1d(np.asarray(vk, dtype=np.float64), k, 0)
        t5 = time.perf_counter()
        kind_s = "port"
        sample = (f"oracle port of the reference's parallel backend: {rows} of {n} affinity rows "
                  f"in {chunk}-row blocks + {iters} matvecs, scaled x{n / rows:.1f}; k-means on "
                  f"n={n}")
    scale = n / rows
    phases = {"affinity_s": (t1 - t0) * scale, "rowsum_normalize_s": (t2 - t1) * scale,
              "iterate_s": t_mul * scale + t_vec, "kmeans_s": t5 - t4}
    full = sum(phases.values())
    return full, phases, (t5 - t0), kind_s, sample


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    c = CONFIGS[cfg]
    d = config_dataset(cfg, seed=0)
    threads = os.cpu_count() or 1
    fx = fixture(cfg)
    iters = int(fx["iterations"]) if fx is not None else args.ref_iters
    v_real = fx["v"] if fx is not None else None
    times, phases, walls = [], [], []
    kind = sample = None
    # bounded run: one reference-sized 256 MiB block per worker costs ~23 s
    # at config 3 on 16 cores; with many steps each worker's block shrinks
    # (>= 64 MiB, still ~1000x the LLC share, so the run stays memory-bound
    # like the full job) so that W + K steps end within ~3 minutes
    nsteps = args.warmup + args.steps
    chunk_full = max(1, min(c["n"], 256 * 1024 * 1024 // (8 * c["n"])))
    block = max(min(chunk_full, 16), chunk_full * 8 // max(nsteps, 8))
    for i in range(nsteps):
        full, det, w, kind, sample = cpu_reference_sample(d.points, c["sigma"], c["k"], iters,
                                                          threads, v_real, offset=i, block=block)
        if i >= args.warmup:
            times.append(full)
            phases.append(det)
            walls.append(w)
    value = statistics.mean(times)
    line = {
        "metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY App. B gaussian blobs, seed 0)", "impl": "reference",
        "config": workload(cfg, args.gpus),
        "cpu_baseline": dict(value=value, unit="s", kind=kind, sample=sample,
                             phases={k: statistics.mean(p[k] for p in phases) for k in phases[0]},
                             extrapolated=True,
                             measured_cpu_seconds_per_step=statistics.mean(walls),
                             **host_info(threads)),
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "PIC end-to-end s (power-iter HBM GB/s alongside)"


def workload(cfg, gpus):
    c = CONFIGS[cfg]
    return {"workload": f"config{cfg}: gaussian blobs n={c['n']} d={c['d']} k={c['k']} "
                        f"sigma={c['sigma']:.4f}",
            "n": c["n"], "d": c["d"], "k": c["k"], "sigma": c["sigma"],
            "parallelism": f"row-shard x{gpus}", "l2": "inputs > L2 (W = 4n^2 bytes)"}


# ---------------------------------------------------------- ours
def _gemv_roofline(args, L, C, torch, stream, st, n, m, k, T, work, v, storage):
    """Time the dominant kernel (the power-iteration GEMV) on the resident
    affinity storage, CUDA events on the launching stream."""
    scratch = int(L.gpic_workspace_bytes(n, m, k, n, T))
    base = work.data_ptr() + scratch
    dev = work.device
    vp = int(L.gpic_vector_pitch(n))
    v32 = torch.zeros(vp, dtype=torch.float32, device=dev)
    v32[:n] = v.to(torch.float32)
    yv = torch.empty(n, dtype=torch.float64, device=dev)
    deg1 = torch.ones(n, dtype=torch.float64, device=dev)
    if storage == 2:
        # matrix-free: the power loop's own A v pass (tcgen05 3-term fp16 Gram
        # + exp + v, over the kept tiles after pruning), rerun on the
        # operands / mask the cluster run left in `work`
        dp = int(L.gpic_feature_pitch(m))
        sigma = CONFIGS_SIGMA[n]
        pruned = 1 if os.environ.get("GPIC_PRUNE", "1") != "0" and os.environ.get(
            "GPIC_SPARSE", "1") != "0" and m > 8 else 0

        from paper_1604_02700_b200 import _lib

        def launch():
            return L.gpic_cluster_mf_pass(C.c_void_p(work.data_ptr()), n, m, k, T, sigma,
                                          _lib.KIND_RBF, pruned, C.c_void_p(v32.data_ptr()),
                                          C.c_void_p(yv.data_ptr()), st)
        # units computed (MB row tiles x 1 column tile each, J >= MB * I,
        # minus the pruned ones) x 128 MB x 128 entries x 3 terms x 2 x
        # (dp + 16 norm-block columns)
        mb = 2 if dp == 64 else 1
        kept, tot = C.c_int64(0), C.c_int64(0)
        assert L.gpic_cluster_pruned_work(C.c_void_p(work.data_ptr()), n, m, k, T, storage,
                                          C.byref(kept), C.byref(tot), st) == 0
        units = kept.value if pruned else tot.value
        if os.environ.get("GPIC_MF_SYM", "1") == "0":
            units = -(-n // (128 * mb)) * -(-n // 128)
        alg = 3.0 * 2.0 * (dp + 16) * float(units) * 128 * mb * 128
        name = ("affinity_tc_kernel<matvec> (matrix-free symmetric A v pass: 3-term fp16 Gram "
                "with the distance from the MMA, exp2, row + column products; "
                f"{units} of {tot.value} tile units after pruning)")
    elif storage in (1, 3):
        # the packed GEMV as the run executes it: only tiles with a stored
        # box are read (block sparsity, csrc/sparse.cu); algorithmic bytes =
        # the stored tiles' bytes, counted from the run's own box flags
        offs = (C.c_int64 * 8)()
        assert L.gpic_cluster_workspace_layout(n, m, k, T, storage, offs) == 0
        base0 = work.data_ptr()
        tiles, rowp, colp = base0 + offs[0], base0 + offs[1], base0 + offs[2]
        boxnz_p, sbp_p = base0 + offs[3], base0 + offs[4]
        ntiles = int(L.gpic_packed_tiles(n))
        elem = 4 if storage == 1 else 2
        sparse = os.environ.get("GPIC_SPARSE", "1") != "0"
        stored = None
        if sparse:  # the run's flags, read in place from the workspace
            flags = work[offs[3]: offs[3] + ntiles * 16].view(ntiles, 16)
            stored = int((flags.amax(dim=1) > 0).sum().item())
        tile_bytes = (stored if stored is not None else ntiles) * 128 * 128 * elem

        def launch():
            return L.gpic_sym_matvec_sparse(
                C.c_void_p(tiles), 0 if storage == 1 else 1, n, C.c_void_p(v32.data_ptr()),
                C.c_void_p(rowp), C.c_void_p(colp), C.c_void_p(deg1.data_ptr()),
                C.c_void_p(yv.data_ptr()), C.c_void_p(boxnz_p if sparse else 0),
                C.c_void_p(sbp_p if sparse else 0), st)
        alg = float(tile_bytes)
        name = ("sym_gemv_kernel + sym_reduce_kernel (packed symmetric tiles, "
                + ("fp32" if storage == 1 else "fp16")
                + (f", block-sparse: {stored} of {ntiles} tiles stored)" if sparse else ")"))
    else:
        lda = int(L.gpic_affinity_pitch(n))

        def launch():
            return L.gpic_matvec(C.c_void_p(base), lda, n, n, C.c_void_p(v32.data_ptr()),
                                 C.c_void_p(deg1.data_ptr()), C.c_void_p(yv.data_ptr()), st)
        alg = float(n) * n * 4
        name = "gemv_bulk_kernel (dense rows)"
    times = []
    for rep in range(args.gemv_reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rc = launch()
        e1.record(stream)
        e1.synchronize()
        if rc:
            raise RuntimeError(f"GEMV launch failed: {rc}")
        if rep >= 2:
            times.append(e0.elapsed_time(e1))
    return name, alg, statistics.mean(times)


def run_ours(args, cfg, rank, world):
    import ctypes as C

    import torch

    from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams, cluster
    from paper_1604_02700_b200 import _lib, gpu
    from paper_1604_02700_b200.validation import adjusted_rand_index, contingency

    if world > 1:
        return run_ours_sharded(args, cfg, rank, world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    c = CONFIGS[cfg]
    d = config_dataset(cfg, seed=0)
    n, m, k = d.n, d.m, c["k"]
    sigma = c["sigma"]
    params = PicParams(k=k)
    impl_name = args.engine
    cfg_api = KernelConfig(affinity_impl=impl_name, storage=args.storage)
    impl = _lib.AFFINITY_TC if impl_name == "tc" else _lib.AFFINITY_SIMT
    storage = cfg_api.storage_code()
    L = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    st = C.c_void_p(stream.cuda_stream)

    # pinned host input for the e2e leg (DataSet keeps the buffer, no copy)
    host = torch.empty((n, m), dtype=torch.float64).pin_memory()
    host.numpy()[:] = d.points
    d_host = DataSet(host.numpy(), d.labels)

    # device-resident leg: one libgpic call per step on X already in HBM
    x = torch.from_numpy(d.points).to(dev)
    T = params.max_iterations
    nbytes = gpu.workspace_bytes(n, m, k, T, storage)
    work = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    labels = torch.empty(n, dtype=torch.int64, device=dev)
    v = torch.empty(n, dtype=torch.float64, device=dev)
    hist = torch.zeros(T, dtype=torch.float64, device=dev)
    first, u = gpu.kmeans_draws(n, k, 0)
    eps = params.resolved_epsilon(n)
    iters, conv = C.c_int32(0), C.c_int32(0)

    def step():
        rc = L.gpic_cluster(C.c_void_p(x.data_ptr()), n, m, sigma, _lib.KIND_RBF, k, eps, T, first,
                            u.ctypes.data_as(C.c_void_p), impl, storage, None,
                            C.c_void_p(labels.data_ptr()), C.c_void_p(v.data_ptr()),
                            C.c_void_p(hist.data_ptr()), C.byref(iters), C.byref(conv),
                            C.c_void_p(work.data_ptr()), nbytes, st)
        _lib.raise_for(rc)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = L.gpic_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = (L.gpic_launch_count() - launches0) // args.steps
    ms = ev0.elapsed_time(ev1) / args.steps
    lab_np = labels.cpu().numpy()
    ari = adjusted_rand_index(contingency(d.labels, lab_np))
    fx = fixture(cfg)
    parity = None
    if fx is not None:
        ref_lab = fx["labels"].astype(np.int64)
        v_np = v.cpu().numpy()
        parity = {"ari_vs_cpu": adjusted_rand_index(contingency(ref_lab, lab_np)),
                  "labels_identical": bool(np.array_equal(ref_lab, lab_np)),
                  "iterations_cpu": int(fx["iterations"]),
                  "rel_l1_v_vs_cpu": float(np.abs(v_np - fx["v"]).sum() / np.abs(fx["v"]).sum()),
                  "cpu_reference": str(fx["provenance"])}

    kname, alg_bytes, gemv_ms = _gemv_roofline(args, L, C, torch, stream, st, n, m, k, T, work,
                                               v, storage)
    pruning = None
    if storage in (1, 2, 3) and args.engine == "tc":
        kept, tot = C.c_int64(0), C.c_int64(0)
        if L.gpic_cluster_pruned_work(C.c_void_p(work.data_ptr()), n, m, k, T, storage,
                                      C.byref(kept), C.byref(tot), st) == 0:
            pruning = {"tensor_units_computed": int(kept.value), "tensor_units_total": int(tot.value),
                       "rule": "block pairs whose projection bound puts every entry below 2^-66 "
                               "are not computed (bit-identical: they flush to 0 at 2^-64)"}
    achieved = alg_bytes / (gemv_ms * 1e-3) / 1e9
    dense_equiv = float(n) * n * 4 / (gemv_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    bound, unit = "hbm", "GB/s"
    if storage == 2:
        # tensor-bound: the fp16 MMA rate = the measured bf16 cuBLAS rate
        achieved = alg_bytes / (gemv_ms * 1e-3) / 1e12
        peak, peak_kind = f16_peak()
        bound, unit = "tensor", "TFLOP/s"

    # e2e leg through the public API from pinned host memory. Warm-up in
    # the timed loop's own pattern: the returned arrays are views of a
    # page-locked block that stays alive while the caller holds them, so two
    # blocks alternate once the previous result is still referenced (the
    # second one's first page-locking is not a per-call cost)
    for _ in range(max(3, args.warmup)):
        lab_e, v_e, tr_e = cluster(d_host, GaussianRbf(sigma), params, config=cfg_api, seed=0)
    torch.cuda.synchronize()
    e2e = []
    for _ in range(max(1, args.e2e_steps)):
        t0 = time.perf_counter()
        lab_e, v_e, tr_e = cluster(d_host, GaussianRbf(sigma), params, config=cfg_api, seed=0)
        e2e.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e)
    assert np.array_equal(lab_e, lab_np), "public-API labels differ from the device-resident run"

    # phase breakdown (report.run_timed, CUDA events at the phase boundaries)
    from paper_1604_02700_b200 import report as R

    rep, _ = R.benchmark(d_host, GaussianRbf(sigma), params, backend="gpu", config=cfg_api,
                         seed=0, repetitions=3)
    if args.report:
        rep.write(args.report)
    phases_ms = {p: statistics.median(r["phases"][p] for r in rep.runs) * 1e3 for p in R.PHASES}

    traffic = None
    prof = ROOT / "profiles" / "gemv_traffic.json"
    if prof.exists():
        for ent in json.loads(prof.read_text()).get("entries", []):
            if ent.get("storage") == args.storage and ent.get("n") == n:
                traffic = ent.get("dram_bytes_per_launch")

    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None,
        "dtype": ("f32 (3-term fp16-split tensor Gram, fp32 accumulate; fp64 vectors/reductions)"
                  if storage != 3 else
                  "f16 W storage (fp32 Gram/exp, fp32 accumulate; fp64 vectors/reductions)"),
        "data": "synthetic (SURVEY App. B gaussian blobs, seed 0)",
        "config": workload(cfg, world),
        "engine": {"affinity_engine": impl_name, "storage": args.storage},
        "power_iter_hbm_gbs": achieved, "power_iter_dense_equiv_gbs": dense_equiv,
        "iterations": int(iters.value), "converged": bool(conv.value), "ari_vs_truth": ari,
        "ari_vs_cpu": parity["ari_vs_cpu"] if parity else None,
        "parity_vs_cpu": parity,
        "roofline": {"kernel": kname, "bound": bound, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": unit, "frac": achieved / peak,
                     "traffic": traffic,
                     ("algorithmic_flops_per_launch" if storage == 2
                      else "algorithmic_bytes_per_launch"): alg_bytes,
                     "avg_launch_ms": gemv_ms},
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(n * m * 8),
                "d2h_bytes_per_step": int(n * 8 * 2 + T * 8), "steps": len(e2e),
                "median": statistics.median(e2e), "max": max(e2e)},
        "phases_ms": phases_ms,
        "pruning": pruning,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        full, det, wall, kind_s, sample = cpu_reference_sample(
            d.points, sigma, k, max(int(iters.value), 1), threads,
            fx["v"] if fx is not None else None)
        line["cpu_baseline"] = dict(value=full, unit="s", kind=kind_s, sample=sample, phases=det,
                                    extrapolated=True, measured_cpu_seconds=wall,
                                    **host_info(threads))
    print(json.dumps(line), flush=True)


def run_ours_sharded(args, cfg, rank, world):
    """N > 1: one rank per GPU, packed symmetric super-row shards balanced by
    kept tensor units, P2P partial-y exchange (reduce-scatter + all-gather
    from N = 3); dense row shards with the fused y all-gather otherwise."""
    import torch
    import torch.distributed as dist

    from paper_1604_02700_b200 import DataSet, GaussianRbf, KernelConfig, PicParams
    from paper_1604_02700_b200 import _lib, sharded
    from paper_1604_02700_b200.validation import adjusted_rand_index, contingency

    # GPIC_BENCH_SAME_DEVICE=1 (functional check on a one-GPU box only): every
    # rank shares device 0 (CUDA IPC still carries the exchange) and the
    # timing collectives go over gloo; the timings it prints are not N-GPU
    # numbers
    same = os.environ.get("GPIC_BENCH_SAME_DEVICE") == "1"
    local = 0 if same else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if same:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cdev = torch.device("cpu") if same else dev
    c = CONFIGS[cfg]
    d = config_dataset(cfg, seed=0)
    n, m, k, sigma = d.n, d.m, c["k"], c["sigma"]
    params = PicParams(k=k)
    storage = "packed" if args.storage == "packed" and args.engine == "tc" else "dense"
    config = KernelConfig(p=world, device=local, affinity_impl=args.engine, storage=storage)
    runner = sharded.ShardedRunner(n, config)
    x = torch.from_numpy(d.points).to(dev)
    stream = torch.cuda.current_stream(dev)
    L = _lib.lib()
    for _ in range(args.warmup):
        runner.run(x, GaussianRbf(sigma), params, 0)
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = L.gpic_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            labels, v, trace = runner.run(x, GaussianRbf(sigma), params, 0)
        ev1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms_local], device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    launches = (L.gpic_launch_count() - launches0) // args.steps
    lab_np = labels.cpu().numpy()
    agree = sharded.all_ranks_agree(lab_np, v.cpu().numpy())
    # e2e: host X in, host labels / v out, through the public runner
    host = torch.empty((n, m), dtype=torch.float64).pin_memory()
    host.numpy()[:] = d.points
    d_host = DataSet(host.numpy(), d.labels)
    e2e = []
    for _ in range(max(1, args.e2e_steps)):
        dist.barrier()
        t0 = time.perf_counter()
        lab_e, v_e, _ = runner.run(d_host, GaussianRbf(sigma), params, 0)
        lab_e, v_e = lab_e.cpu().numpy(), v_e.cpu().numpy()
        e2e.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.mean(e2e)], device=cdev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    runner.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (3-term fp16-split tensor Gram, fp32 accumulate; fp64 vectors/reductions)",
            "data": "synthetic (SURVEY App. B gaussian blobs, seed 0)",
            "config": dict(workload(cfg, world),
                           parallelism=(f"packed symmetric super-row shards x{world}, P2P partial-y "
                                        "exchange (reduce-scatter + all-gather from 3 ranks) summed "
                                        "in rank order" if storage == "packed" else
                                        f"row-shard x{world}, fused P2P y all-gather")),
            "engine": {"affinity_engine": args.engine, "storage": storage},
            "iterations": trace.iterations_run, "converged": trace.converged,
            "ari_vs_truth": adjusted_rand_index(contingency(d.labels, lab_np)),
            "ari_vs_cpu": (adjusted_rand_index(contingency(fixture(cfg)["labels"].astype(np.int64),
                                                           lab_np))
                           if fixture(cfg) is not None else None),
            "ranks_agree_bitwise": agree,
            "e2e": {"value": float(te.item()), "unit": "s", "h2d_bytes_per_step": int(n * m * 8),
                    "d2h_bytes_per_step": int(n * 8 * 2)},
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--engine", choices=["tc", "simt"], default="tc")
    ap.add_argument("--storage", choices=["packed", "dense", "none", "packed16"], default="packed")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--gemv-reps", type=int, default=10)
    ap.add_argument("--ref-iters", type=int, default=7)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--report", default=None,
                    help="also write a BenchReport (schema 1, report.py) of 3 timed runs here")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, args.config, rank)
        return
    run_ours(args, args.config, rank, world)


if __name__ == "__main__":
    main()
