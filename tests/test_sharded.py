"""Multi-rank path: host logic on CPU (gloo, world_size 2) and GPU-count
invariance on one GPU (virtual ranks + two processes sharing the device).

Mirrors the reference's bitwise p-invariance tests (test_parallel.py:194-223,
test_acceptance.py:127-155): the embedding, deltas and labels must be
IDENTICAL for any rank count.
"""

import os
import pathlib
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_02700_b200 import GaussianRbf, KernelConfig, PicParams, cluster, gaussian_blobs
from paper_1604_02700_b200 import _lib, errors, sharded

ROOT = pathlib.Path(__file__).resolve().parent.parent


# ------------------------------------------------------------- CPU / gloo
@pytest.mark.parametrize("n,p", [(10, 4), (9, 4), (100_000, 8), (8, 8), (1000, 3)])
def test_shard_ranges_cover_and_nonempty(n, p):
    r = sharded.shard_ranges(n, p)
    assert len(r) == p and r[0][0] == 0 and r[-1][1] == n
    assert all(b > a for a, b in r)
    assert all(r[i][1] == r[i + 1][0] for i in range(p - 1))
    assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1


def test_shard_ranges_rejects():
    with pytest.raises(errors.InvalidSpec):
        sharded.shard_ranges(3, 4)
    with pytest.raises(errors.InvalidSpec):
        sharded.shard_ranges(100, 9)


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        assert sharded.dist_context() == (rank, world)
        mine = bytes([rank]) * _lib.IPC_HANDLE_BYTES
        got = sharded.exchange_handles(mine, world)
        blob = sharded.assemble_handles(got)
        ok_handles = blob == b"".join(bytes([r]) * _lib.IPC_HANDLE_BYTES for r in range(world))
        same = sharded.all_ranks_agree(np.arange(5), np.ones(5))
        diff = sharded.all_ranks_agree(np.arange(5) + rank, np.ones(5))
        q.put((rank, ok_handles, same, diff))
    finally:
        dist.destroy_process_group()


def test_handle_exchange_and_agreement_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] for r in res)          # every rank saw every handle, in rank order
    assert all(r[2] for r in res)          # identical results agree
    assert not any(r[3] for r in res)      # differing results are caught


def test_world_mismatch_is_rejected_without_a_gpu_call():
    cfg = KernelConfig(p=2)
    assert sharded.dist_context() == (0, 1)
    if torch.cuda.is_available():
        with pytest.raises(errors.InvalidSpec):
            cluster(gaussian_blobs(100, 4, 2, seed=0), GaussianRbf(1.0), PicParams(k=2), config=cfg)


def test_malformed_handle_rejected():
    with pytest.raises(errors.DeviceError):
        sharded.assemble_handles([b"x" * 64, b"y" * 10])


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["tc", "simt"])
def test_virtual_ranks_bitwise_invariant(engine):
    d = gaussian_blobs(3000, 32, 5, seed=2)
    kind, params = GaussianRbf(float(np.sqrt(32) / 2)), PicParams(k=5)
    # ranks hold dense row shards: the single-rank reference is dense too
    base = cluster(d, kind, params, config=KernelConfig(affinity_impl=engine, storage="dense"),
                   seed=1)
    for p in (2, 3, 4, 8):
        got = cluster(d, kind, params, seed=1,
                      config=KernelConfig(p=p, virtual_ranks=True, affinity_impl=engine,
                                          storage="dense"))
        assert np.array_equal(got[0], base[0]), p
        assert np.array_equal(got[1], base[1]), p
        assert got[2].iterations_run == base[2].iterations_run
        assert np.array_equal(got[2].delta_history, base[2].delta_history), p


@pytest.mark.gpu
def test_virtual_ranks_forced_iterations_and_repeat():
    d = gaussian_blobs(2048, 16, 4, seed=3)
    kind = GaussianRbf(2.0)
    params = PicParams(k=4, epsilon=5e-324, max_iterations=9)
    base = cluster(d, kind, params, config=KernelConfig(storage="dense"))
    cfg = KernelConfig(p=4, virtual_ranks=True, storage="dense")
    a = cluster(d, kind, params, config=cfg)
    b = cluster(d, kind, params, config=cfg)   # second run: epochs keep increasing
    for r in (a, b):
        assert r[2].iterations_run == 9 and not r[2].converged
        assert np.array_equal(r[1], base[1])


@pytest.mark.gpu
def test_virtual_ranks_zero_degree():
    pts = np.array([[0.0], [0.05], [0.1], [100.0], [0.2], [0.3]])
    from paper_1604_02700_b200 import DataSet

    with pytest.raises(errors.ZeroDegree) as e:
        cluster(DataSet(pts), GaussianRbf(1.0), PicParams(k=2),
                config=KernelConfig(p=3, virtual_ranks=True))
    assert e.value.index == 3


@pytest.mark.gpu
def test_two_processes_one_device_ipc():
    """Real ranks (torchrun, 2 processes) sharing one GPU through CUDA IPC."""
    script = ROOT / "tests" / "dist_worker.py"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + os.getpid() % 300),
           str(script)]
    env = dict(os.environ, GPIC_SAME_DEVICE="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "RANKS_AGREE True" in res.stdout and "MATCHES_SINGLE True" in res.stdout


@pytest.mark.gpu
def test_matrix_free_item_shards_match_single_rank():
    """Matrix-free item shards: the pruned symmetric pass's kept items split
    across P ranks by tile count, partial y summed in rank order. Same labels
    and iteration count as one rank, embedding within 1e-6 relative L1 (only
    the summation grouping changes), deterministic across repeats; forced
    iterations too."""
    d = gaussian_blobs(9000, 64, 6, seed=8)
    kind, params = GaussianRbf(4.0), PicParams(k=6)
    single = cluster(d, kind, params, config=KernelConfig(storage="none"), seed=3)
    for p in (2, 3, 8):
        cfg = KernelConfig(p=p, virtual_ranks=True, storage="none")
        a = cluster(d, kind, params, config=cfg, seed=3)
        b = cluster(d, kind, params, config=cfg, seed=3)
        assert np.array_equal(a[0], single[0]), p
        assert a[2].iterations_run == single[2].iterations_run, p
        assert np.abs(a[1] - single[1]).sum() / np.abs(single[1]).sum() <= 1e-6, p
        assert np.array_equal(a[1], b[1]), p
    forced = PicParams(k=6, epsilon=5e-324, max_iterations=6)
    f1 = cluster(d, kind, forced, config=KernelConfig(storage="none"), seed=3)
    f4 = cluster(d, kind, forced, config=KernelConfig(p=4, virtual_ranks=True, storage="none"), seed=3)
    assert f4[2].iterations_run == 6
    assert np.abs(f4[1] - f1[1]).sum() / np.abs(f1[1]).sum() <= 1e-6


@pytest.mark.gpu
def test_matrix_free_virtual_ranks_bitwise(monkeypatch):
    # without pruning the matrix-free shards are row bands (full-square
    # pass), bitwise P-invariant; one rank runs the upper-triangle pass
    monkeypatch.setenv("GPIC_PRUNE", "0")
    d = gaussian_blobs(2600, 64, 4, seed=8)
    kind, params = GaussianRbf(4.0), PicParams(k=4)
    single = cluster(d, kind, params, config=KernelConfig(storage="none"), seed=3)
    base = cluster(d, kind, params, seed=3,
                   config=KernelConfig(p=2, virtual_ranks=True, storage="none"))
    assert np.array_equal(single[0], base[0])
    assert np.abs(single[1] - base[1]).sum() / np.abs(base[1]).sum() <= 1e-6
    for p in (3, 5):
        got = cluster(d, kind, params, seed=3,
                      config=KernelConfig(p=p, virtual_ranks=True, storage="none"))
        assert np.array_equal(got[0], base[0]) and np.array_equal(got[1], base[1]), p
        assert np.array_equal(got[2].delta_history, base[2].delta_history)


@pytest.mark.gpu
def test_packed_shards_match_single_rank():
    """Symmetric packed storage across ranks (super-row shards, partial y
    summed in rank order): same labels and iteration count as one rank,
    embedding within 1e-6 relative L1 (only the summation grouping changes),
    deterministic across repeats, forced iterations and a second run."""
    d = gaussian_blobs(6000, 64, 6, seed=5)
    kind, params = GaussianRbf(4.0), PicParams(k=6)
    single = cluster(d, kind, params, config=KernelConfig(), seed=4)
    for p in (2, 3, 5):
        cfg = KernelConfig(p=p, virtual_ranks=True)
        a = cluster(d, kind, params, config=cfg, seed=4)
        b = cluster(d, kind, params, config=cfg, seed=4)
        assert np.array_equal(a[0], single[0]), p
        assert a[2].iterations_run == single[2].iterations_run, p
        assert np.abs(a[1] - single[1]).sum() / np.abs(single[1]).sum() <= 1e-6, p
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0]), p
    forced = PicParams(k=6, epsilon=5e-324, max_iterations=8)
    f1 = cluster(d, kind, forced, config=KernelConfig(), seed=4)
    f3 = cluster(d, kind, forced, config=KernelConfig(p=3, virtual_ranks=True), seed=4)
    assert f3[2].iterations_run == 8 and not f3[2].converged
    assert np.abs(f3[1] - f1[1]).sum() / np.abs(f1[1]).sum() <= 1e-6


@pytest.mark.gpu
def test_packed_shard_ranges_cover_the_triangle():
    """gpic_packed_shard_range: 512-row aligned, contiguous, covering, and
    balanced by stored tiles; too many ranks for the rows is rejected."""
    from paper_1604_02700_b200 import _lib
    import ctypes as C

    L = _lib.lib()
    for n, P in ((6000, 2), (6000, 5), (100000, 8), (1025, 2)):
        lo_prev, tiles = 0, []
        for r in range(P):
            lo, hi = C.c_int64(), C.c_int64()
            assert L.gpic_packed_shard_range(n, P, r, C.byref(lo), C.byref(hi)) == 0
            assert lo.value == lo_prev and lo.value % 512 == 0 and hi.value > lo.value
            tiles.append(L.gpic_packed_shard_tiles(n, lo.value, hi.value))
            lo_prev = hi.value
        assert lo_prev == n
        assert sum(tiles) == L.gpic_packed_tiles(n)
        if n >= 100000:
            assert max(tiles) / min(tiles) < 1.15, tiles  # 512-row granularity
    lo, hi = C.c_int64(), C.c_int64()
    assert L.gpic_packed_shard_range(1000, 3, 0, C.byref(lo), C.byref(hi)) != 0


@pytest.mark.gpu
@pytest.mark.parametrize("m,kind_name", [(100, "rbf"), (20, "cosine")])
def test_packed_shards_other_shapes_and_kinds(m, kind_name):
    """Packed shards with 128-row affinity blocks (d > 64) and with the
    cosine kind: labels and iterations equal to one rank."""
    from paper_1604_02700_b200 import Cosine

    d = gaussian_blobs(5000, m, 4, seed=11)
    kind = GaussianRbf(float(np.sqrt(m) / 2)) if kind_name == "rbf" else Cosine()
    params = PicParams(k=4)
    single = cluster(d, kind, params, config=KernelConfig(), seed=2)
    for p in (2, 4):
        got = cluster(d, kind, params, config=KernelConfig(p=p, virtual_ranks=True), seed=2)
        assert np.array_equal(got[0], single[0]), p
        assert got[2].iterations_run == single[2].iterations_run, p
        assert np.abs(got[1] - single[1]).sum() / np.abs(single[1]).sum() <= 1e-6, p


@pytest.mark.gpu
@pytest.mark.parametrize("storage", ["packed", "none"])
def test_reduce_scatter_exchange_matches_all_to_all(monkeypatch, storage):
    """The slotted shards' two exchanges (every partial to every rank, or
    reduce-scatter of the partials + all-gather of the y slices) add the
    same terms in the same rank order: bitwise-equal embeddings, labels and
    delta histories, for P = 2..5 virtual ranks."""
    d = gaussian_blobs(7000, 64, 5, seed=12)
    kind, params = GaussianRbf(4.0), PicParams(k=5)
    for p in (2, 3, 5):
        cfg = KernelConfig(p=p, virtual_ranks=True, storage=storage)
        monkeypatch.setenv("GPIC_EXCHANGE", "bcast")
        a = cluster(d, kind, params, config=cfg, seed=2)
        monkeypatch.setenv("GPIC_EXCHANGE", "rs")
        b = cluster(d, kind, params, config=cfg, seed=2)
        assert np.array_equal(a[0], b[0]), p
        assert np.array_equal(a[1], b[1]), p
        assert np.array_equal(a[2].delta_history, b[2].delta_history), p


@pytest.mark.gpu
def test_work_balanced_packed_shard_ranges():
    """gpic_packed_shard_ranges_pruned: 512-aligned, strictly increasing,
    covering [0, n), every rank a super-row, identical on repeat (every rank
    computes it independently), and balanced by kept tensor units."""
    import ctypes as C

    import torch

    from paper_1604_02700_b200 import _lib, gpu

    L = _lib.lib()
    d = gaussian_blobs(20000, 64, 8, seed=3)
    dev = torch.device("cuda", 0)
    prep = gpu.prepare_points(torch.from_numpy(d.points).to(dev), dev, _lib.KIND_RBF)
    scratch = torch.empty(int(L.gpic_prune_scratch_bytes(d.n, prep.d)), dtype=torch.uint8,
                          device=dev)
    st = gpu._stream(dev)
    for P in (2, 3, 8):
        got = []
        for _ in range(2):
            b = (C.c_int64 * (P + 1))()
            assert L.gpic_packed_shard_ranges_pruned(gpu._ptr(prep.xlo), gpu._ptr(prep.work),
                                                     d.n, prep.d, 4.0, P, gpu._ptr(scratch), b,
                                                     st) == _lib.GPIC_OK
            got.append(list(b))
        assert got[0] == got[1]
        b = got[0]
        assert b[0] == 0 and b[-1] == d.n
        assert all(x % 512 == 0 for x in b[:-1])
        assert all(b[r + 1] > b[r] for r in range(P))
    b = (C.c_int64 * 42)()  # 40 super-rows: 41 ranks are too many
    assert L.gpic_packed_shard_ranges_pruned(gpu._ptr(prep.xlo), gpu._ptr(prep.work), d.n,
                                             prep.d, 4.0, 41, gpu._ptr(scratch), b, st) != 0


@pytest.mark.gpu
@pytest.mark.parametrize("storage", ["dense", "packed"])
def test_virtual_ranks_honour_the_start_vector(storage):
    """v0 = 'uniform' and an explicit start vector on p > 1 ranks give the
    single-rank run's embedding (parallel.py:210-214 honours v0 for any p):
    bitwise on dense row shards, within 1e-6 relative L1 on packed shards
    (partial y summed in rank order); a degree start differs from both."""
    d = gaussian_blobs(3000, 32, 5, seed=2)
    kind = GaussianRbf(float(np.sqrt(32) / 2))
    rng = np.random.default_rng(7)
    w = rng.uniform(0.5, 1.5, d.n)
    for v0 in ("uniform", w / w.sum()):
        params = PicParams(k=5, epsilon=5e-324, max_iterations=5, v0=v0)
        base = cluster(d, kind, params, config=KernelConfig(storage=storage), seed=1)
        deg = cluster(d, kind, PicParams(k=5, epsilon=5e-324, max_iterations=5),
                      config=KernelConfig(storage=storage), seed=1)
        assert not np.array_equal(base[1], deg[1])
        for p in (2, 3):
            got = cluster(d, kind, params, seed=1,
                          config=KernelConfig(p=p, virtual_ranks=True, storage=storage))
            assert got[2].iterations_run == 5
            if storage == "dense":
                assert np.array_equal(got[1], base[1]), (p, storage)
            else:
                assert np.abs(got[1] - base[1]).sum() / np.abs(base[1]).sum() <= 1e-6, (p, storage)
