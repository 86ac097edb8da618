"""Row-sharded PIC over P ranks.

Rank r owns the contiguous rows [r*n//P, (r+1)*n//P) of A — the reference's
row-range plan (plan_rows, parallel.py:90-98) balanced so every rank is
non-empty. Each rank builds its own row block with no communication; the
degree slices are all-gathered once and the y slices every iteration, both
by P2P stores fused into the producing kernels (csrc/comm.cu). Every rank
then runs the (bitwise identical) tau / normalise / stop tail and the
k-means on the full embedding, so all ranks return the same result.

Two launch modes share that code path:

* real ranks: one process per GPU under torch.distributed (torchrun); the
  host only exchanges the 64-byte CUDA-IPC handles of the exchange buffers
  (all_gather_object, any backend) once per run;
* virtual ranks (KernelConfig(p=P, virtual_ranks=True)): all P shards in
  this process on one device — how the multi-rank path is tested on a
  single B200; results are bitwise equal to p=1.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .errors import DeviceError, InvalidSpec, ZeroDegree
from .params import KMeansParams, PicTrace


def shard_ranges(n: int, p: int):
    """Balanced contiguous row ranges, all non-empty (n >= p)."""
    if p < 1 or p > _lib.MAX_RANKS:
        raise InvalidSpec(f"the sharded engine runs 1..{_lib.MAX_RANKS} ranks, got {p}")
    if n < p:
        raise InvalidSpec(f"cannot shard n={n} points over {p} ranks")
    return [(r * n // p, (r + 1) * n // p) for r in range(p)]


def dist_context():
    """(rank, world_size) of an initialised torch.distributed job, else (0, 1)."""
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def exchange_handles(mine: bytes, world: int) -> list[bytes]:
    """All-gather the per-rank IPC handles (host plumbing, once per run)."""
    if world == 1:
        return [mine]
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, bytes(mine))
    return [bytes(h) for h in out]


def assemble_handles(handles: list[bytes]) -> bytes:
    if any(len(h) != _lib.IPC_HANDLE_BYTES for h in handles):
        raise DeviceError("malformed CUDA IPC handle from a peer rank")
    return b"".join(handles)


class Comm:
    """Owns a gpic_comm (exchange buffers of this process's shards)."""

    def __init__(self, n: int, p: int, virtual: bool, rank: int = 0):
        self.L = _lib.lib()
        self.ptr = C.c_void_p()
        if virtual:
            _lib.check(self.L.gpic_comm_create_virtual(p, n, C.byref(self.ptr)))
        else:
            handle = (C.c_uint8 * _lib.IPC_HANDLE_BYTES)()
            _lib.check(self.L.gpic_comm_create(p, rank, n, C.byref(self.ptr), handle))
            allh = assemble_handles(exchange_handles(bytes(handle), p))
            buf = (C.c_uint8 * len(allh)).from_buffer_copy(allh)
            _lib.check(self.L.gpic_comm_open(self.ptr, buf))

    def close(self):
        if self.ptr:
            self.L.gpic_comm_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class ShardedRunner:
    """The sharded pipeline for a fixed (n, P): exchange buffers live across runs.

    ``run(dataset_or_device_points, sigma, params, seed)`` returns device
    tensors (labels, v) and the PicTrace; the comm (CUDA-IPC mappings of the
    peers' exchange buffers) is set up once in the constructor, outside any
    timed region.
    """

    def __init__(self, n: int, config):
        from . import gpu

        self.gpu = gpu
        self.n = n
        self.config = config
        P = config.p
        self.ranges = shard_ranges(n, P)
        if config.virtual_ranks:
            self.locals = list(range(P))
            self.rank = 0
        else:
            self.rank, world = dist_context()
            if world != P:
                raise InvalidSpec(
                    f"KernelConfig(p={P}) without virtual_ranks needs a torch.distributed job of "
                    f"{P} ranks (one per GPU); world size is {world}"
                )
            self.locals = [self.rank]
        self.dev = gpu._device(config)
        # packed symmetric shards (tcgen05 engine) unless dense rows were asked
        # for (dense row shards are bitwise independent of P)
        self.packed = config.storage == "packed" and config.affinity_impl == "tc"
        if self.packed:
            L = _lib.lib()
            self.packed_ranges = []
            for r in range(P):
                lo, hi = C.c_int64(), C.c_int64()
                if L.gpic_packed_shard_range(n, P, r, C.byref(lo), C.byref(hi)) != _lib.GPIC_OK:
                    self.packed = False  # fewer 512-row super-rows than ranks: dense rows
                    break
                self.packed_ranges.append((lo.value, hi.value))
        self.comm = Comm(n, P, config.virtual_ranks, self.rank)

    def close(self):
        self.comm.close()

    def run(self, points, kind, params, seed: int = 0, v0=None):
        gpu = self.gpu
        torch = gpu._torch()
        n, dev, cfg = self.n, self.dev, self.config
        st = gpu._stream(dev)
        code, sigma = gpu._check_kind(kind)
        prep = gpu.prepare_points(points, dev, code)
        # the engine routing of gpic_cluster (capi.cu effective_engine): d > 192,
        # RBF with d <= 8 and RBF with a large spread against sigma run on the
        # SIMT engine, here with dense row shards
        packed = (self.packed and int(_lib.lib().gpic_feature_pitch(prep.d)) <= 192
                  and prep.engine(sigma, "tc", _lib.STORAGE_PACKED) == "tc")
        nl = len(self.locals)
        shards = (_lib.Shard * nl)()
        keep = []  # device buffers referenced by the shard structs
        L = _lib.lib()
        # matrix-free item shards: the pruned symmetric pass's kept items split
        # across the ranks by tile count (RBF, d > 8 on the tensor engine);
        # other matrix-free inputs fall back to row bands (full-square rows)
        item_shards = (cfg.storage == "none" and cfg.affinity_impl == "tc"
                       and code == _lib.KIND_RBF and prep.d > 8
                       and prep.engine(sigma, "tc", _lib.STORAGE_NONE) == "tc")
        if item_shards:
            P = cfg.p
            for i, r in enumerate(self.locals):
                deg = torch.empty(n, dtype=torch.float64, device=dev)
                scratch = torch.empty(int(L.gpic_mf_shard_scratch_bytes(n, prep.d)),
                                      dtype=torch.uint8, device=dev)
                rc = L.gpic_mf_shard_build(gpu._ptr(prep.xhi), gpu._ptr(prep.xlo),
                                           gpu._ptr(prep.sqn), gpu._ptr(prep.work), n, prep.d,
                                           sigma, P, r, gpu._ptr(deg), gpu._ptr(scratch), st)
                if rc == _lib.GPIC_E_UNSUPPORTED:  # pruning disabled (GPIC_PRUNE=0 ...)
                    item_shards = False
                    keep.clear()
                    break
                _lib.check(rc)
                keep += [deg, scratch]
                shards[i] = _lib.Shard(None, 1, deg.data_ptr(), 0, n, _lib.STORAGE_NONE, prep.d,
                                       prep.xhi.data_ptr(), prep.xlo.data_ptr(),
                                       prep.sqn.data_ptr(), sigma, code, scratch.data_ptr(),
                                       prep.x.data_ptr())
        if item_shards:
            pass
        elif cfg.storage == "none":
            if cfg.affinity_impl != "tc":
                raise InvalidSpec("matrix-free storage runs on the tcgen05 engine")
            ones = torch.empty(int(L.gpic_vector_pitch(n)), dtype=torch.float32, device=dev)
            for i, r in enumerate(self.locals):
                lo, hi = self.ranges[r]
                deg = torch.empty(hi - lo, dtype=torch.float64, device=dev)
                ypart = torch.empty(int(L.gpic_mf_ypart_doubles(n, prep.d, hi - lo)),
                                    dtype=torch.float64, device=dev)
                _lib.check(L.gpic_mf_degrees(gpu._ptr(prep.xhi), gpu._ptr(prep.xlo),
                                             gpu._ptr(prep.sqn), n, prep.d, lo, hi, sigma, code,
                                             gpu._ptr(ones), gpu._ptr(ypart), gpu._ptr(deg), st))
                keep += [deg, ypart]
                shards[i] = _lib.Shard(None, 0, deg.data_ptr(), lo, hi - lo, _lib.STORAGE_NONE,
                                       prep.d, prep.xhi.data_ptr(), prep.xlo.data_ptr(),
                                       prep.sqn.data_ptr(), sigma, code, ypart.data_ptr(),
                                       prep.x.data_ptr())
        elif packed:
            # symmetric packed shards: upper-triangle tiles of the rank's
            # 512-row super-rows, partial degrees summed across ranks; rows
            # balanced by the pruning mask's kept units (the same on every
            # rank) when the RBF kind prunes, else by triangle tiles
            ranges = self.packed_ranges
            if code == _lib.KIND_RBF and os.environ.get("GPIC_SHARD_BALANCE", "1") != "0":
                scratch = torch.empty(int(L.gpic_prune_scratch_bytes(n, prep.d)),
                                      dtype=torch.uint8, device=dev)
                bounds = (C.c_int64 * (cfg.p + 1))()
                _lib.check(L.gpic_packed_shard_ranges_pruned(
                    gpu._ptr(prep.xlo), gpu._ptr(prep.work), n, prep.d, sigma, cfg.p,
                    gpu._ptr(scratch), bounds, st))
                ranges = [(bounds[r], bounds[r + 1]) for r in range(cfg.p)]
            for i, r in enumerate(self.locals):
                lo, hi = ranges[r]
                ntile = int(L.gpic_packed_shard_tiles(n, lo, hi))
                tiles = torch.empty(ntile * 128 * 128, dtype=torch.float32, device=dev)
                deg = torch.empty(n, dtype=torch.float64, device=dev)
                scratch = torch.empty(int(L.gpic_packed_shard_scratch_bytes(n, lo, hi)),
                                      dtype=torch.uint8, device=dev)
                _lib.check(L.gpic_packed_shard_build(
                    gpu._ptr(prep.xhi), gpu._ptr(prep.xlo), gpu._ptr(prep.sqn), n, prep.d, lo, hi,
                    sigma, code, gpu._ptr(tiles), gpu._ptr(deg), gpu._ptr(scratch),
                    gpu._ptr(prep.work), st))
                keep += [tiles, deg, scratch]
                shards[i] = _lib.Shard(tiles.data_ptr(), 0, deg.data_ptr(), lo, hi - lo,
                                       _lib.STORAGE_PACKED, prep.d, None, None, None, sigma, code,
                                       scratch.data_ptr(), prep.x.data_ptr())
        else:
            for i, r in enumerate(self.locals):
                lo, hi = self.ranges[r]
                blk = gpu.affinity_rows(prep, lo, hi, sigma, cfg.affinity_impl)
                keep.append(blk)
                shards[i] = _lib.Shard(blk.a.data_ptr(), blk.lda, blk.deg.data_ptr(), lo, hi - lo,
                                       _lib.STORAGE_DENSE, prep.d, None, None, None, sigma, code,
                                       None, prep.x.data_ptr())
        T = params.max_iterations
        eps = params.resolved_epsilon(n)
        hist = torch.zeros(nl * T, dtype=torch.float64, device=dev)
        vout = torch.empty(nl * n, dtype=torch.float64, device=dev)
        ctls = (_lib.Ctl * nl)()
        L = self.comm.L
        keep.append(prep.x)
        rc = L.gpic_comm_gather_degrees(self.comm.ptr, shards, nl, None, st)
        if rc == _lib.GPIC_E_ZERO_DEGREE:
            raise ZeroDegree(int(_lib.last_error().split()[1]))
        _lib.check(rc)
        if v0 is None:
            v0 = gpu.start_vector(params.v0, n)
        v0_t = None if v0 is None else torch.from_numpy(np.ascontiguousarray(v0)).to(dev)
        rc = L.gpic_comm_iterate(self.comm.ptr, shards, nl, eps, T, gpu._ptr(v0_t),
                                 gpu._ptr(hist), gpu._ptr(vout), ctls, st)
        if rc != _lib.GPIC_OK:
            bad = next((c for c in ctls if c.status != _lib.GPIC_OK), None)
            _lib.raise_for(rc, bad)
        # every shard holds the same embedding; local shard 0 speaks for the rank
        h = ctls[0]
        for c in ctls[1:]:
            if c.iter != h.iter or c.converged != h.converged:
                raise DeviceError("ranks disagree on the stop decision")
        v = vout[:n]
        labels = gpu.kmeans_1d(v, KMeansParams(k=params.k, seed=seed), cfg)
        it = int(h.iter)
        return labels, v, PicTrace(it, hist[:it].cpu().numpy(), bool(h.converged))


def cluster(d, kind, params, config, seed, v0=None):
    """Sharded counterpart of gpu.cluster (same return contract); ``v0`` as
    gpu.start_vector returns it (None: the degree start)."""
    from . import gpu

    gpu._check_kind(kind)
    runner = ShardedRunner(d.n, config)
    try:
        labels, v, trace = runner.run(d, kind, params, seed, v0=v0)
        return labels.cpu().numpy(), v.cpu().numpy(), trace
    finally:
        runner.close()


def all_ranks_agree(labels: np.ndarray, v: np.ndarray) -> bool:
    """Host check (real ranks): every rank returned bit-identical results."""
    rank, world = dist_context()
    if world == 1:
        return True
    import hashlib

    import torch.distributed as dist

    digest = hashlib.sha256(labels.tobytes() + v.tobytes()).hexdigest()
    out = [None] * world
    dist.all_gather_object(out, digest)
    return all(x == out[0] for x in out)
