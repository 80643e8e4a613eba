"""Multi-GPU coordination for the sketch path, one process per GPU
over torch.distributed (NCCL on B200; gloo in the CPU tests).

Where the path shards:
  * dense build — rank r sketches its equal-work i-slice of the sorted-triple loop
    (sketch.cpp:328-343); sketches are linear, so one all-reduce(sum) of the
    B x b complex data finishes the build;
  * factored / moment build — samples are split across ranks, same all-reduce;
  * LDA whitened moment — documents are split across ranks; the per-document terms are
    linear, the corpus-wide M1 and document count are all-reduced first (sums of the
    shards' partials), each rank sketches its shard with those globals, and one
    all-reduce of the B x b data completes sketch_whitened_m3 (lda.cpp:145-226);
  * RTPM — every rank holds the full sketch, the L restarts of a component are
    split across ranks; selection is an all-gather of (value, global tau) with the
    reference's strict '>' over ascending tau (decompose.cpp:105-109), the owner
    broadcasts v, and every rank applies the identical deflation.

The compute backend is passed in (``ShardCompute``): the product uses the GPU set
(:class:`GpuShardCompute`); tests may plug a CPU checker to exercise the
collective logic without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Protocol, Sequence

import numpy as np


def simplex_rows_work(n: int, i: int) -> int:
    """Sorted triples (i, j, k) with i <= j <= k for a fixed i."""
    return (n - i) * (n - i + 1) // 2


def equal_work_slices(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous i-ranges [i0, i1) with about equal sorted-triple counts."""
    if world < 1:
        raise ValueError("world size must be positive")
    tot = sum(simplex_rows_work(n, i) for i in range(n))
    bounds, acc, r = [0], 0, 1
    for i in range(n):
        acc += simplex_rows_work(n, i)
        while r < world and acc >= tot * r / world:
            bounds.append(i + 1)
            r += 1
    while len(bounds) < world:
        bounds.append(n)
    bounds.append(n)
    return [(bounds[k], bounds[k + 1]) for k in range(world)]


def split_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous block [lo, hi) of `total` items for `rank`."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def select_best(values: Sequence[float], taus: Sequence[int]) -> tuple[float, int]:
    """Reference selection: strict '>' scanning tau ascending, so ties go to the
    lowest tau (decompose.cpp:101-109)."""
    order = np.argsort(np.asarray(taus), kind="stable")
    best, best_tau = -np.inf, int(taus[order[0]]) if len(taus) else 0
    for k in order:
        if values[k] > best:
            best, best_tau = float(values[k]), int(taus[k])
    return best, best_tau


class ShardCompute(Protocol):
    def n(self) -> int: ...

    def restarts(self, U0: np.ndarray, T_iters: int, tol: float) -> tuple[np.ndarray, np.ndarray]:
        """Runs T_iters normalised power steps on U0 (L, n); returns (finals, values)."""

    def deflate(self, v: np.ndarray, alpha: float) -> None: ...

    def inits(self, seed: int, c: int, tau0: int, L: int) -> np.ndarray: ...


@dataclass
class RtpmResult:
    lambda_: np.ndarray
    V: np.ndarray  # n x k
    best_tau: np.ndarray


def distributed_rtpm(compute: ShardCompute, k: int, L: int, T_iters: int, seed: int, tol: float, group=None,
                     inits: np.ndarray | None = None) -> RtpmResult:
    """robust_tpm_fast (decompose.cpp:83-115) with the L restarts split over ranks."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = compute.n()
    if k < 1 or L < 1 or T_iters < 1:
        raise ValueError("power method: k, L and T must be positive")
    if k > n:
        raise ValueError("power method: target rank exceeds tensor dimension")
    t0, t1 = split_range(L, world, rank)
    lam = np.empty(k)
    V = np.empty((n, k))
    taus = np.empty(k, dtype=np.int64)
    backend_dev = None
    if world > 1 and dist.get_backend(group) == "nccl":
        backend_dev = torch.device("cuda", torch.cuda.current_device())
    for c in range(k):
        if t1 > t0:
            U0 = inits[c, t0:t1] if inits is not None else compute.inits(seed, c, t0, t1 - t0)
            finals, values = compute.restarts(np.ascontiguousarray(U0), T_iters, tol)
            lb, lt = select_best(values, list(range(t0, t1)))
        else:
            finals, values, lb, lt = np.zeros((0, n)), np.zeros(0), -np.inf, L
        if world > 1:
            pair = torch.tensor([lb, float(lt)], dtype=torch.float64, device=backend_dev)
            gathered = [torch.empty_like(pair) for _ in range(world)]
            dist.all_gather(gathered, pair, group=group)
            vals = [float(g[0]) for g in gathered]
            tts = [int(g[1]) for g in gathered]
            best, best_tau = select_best(vals, tts)
            owner = next(r for r in range(world) if split_range(L, world, r)[0] <= best_tau < split_range(L, world, r)[1])
            v = torch.zeros(n, dtype=torch.float64, device=backend_dev)
            if rank == owner:
                v.copy_(torch.from_numpy(finals[best_tau - t0]))
            dist.broadcast(v, src=owner if group is None else dist.get_global_rank(group, owner), group=group)
            vec = v.cpu().numpy()
        else:
            best, best_tau = lb, lt
            vec = finals[best_tau - t0]
        lam[c] = best
        V[:, c] = vec
        taus[c] = best_tau
        if best != 0.0:
            compute.deflate(vec, -best)
    return RtpmResult(lam, V, taus)


def allreduce_sketch(data_tensor, group=None) -> None:
    """Sum the per-rank partial sketches (B x b complex viewed as float64)."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(data_tensor, group=group)


class GpuShardCompute:
    """ShardCompute over a device-resident SymTensorSketchSet (C-ABI calls)."""

    def __init__(self, sset):
        self.s = sset

    def n(self) -> int:
        return self.s.n()

    def restarts(self, U0, T_iters, tol):
        import ctypes as C

        from . import _lib

        L, n = U0.shape
        finals = np.empty_like(U0)
        values = np.empty(L)
        dp = C.POINTER(C.c_double)
        _lib.check(_lib.lib.skc_sym_rtpm_restarts(self.s.handle, U0.ctypes.data_as(dp), L, T_iters, float(tol),
                                                  finals.ctypes.data_as(dp), values.ctypes.data_as(dp)))
        return finals, values

    def deflate(self, v, alpha):
        self.s.add_scaled_rank1(v, alpha)

    def inits(self, seed, c, tau0, L):
        from . import power_inits

        return power_inits(seed, self.n(), 1, L, c0=c, tau0=tau0)[0]


def sharded_dense_build(sset, T, group=None, assume_symmetric: bool = True) -> None:
    """Each rank sketches its equal-work i-slice; the partial sketches are summed."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = sset.n()
    i0, i1 = equal_work_slices(n, world)[rank]
    if world > 1 and rank != 0:
        # every rank holds the same prior sketch; only rank 0 keeps it so the
        # all-reduce adds it once (accumulate semantics, sketch.cpp:315)
        sset.set_data(None, np.zeros((sset.replicates(), sset.b()), dtype=np.complex128))
    sset.accumulate_dense(T, assume_symmetric=assume_symmetric, i0=i0, i1=i1)
    if world > 1:
        ptr, nbytes = sset.data_device()
        sset.ctx.synchronize()

        class _CAI:
            __cuda_array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8", "data": (ptr, False), "version": 3}

        view = torch.as_tensor(_CAI(), device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(view, group=group)
        torch.cuda.synchronize()
        sset.bump_version()


def _allreduce_data(sset, group=None) -> None:
    import torch
    import torch.distributed as dist

    ptr, nbytes = sset.data_device()
    sset.ctx.synchronize()

    class _CAI:
        __cuda_array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8", "data": (ptr, False), "version": 3}

    view = torch.as_tensor(_CAI(), device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(view, group=group)
    torch.cuda.synchronize()
    sset.bump_version()


def sharded_moment(sset, X_local, w_local=None, group=None) -> None:
    """accumulate_moment over the samples split across ranks (each passes its own rows
    with globally normalised weights); one all-reduce of the data."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world > 1 and rank != 0:
        sset.set_data(None, np.zeros((sset.replicates(), sset.b()), dtype=np.complex128))
    sset.accumulate_moment(X_local, w_local)
    if world > 1:
        _allreduce_data(sset, group)


def lda_shard_globals(V: int, doc_ptr, word, count, group=None):
    """Corpus-wide (documents with >= 3 tokens, averaged M1) from this rank's document
    shard: local sums (lda.cpp:88-100) combined by one all-reduce. Returns
    (global_used, global_m1, local_used1, local_used3)."""
    import torch
    import torch.distributed as dist

    doc_ptr = np.asarray(doc_ptr, dtype=np.int64)
    word = np.asarray(word, dtype=np.int64)
    count = np.asarray(count, dtype=np.float64)
    D = doc_ptr.size - 1
    tot = np.add.reduceat(count, doc_ptr[:-1]) if word.size else np.zeros(D)
    tot[doc_ptr[:-1] == doc_ptr[1:]] = 0.0
    lens = np.diff(doc_ptr)
    m1 = np.zeros(V)
    doc_of = np.repeat(np.arange(D), lens)
    ok = tot[doc_of] >= 1
    np.add.at(m1, word[ok], count[ok] / tot[doc_of[ok]])
    used1 = float(np.sum(tot >= 1))
    used3 = float(np.sum(tot >= 3))
    buf = torch.from_numpy(np.concatenate([m1, [used1, used3]]))
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        buf = buf.to(_backend_device(group))  # an NCCL group reduces device tensors only
        dist.all_reduce(buf, group=group)
    g = buf.cpu().numpy()
    if g[V] <= 0:
        raise ValueError("compute_m1: no nonempty documents")
    return int(round(g[V + 1])), g[:V] / g[V], int(used1), int(used3)


def sharded_sketch_whitened_m3(sset, V: int, doc_ptr, word, count, W, alpha0: float, group=None):
    """sketch_whitened_m3 with the documents split across ranks (each passes its shard in
    CSR form); returns the corpus-wide (used, skipped) StreamStats."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    g_used, g_m1, _, _ = lda_shard_globals(V, doc_ptr, word, count, group)
    if world > 1 and rank != 0:
        sset.set_data(None, np.zeros((sset.replicates(), sset.b()), dtype=np.complex128))
    used, skipped = sset.sketch_whitened_m3_shard(V, doc_ptr, word, count, W, alpha0, g_used, g_m1, rank == 0)
    if world > 1:
        _allreduce_data(sset, group)
    import torch

    stats = torch.tensor([used, skipped], dtype=torch.int64)
    if world > 1:
        stats = stats.to(_backend_device(group))
        dist.all_reduce(stats, group=group)
    return int(stats[0]), int(stats[1])


def _backend_device(group=None):
    """Where collective buffers must live for the group's backend (cuda for NCCL)."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def process_group_replicas(n: int, b: int, B: int, master_seed: int, ctx, group=None):
    """SymReplicas over the ranks of a torch.distributed group, one GPU each: rank 0 makes
    the NCCL id in the library, torch.distributed only carries it. The returned replicas'
    collective calls (dense build, moment, LDA, RTPM) run the in-library NCCL paths of
    include/sketchcp_b200.h (exact accumulator all-reduce, device-side M1, split restarts)."""
    import torch.distributed as dist

    from . import SymReplicas, nccl_unique_id

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    uid = [nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0, group=group)
    ctx.comm_init(world, rank, uid[0])
    return SymReplicas(n, b, B, master_seed, [ctx])
