"""Multi-rank host logic of paper_1506_04448_b200.distributed on CPU (gloo,
world_size 2): slice partitioning, sketch all-reduce, and the split-restart
RTPM with all-gather argmax + broadcast, with the oracle as the compute backend
(test-only). The GPU backend plugs into the same functions."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle_py as O
from paper_1506_04448_b200.distributed import (distributed_rtpm, equal_work_slices, select_best,
                                               simplex_rows_work, split_range)


def test_equal_work_slices_cover_and_balance():
    for n, w in [(400, 8), (10, 3), (5, 8), (1000, 2)]:
        sl = equal_work_slices(n, w)
        assert len(sl) == w and sl[0][0] == 0 and sl[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        if n >= 8 * w:
            work = [sum(simplex_rows_work(n, i) for i in range(a, b)) for a, b in sl]
            assert max(work) / min(work) < 1.2


def test_split_range_and_selection_ties():
    assert [split_range(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert select_best([1.0, 2.0, 2.0], [5, 3, 7]) == (2.0, 3)  # lowest tau wins a tie
    assert select_best([2.0, 2.0], [9, 2]) == (2.0, 2)


class OracleCompute:
    """Test-only backend: the CPU oracle stands in for the GPU set."""

    def __init__(self, n, b, B, seed, T):
        self.s = O.SymSet(n, b, B, seed)
        self.s.accumulate_dense(T, True)
        self._n = n

    def n(self):
        return self._n

    def restarts(self, U0, T_iters, tol):
        finals = []
        vals = []
        for u in U0:
            u = u.copy()
            for _ in range(T_iters):
                u = self.s.ivv(u)
                u /= np.linalg.norm(u)
            finals.append(u)
            vals.append(self.s.vvv(u))
        return np.array(finals), np.array(vals)

    def deflate(self, v, alpha):
        self.s.add_scaled_rank1(v, alpha)

    def inits(self, seed, c, tau0, L):
        return np.array([O.unit_sphere(O.derive_seed(seed, 0x31, c, tau0 + t), self._n) for t in range(L)])


def _planted(n, k, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.normal(size=(n, k)))
    lam = 1 + rng.uniform(size=k)
    return np.einsum("r,ir,jr,kr->ijk", lam, Q, Q, Q)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, b, B = 10, 256, 4
    T = _planted(n, 3, 1)
    # sharded build: slice sketches summed == whole sketch
    i0, i1 = equal_work_slices(n, world)[rank]
    Ts = T.copy()
    Ts[:i0] = 0
    Ts[i1:] = 0
    part = O.SymSet(n, b, B, 7)
    part.accumulate_dense(Ts, True)
    d = torch.from_numpy(part.data().view(np.float64).copy())
    dist.all_reduce(d)
    # split-restart RTPM
    comp = OracleCompute(n, b, B, 7, T)
    res = distributed_rtpm(comp, k=2, L=5, T_iters=6, seed=3, tol=1e-12)
    if rank == 0:
        out.put((d.numpy().copy(), res.lambda_, res.V, res.best_tau))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_build_and_rtpm():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    d, lam, V, taus = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    n, b, B = 10, 256, 4
    T = _planted(n, 3, 1)
    whole = O.SymSet(n, b, B, 7)
    whole.accumulate_dense(T, True)
    ref = whole.data().view(np.float64).reshape(-1)
    assert np.max(np.abs(d.reshape(-1) - ref)) <= 1e-12 * np.max(np.abs(ref))
    lam_o, V_o, bt_o = whole.rtpm(2, 5, 6, seed=3)
    assert np.array_equal(taus, bt_o)
    assert np.allclose(lam, lam_o, rtol=1e-12, atol=0)
    assert np.allclose(V, V_o, rtol=0, atol=1e-12)


def _lda_worker(rank, world, port, out):
    import torch.distributed as dist

    from lda_fixtures import synthetic_corpus
    from paper_1506_04448_b200.distributed import lda_shard_globals

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V = 40
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=4, D=90, mean_len=6, seed=3)
    cut = 37
    if rank == 0:
        dp_, w_, c_ = doc_ptr[:cut + 1], word[:doc_ptr[cut]], count[:doc_ptr[cut]]
    else:
        dp_, w_, c_ = doc_ptr[cut:] - doc_ptr[cut], word[doc_ptr[cut]:], count[doc_ptr[cut]:]
    g_used, g_m1, _, _ = lda_shard_globals(V, dp_, w_, c_)
    if rank == 0:
        out.put((g_used, g_m1))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_lda_shard_globals():
    """Each rank passes its document shard; both see the corpus-wide document count and
    averaged M1 (compute_m1, lda.cpp:88-100) of the whole corpus."""
    from lda_fixtures import synthetic_corpus

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_lda_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    g_used, g_m1 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    V = 40
    doc_ptr, word, count, _ = synthetic_corpus(V=V, k=4, D=90, mean_len=6, seed=3)
    m1 = O.lda_compute_m1(V, doc_ptr, word, count)
    tot = np.array([count[doc_ptr[d]:doc_ptr[d + 1]].sum() for d in range(doc_ptr.size - 1)])
    assert g_used == int(np.sum(tot >= 3))
    assert np.max(np.abs(g_m1 - m1)) <= 1e-15
