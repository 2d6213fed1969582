"""The contour-point sharded engine with real GPU kernels: two ranks (gloo
collectives, both on cuda:0 -- a functional check of the sharding and the
per-pass Q all-reduce, not a scaling measurement; NCCL is what bench.py uses
with one GPU per rank) reproduce the single-process solve."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(herm):
    rng = np.random.default_rng(17 if herm else 16)
    n = 160
    g = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if herm else 0)
    a = (g + g.conj().T) / (2 * np.sqrt(n))
    h = rng.standard_normal((n, n))
    b = None if herm else np.eye(n) + 0.1 * h @ h.T / n
    ev = np.sort(np.linalg.eigvals(a if b is None else np.linalg.solve(b, a)).real)
    i0 = int(np.searchsorted(ev, 0.0))
    return a, b, 0.5 * (ev[i0 - 7] + ev[i0 - 6]), 0.5 * (ev[i0 + 5] + ev[i0 + 6])


def _init(rank, world, port, backend="gloo"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)


def _worker(rank, world, port, herm, shard_rows, backend, out):
    _init(rank, world, port, backend)
    from paper_1203_4031_b200.distributed import feast_he_distributed, feast_sy_distributed
    a, b, lo, hi = _problem(herm)
    fn = feast_he_distributed if herm else feast_sy_distributed
    r = fn(a, lo, hi, 20, b=b, shard_rows=shard_rows)
    out[rank] = (int(r.info), int(r.m), int(r.loop), r.e[:r.m].copy(), r.res[:r.m].copy())
    dist.destroy_process_group()


def _check_against_single(out, one, lo, hi, world=2):
    s = max(abs(lo), abs(hi))
    for rank in range(world):
        info, m, loop, e, res = out[rank]
        assert info == one.info == 0 and m == one.m
        assert abs(loop - one.loop) <= 1
        assert np.abs(e - one.e[:one.m]).max() <= 1e-10 * s
        assert res.max() <= 1e-10
    assert np.array_equal(out[0][3], out[1][3])   # replicated reduced step: ranks agree bit for bit
    assert np.array_equal(out[0][4], out[1][4])   # all-reduced residual sums: identical on every rank


@pytest.mark.parametrize("herm,shard_rows", [(False, False), (True, False), (False, True), (True, True)])
def test_two_ranks_match_single_process(herm, shard_rows):
    """Contour points over 2 ranks; shard_rows adds the row-sharded projection /
    Ritz / residual products with their all-reduces (A_Q, B_Q, residual sums,
    next right-hand side)."""
    import paper_1203_4031_b200 as fb
    a, b, lo, hi = _problem(herm)
    one = (fb.feast_he if herm else fb.feast_sy)(a, lo, hi, 20, b=b)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _port(), herm, shard_rows, "gloo", out), nprocs=2, join=True)
    _check_against_single(out, one, lo, hi)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (one NCCL rank per GPU)")
@pytest.mark.parametrize("herm", [False, True])
def test_two_ranks_nccl(herm):
    """The production path: one rank per GPU, NCCL all-reduces."""
    import paper_1203_4031_b200 as fb
    a, b, lo, hi = _problem(herm)
    one = (fb.feast_he if herm else fb.feast_sy)(a, lo, hi, 20, b=b)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _port(), herm, True, "nccl", out), nprocs=2, join=True)
    _check_against_single(out, one, lo, hi)


def _band_problem():
    rng = np.random.default_rng(23)
    n, kd = 3000, 4
    ab = np.zeros((kd + 1, n))
    ab[0] = 2.0 * (np.arange(n) / n - 0.5) + 0.1 * rng.standard_normal(n)
    for d in range(1, kd + 1):
        ab[d, : n - d] = 0.3 * rng.standard_normal(n - d)
    bb = np.zeros((2, n))
    bb[0], bb[1, : n - 1] = 4.0 / 6.0, 1.0 / 6.0
    return ab, kd, bb, 1, -0.004, 0.0041


def _band_worker(rank, world, port, out):
    _init(rank, world, port)
    from paper_1203_4031_b200.distributed import feast_sb_distributed
    ab, kd, bb, klb, lo, hi = _band_problem()
    r = feast_sb_distributed(ab, kd, lo, hi, 30, uplo="L", b=bb, klb=klb)
    out[rank] = (int(r.info), int(r.m), int(r.loop), r.e[:r.m].copy(), r.res[:r.m].copy())
    dist.destroy_process_group()


def test_two_ranks_banded_match_single_process():
    """feast_sb_distributed: each rank factors and sweeps its own shifts of the
    band (partitioned path forced by a small partition target)."""
    import paper_1203_4031_b200 as fb
    ab, kd, bb, klb, lo, hi = _band_problem()
    one = fb.feast_sb(ab, kd, lo, hi, 30, uplo="L", b=bb, klb=klb)
    assert one.info == 0 and one.m > 0
    out = mp.Manager().dict()
    mp.spawn(_band_worker, args=(2, _port(), out), nprocs=2, join=True)
    _check_against_single(out, one, lo, hi)


def _fail_worker(rank, world, port, out):
    _init(rank, world, port)
    from paper_1203_4031_b200 import dense
    from paper_1203_4031_b200._errors import SingularMatrixError
    from paper_1203_4031_b200.distributed import feast_sy_distributed
    if rank == 1:
        def boom(self, zs):
            raise SingularMatrixError("injected: zero pivot on this rank only")
        dense.DeviceDenseOps.prefactorize = boom
    a, b, lo, hi = _problem(False)
    r = feast_sy_distributed(a, lo, hi, 20, b=b)
    out[rank] = int(r.info)
    dist.destroy_process_group()


def test_failure_on_one_rank_aborts_all_ranks():
    """A singular shift on one rank: every rank returns info -2 (the abort flag
    travels through the all-reduce after the factorizations) -- no deadlock."""
    out = mp.Manager().dict()
    mp.spawn(_fail_worker, args=(2, _port(), out), nprocs=2, join=True)
    assert out[0] == out[1] == -2
