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


def _worker(rank, world, port, herm, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1203_4031_b200.distributed import feast_he_distributed, feast_sy_distributed
    a, b, lo, hi = _problem(herm)
    fn = feast_he_distributed if herm else feast_sy_distributed
    r = fn(a, lo, hi, 20, b=b)
    out[rank] = (int(r.info), int(r.m), int(r.loop), r.e[:r.m].copy(), r.res[:r.m].copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("herm", [False, True])
def test_two_ranks_match_single_process(herm):
    import paper_1203_4031_b200 as fb
    a, b, lo, hi = _problem(herm)
    one = (fb.feast_he if herm else fb.feast_sy)(a, lo, hi, 20, b=b)
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _port(), herm, out), nprocs=2, join=True)
    s = max(abs(lo), abs(hi))
    for rank in range(2):
        info, m, loop, e, res = out[rank]
        assert info == one.info == 0 and m == one.m
        assert abs(loop - one.loop) <= 1
        assert np.abs(e - one.e[:one.m]).max() <= 1e-10 * s
        assert res.max() <= 1e-10
    assert np.array_equal(out[0][3], out[1][3])   # replicated reduced step: ranks agree bit for bit
