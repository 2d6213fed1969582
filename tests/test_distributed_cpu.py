"""Multi-rank host logic on CPU (gloo, world_size 2): the contour-point
sharding and the per-pass all-reduce of the partial subspace reproduce the
serial quadrature sum (kernel.py:350-361) — checked against the oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1203_4031_b200.distributed import make_q_reduce, shard_points


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ne,world", [(8, 1), (8, 2), (8, 8), (16, 8), (5, 2), (3, 4)])
def test_shard_points_partition(ne, world):
    parts = [shard_points(ne, r, world) for r in range(world)]
    flat = sorted(k for p in parts for k in p)
    assert flat == list(range(ne))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, herm, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_1203_4031_b200.device import Planar
    rng = np.random.default_rng(7)
    n, m0, ne = 30, 6, 8
    a = rng.standard_normal((n, n))
    if herm:
        a = a + 1j * rng.standard_normal((n, n))
    a = (a + a.conj().T) / 2
    y = O.start_block(42, n, m0, herm)
    nodes, w = O.gl_rule(ne)
    theta, z, w, r, _ = O.half_circle(nodes, w, -0.5, 0.5)
    dt = np.complex128 if herm else np.float64
    q = np.zeros((n, m0), dtype=dt)
    for k in shard_points(ne, rank, world):
        x = np.linalg.solve(z[k] * np.eye(n) - a, y)
        O.accumulate(q, x, w[k], r, theta[k], "hermitian-direct" if herm else "symmetric")
        if herm:
            xa = np.linalg.solve((z[k] * np.eye(n) - a).conj().T, y)
            O.accumulate(q, xa, w[k], r, theta[k], "hermitian-adjoint")
    if herm:
        t = torch.from_numpy(np.stack([q.real, q.imag]).copy())
    else:
        t = torch.from_numpy(q.copy())
    make_q_reduce()(Planar(t, herm, n, m0, m0))
    if rank == 0:
        out.put(t.numpy().copy())
    dist.destroy_process_group()


@pytest.mark.parametrize("herm", [False, True])
def test_partial_q_allreduce_matches_serial_sum(herm):
    import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, herm, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    n, m0, ne = 30, 6, 8
    a = rng.standard_normal((n, n))
    if herm:
        a = a + 1j * rng.standard_normal((n, n))
    a = (a + a.conj().T) / 2
    y = O.start_block(42, n, m0, herm)
    nodes, w = O.gl_rule(ne)
    theta, z, w, r, _ = O.half_circle(nodes, w, -0.5, 0.5)
    ref = np.zeros((n, m0), dtype=np.complex128 if herm else np.float64)
    for k in range(ne):
        x = np.linalg.solve(z[k] * np.eye(n) - a, y)
        O.accumulate(ref, x, w[k], r, theta[k], "hermitian-direct" if herm else "symmetric")
        if herm:
            xa = np.linalg.solve((z[k] * np.eye(n) - a).conj().T, y)
            O.accumulate(ref, xa, w[k], r, theta[k], "hermitian-adjoint")
    if herm:
        got = got[0] + 1j * got[1]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
