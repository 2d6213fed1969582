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


@pytest.mark.parametrize("world,nint", [(1, 1), (1, 3), (2, 1), (3, 2), (8, 2), (8, 3), (2, 5), (8, 8)])
def test_split_ranks(world, nint):
    from paper_1203_4031_b200.distributed import split_ranks
    blocks = split_ranks(world, nint)
    assert len(blocks) == nint and all(blocks)
    if world >= nint:   # disjoint contiguous blocks covering every rank, balanced
        assert sorted(r for b in blocks for r in b) == list(range(world))
        assert max(map(len, blocks)) - min(map(len, blocks)) <= 1
    else:               # one rank per interval, round robin
        assert [b[0] for b in blocks] == [i % world for i in range(nint)]


def _interval_worker(rank, world, port, nint, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1203_4031_b200.distributed import feast_intervals, split_ranks

    def solve(i, sub):
        # stands in for feast_*_distributed on the sub-communicator: a collective
        # inside the sub-group (all its ranks must take part, no other rank)
        t = torch.tensor([float(rank + 1)])
        if sub is not None:
            dist.all_reduce(t, group=sub)
        return {"interval": i, "sum": float(t.item())}

    res = feast_intervals(solve, nint)
    blocks = split_ranks(world, nint)
    want = [{"interval": i, "sum": float(sum(r + 1 for r in b))} for i, b in enumerate(blocks)]
    out[rank] = int(res == want)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nint", [(2, 1), (3, 2), (4, 2), (2, 3)])
def test_feast_intervals_subgroups(world, nint):
    """First-level parallelism (fpm(9) analogue): every interval solved on its
    own rank sub-group, every rank gets every interval's result."""
    out = mp.Manager().dict()
    mp.spawn(_interval_worker, args=(world, _free_port(), nint, out), nprocs=world, join=True)
    assert [out[r] for r in range(world)] == [1] * world


@pytest.mark.parametrize("n,world", [(10, 1), (10, 3), (8192, 8), (7, 8), (4096, 2)])
def test_row_blocks_partition(n, world):
    from paper_1203_4031_b200.distributed import row_block
    blocks = [row_block(n, r, world) for r in range(world)]
    assert blocks[0][0] == 0 and blocks[-1][1] == n
    for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
        assert a1 == b0 and a0 <= a1
    sizes = [b - a for a, b in blocks]
    assert max(sizes) - min(sizes) <= 1


def _shard_worker(rank, world, port, fail_rank, out):
    """Row-sharded projection / residual / next-right-hand-side algebra of the
    multi-GPU path (kernel.py _run with rows/sum_reduce) on CPU tensors."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1203_4031_b200.distributed import make_flag_reduce, make_sum_reduce, row_block
    rng = np.random.default_rng(11)
    n, m0 = 41, 5
    a = rng.standard_normal((n, n)); a = (a + a.T) / 2
    h = rng.standard_normal((n, n)); b = np.eye(n) + 0.1 * h @ h.T / n
    q = rng.standard_normal((n, m0))
    lam = rng.standard_normal(m0)
    r0, r1 = row_block(n, rank, world)
    red = make_sum_reduce()
    # A_Q, B_Q from row blocks
    aq = torch.from_numpy(q[r0:r1].T @ (a[r0:r1] @ q))
    bq = torch.from_numpy(q[r0:r1].T @ (b[r0:r1] @ q))
    red(aq); red(bq)
    # residual sums from row blocks
    ax, bx = a[r0:r1] @ q, b[r0:r1] @ q
    sums = torch.from_numpy(np.stack([np.abs(ax - lam * bx).sum(0), np.abs(0.3 * bx).sum(0)], 1).reshape(-1).copy())
    red(sums)
    # next right-hand side: own rows, zeros elsewhere
    y = torch.zeros(n, m0, dtype=torch.float64)
    y[r0:r1] = torch.from_numpy(b[r0:r1] @ q)
    red(y)
    flag = make_flag_reduce()
    code = flag(-2 if rank == fail_rank else 0)
    out[rank] = (aq.numpy(), bq.numpy(), sums.numpy(), y.numpy(), code)
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_row_sharded_reductions_match_serial(fail_rank):
    rng = np.random.default_rng(11)
    n, m0 = 41, 5
    a = rng.standard_normal((n, n)); a = (a + a.T) / 2
    h = rng.standard_normal((n, n)); b = np.eye(n) + 0.1 * h @ h.T / n
    q = rng.standard_normal((n, m0))
    lam = rng.standard_normal(m0)
    out = mp.Manager().dict()
    mp.spawn(_shard_worker, args=(2, _free_port(), fail_rank, out), nprocs=2, join=True)
    for rank in range(2):
        aq, bq, sums, y, code = out[rank]
        assert np.allclose(aq, q.T @ a @ q, rtol=0, atol=1e-12)
        assert np.allclose(bq, q.T @ b @ q, rtol=0, atol=1e-12)
        num, den = sums[0::2], sums[1::2]
        assert np.allclose(num, np.abs(a @ q - lam * (b @ q)).sum(0), rtol=1e-13)
        assert np.allclose(den, np.abs(0.3 * (b @ q)).sum(0), rtol=1e-13)
        assert np.allclose(y, b @ q, rtol=0, atol=1e-13)
        assert code == (-2 if fail_rank >= 0 else 0)
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][2], out[1][2])
