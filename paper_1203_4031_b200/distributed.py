"""Contour-point parallelism over GPUs (FEAST-MPI's second level).

One process per GPU (torch.distributed, NCCL over NVLink).  Every rank holds
A and B, factorizes and solves only its own shifts (point k -> rank k mod G,
perfectly balanced for Ne in {8, 16} and G in {1, 2, 4, 8}) and accumulates
a partial Q; one all-reduce(sum) of Q per refinement pass combines them.  The
projection, reduced eigensolve and Ritz step are then replicated on every
rank (deterministic, identical inputs), so all ranks leave the pass with the
same X and the next pass needs no further exchange.  This is new relative to
the reference (threads only, _driver.py:46-54); SURVEY.md §8(e).
"""

from __future__ import annotations


def shard_points(ne: int, rank: int, world: int):
    """Contour indices served by ``rank`` (round robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return [k for k in range(ne) if k % world == rank]


def make_q_reduce(group=None):
    """all-reduce(sum) of the partial subspace over ``group``.

    The whole planar buffer is reduced (contiguous; columns past the current
    M0 are never read), which keeps it a single NCCL call per pass."""
    import torch.distributed as dist

    def reduce(Q):
        dist.all_reduce(Q.t, op=dist.ReduceOp.SUM, group=group)

    return reduce


def _engine_kwargs(fpm, group):
    import torch.distributed as dist
    from .params import feastinit
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ne = (fpm or feastinit()).slot(2)
    return {"points": shard_points(ne, rank, world), "q_reduce": make_q_reduce(group)}


def feast_sy_distributed(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None,
                         group=None):
    """feast_sy with its contour points sharded over the ranks of ``group``."""
    from .dense import _dense_driver
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, False,
                         engine_kwargs=_engine_kwargs(fpm, group))


def feast_he_distributed(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None,
                         group=None):
    """feast_he with its contour points sharded over the ranks of ``group``."""
    from .dense import _dense_driver
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, True,
                         engine_kwargs=_engine_kwargs(fpm, group))
