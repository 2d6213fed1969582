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

# Three levels as in FEAST-MPI: search intervals over rank
# sub-groups (feast_*_intervals), contour points over the ranks of one group
# (feast_*_distributed), and the batched GPU solves inside each rank.


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


# -- first level: several search intervals (FEAST-MPI's fpm(9) communicators) ----------

def split_ranks(world: int, nint: int):
    """Ranks serving each of ``nint`` search intervals (PAPER.md:456-462,
    1132-1160: one user communicator per interval, fpm(9)).  world >= nint:
    contiguous, balanced rank blocks; world < nint: interval i on rank
    i mod world alone."""
    if world < 1 or nint < 1:
        raise ValueError("bad world/interval count")
    if world >= nint:
        return [list(range(i * world // nint, (i + 1) * world // nint)) for i in range(nint)]
    return [[i % world] for i in range(nint)]


def feast_intervals(solve, nint: int, group=None):
    """Run ``solve(i, subgroup)`` for the intervals i = 0..nint-1 on rank
    sub-groups of ``group`` (contour points sharded inside each sub-group;
    ``subgroup`` is None when one rank serves the interval alone) and return
    the list of all nint results on every rank.  Without an initialised
    process group the intervals are solved one after the other."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [solve(i, None) for i in range(nint)]
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    blocks = split_ranks(world, nint)
    granks = dist.get_process_group_ranks(group) if group is not None else list(range(world))
    # every rank creates every sub-communicator, in the same order
    subs = [dist.new_group([granks[r] for r in b]) if len(b) > 1 else None for b in blocks]
    mine = {}
    for i, b in enumerate(blocks):
        if rank in b:
            res = solve(i, subs[i])
            if rank == b[0]:
                mine[i] = res
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    out = [None] * nint
    for part in gathered:
        for i, res in part.items():
            out[i] = res
    return out


def feast_sy_intervals(a, intervals, m0, *, uplo="F", b=None, fpm=None, options=None, group=None):
    """feast_sy over several search intervals [(emin, emax), ...] (first-level
    parallelism); ``m0`` is one subspace size or one per interval."""
    from .dense import feast_sy
    m0s = list(m0) if hasattr(m0, "__len__") else [m0] * len(intervals)

    def solve(i, sub):
        lo, hi = intervals[i]
        if sub is None:
            return feast_sy(a, lo, hi, m0s[i], uplo=uplo, b=b, fpm=fpm, options=options)
        return feast_sy_distributed(a, lo, hi, m0s[i], uplo=uplo, b=b, fpm=fpm, options=options, group=sub)

    return feast_intervals(solve, len(intervals), group)


def feast_he_intervals(a, intervals, m0, *, uplo="F", b=None, fpm=None, options=None, group=None):
    """feast_he over several search intervals (first-level parallelism)."""
    from .dense import feast_he
    m0s = list(m0) if hasattr(m0, "__len__") else [m0] * len(intervals)

    def solve(i, sub):
        lo, hi = intervals[i]
        if sub is None:
            return feast_he(a, lo, hi, m0s[i], uplo=uplo, b=b, fpm=fpm, options=options)
        return feast_he_distributed(a, lo, hi, m0s[i], uplo=uplo, b=b, fpm=fpm, options=options, group=sub)

    return feast_intervals(solve, len(intervals), group)
