"""Contour-point parallelism over GPUs (FEAST-MPI's second level).

One process per GPU (torch.distributed, NCCL over NVLink).  Every rank holds
A and B, factorizes and solves only its own shifts (point k -> rank k mod G,
perfectly balanced for Ne in {8, 16} and G in {1, 2, 4, 8}) and accumulates
a partial Q; one all-reduce(sum) of Q per refinement pass combines them.

Dense pencils also shard the ROWS of the O(N^2 M0) products over the ranks
(SURVEY.md §8e step 3): rank r computes rows [r N/G, (r+1) N/G) of A*Q, B*Q,
A*X and B*X, the reduced matrices A_Q, B_Q are the all-reduced sums of the
row blocks' contributions (2 M0^2 entries), the residual norms likewise
(2 M0 numbers), and the next right-hand side B*X is assembled by one more
N x M0 sum.  Only the reduced eigensolve (and the N M0^2 Ritz update
X = Q Phi) stays replicated; it runs on bitwise identical inputs, so every
rank takes the same decisions (M0 shrink, convergence) without further
exchange.  Banded pencils shard the contour points only (their multiplies
are O(N kd M0), a few per cent of a pass).

A rank that fails (singular shift, out of memory) reports through a
one-integer all-reduce(min) after the factorizations and before every pass's
Q sum, so all ranks return the same negative info instead of deadlocking.

This is new relative to the reference (threads only, _driver.py:46-54).
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


def row_block(n: int, rank: int, world: int):
    """Rows [r0, r1) of the N^2 M0 products owned by ``rank`` (balanced, contiguous)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * n) // world, ((rank + 1) * n) // world


def make_q_reduce(group=None):
    """all-reduce(sum) of the partial subspace over ``group``.

    The whole planar buffer is reduced (contiguous; columns past the current
    M0 are never read), which keeps it a single NCCL call per pass."""
    import torch.distributed as dist

    def reduce(Q):
        dist.all_reduce(Q.t, op=dist.ReduceOp.SUM, group=group)

    return reduce


def make_sum_reduce(group=None):
    """all-reduce(sum) of a torch tensor in place over ``group``."""
    import torch.distributed as dist

    def reduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return reduce


def make_flag_reduce(group=None, device=None):
    """code -> min over the ranks of ``group`` (0 = fine, info < 0 = abort): one
    int64 all-reduce.  ``device``: where the flag lives (NCCL: the rank's GPU)."""
    import torch
    import torch.distributed as dist

    def reduce(code):
        t = torch.tensor([int(code)], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        return int(t.item())

    return reduce


def _flag_device(group):
    import torch
    import torch.distributed as dist
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None


def _engine_kwargs(fpm, group, n=None, rows=True):
    import torch.distributed as dist
    from .params import FeastParams, feastinit
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    fpm = FeastParams.coerce(fpm) if fpm is not None else feastinit()
    kw = {"points": shard_points(fpm.slot(2), rank, world), "q_reduce": make_q_reduce(group),
          "flag_reduce": make_flag_reduce(group, _flag_device(group))}
    if rows and n is not None and world > 1:
        kw["rows"] = row_block(int(n), rank, world)
        kw["sum_reduce"] = make_sum_reduce(group)
    return fpm, kw


def _order(a):
    shp = a.shape if hasattr(a, "shape") else (getattr(a, "rows", 0),)
    return shp[0] if len(shp) else 0


def feast_sy_distributed(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None,
                         group=None, shard_rows=True):
    """feast_sy with its contour points (and the rows of its N^2 M0 products)
    sharded over the ranks of ``group``."""
    from .dense import _dense_driver
    fpm, kw = _engine_kwargs(fpm, group, _order(a), shard_rows)
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, False, engine_kwargs=kw)


def feast_he_distributed(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None,
                         group=None, shard_rows=True):
    """feast_he with its contour points (and the rows of its N^2 M0 products)
    sharded over the ranks of ``group``."""
    from .dense import _dense_driver
    fpm, kw = _engine_kwargs(fpm, group, _order(a), shard_rows)
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, True, engine_kwargs=kw)


def feast_sb_distributed(a, kla, emin, emax, m0, *, uplo="F", b=None, klb=None, fpm=None, options=None,
                         x0=None, group=None):
    """feast_sb with its contour points sharded over the ranks of ``group``
    (every rank factors and sweeps only its own shifts of the band)."""
    from .banded import _banded_driver
    fpm, kw = _engine_kwargs(fpm, group, rows=False)
    return _banded_driver(a, kla, b, klb, emin, emax, m0, uplo, fpm, options, x0, False, engine_kwargs=kw)


def feast_hb_distributed(a, kla, emin, emax, m0, *, uplo="F", b=None, klb=None, fpm=None, options=None,
                         x0=None, group=None):
    """feast_hb with its contour points sharded over the ranks of ``group``."""
    from .banded import _banded_driver
    fpm, kw = _engine_kwargs(fpm, group, rows=False)
    return _banded_driver(a, kla, b, klb, emin, emax, m0, uplo, fpm, options, x0, True, engine_kwargs=kw)


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
