"""Object / preshape sharding across ranks.

Stein populations are per preshape and particles never migrate
(grasp.cpp:213-234); particle j's minibatch stream is seeded with seed + j over
the preshape-major flattening (grasp.cpp:135-151); the only cross-preshape step
is the final argmin (grasp.cpp:283-306).  So an (object, preshape) unit solved
on its own — the object's problem restricted to that preshape, with the seed
advanced by the unit's first global particle index and the preshape's stacked
SDF offset kept — reproduces exactly the particles the full solve would, and
the per-object answer is a tiny gather of particle summaries followed by the
reference's selection rule.  No collective touches the data path.

Balance (`plan`): whole units go to the least-loaded rank while they fit the
mean load; the units left over are particle-sharded over ALL ranks through the
cfg5 mechanism (asicp_set_partition_nccl: every rank prepares the unit and owns
the slice [r K / R, (r + 1) K / R), one NCCL all-gather of the population's
poses and drifts per Stein iteration).  33 equal units on 8 ranks: 4 whole
units plus 1/8 of the 33rd per rank — 4224 particles each, the exact mean
(longest-processing-time over whole units alone gives a 5 / 4 split, an 82.5 %
efficiency ceiling).

`solve_sharded` is solver-agnostic (the B200 Solver in production, the CPU
restatement in the multi-process tests) and takes an `all_gather` callable
(torch.distributed.all_gather_object over NCCL or gloo).
"""
from __future__ import annotations

import copy
from dataclasses import dataclass
from typing import Callable, List, Sequence

import numpy as np

from .grasp import GraspProblem, GraspStatus, StackedSdf


@dataclass
class Unit:
    obj: int          # object (problem) index
    preshape: int     # preshape index within the object
    first: int        # first global particle index of the preshape
    count: int        # particles


@dataclass
class Piece:
    unit: int         # index into units_of(problems)
    world: int        # ranks sharing the unit (1: the whole unit on one rank)
    rank: int         # this rank's position in the unit's partition
    count: int        # particles this rank owns


def units_of(problems: Sequence[GraspProblem]) -> List[Unit]:
    """Every (object, preshape) population, including empty ones (a preshape
    with no initial poses — the reference accepts it and its Stein step skips
    it); `plan` and `assign` give empty units to no rank."""
    out = []
    for o, p in enumerate(problems):
        first = 0
        for s, init in enumerate(p.initializations):
            k = len(np.asarray(init).reshape(-1, 7))
            out.append(Unit(o, s, first, k))
            first += k
    return out


def assign(units: Sequence[Unit], world: int) -> List[int]:
    """Longest-processing-time assignment of whole units to ranks
    (deterministic); empty units get owner -1."""
    load = [0] * world
    owner = [-1] * len(units)
    for i in sorted((i for i in range(len(units)) if units[i].count > 0), key=lambda i: (-units[i].count, i)):
        r = min(range(world), key=lambda r: (load[r], r))
        owner[i] = r
        load[r] += units[i].count
    return owner


def plan(units: Sequence[Unit], world: int) -> List[List[Piece]]:
    """Per-rank work: whole units by LPT while they fit the mean load, then the
    remaining units particle-sharded over all ranks (same unit order on every
    rank, so the partitions' collectives line up).  Deterministic."""
    total = sum(u.count for u in units)
    target = total / world
    load = [0] * world
    pieces: List[List[Piece]] = [[] for _ in range(world)]
    split = []
    for i in sorted((i for i in range(len(units)) if units[i].count > 0), key=lambda i: (-units[i].count, i)):
        r = min(range(world), key=lambda r: (load[r], r))
        k = units[i].count
        if world == 1 or k < world or load[r] + k <= target * (1.0 + 1e-12):
            pieces[r].append(Piece(i, 1, 0, k))
            load[r] += k
        else:
            split.append(i)
    for s, i in enumerate(sorted(split)):
        for r in range(world):
            pr = (r + s) % world  # rotate the slices so the uneven ones spread over the ranks
            lo, hi = particle_slice(units[i].count, pr, world)
            pieces[r].append(Piece(i, world, pr, hi - lo))
    return pieces


def subproblem(p: GraspProblem, u: Unit) -> GraspProblem:
    """The object's problem restricted to one preshape (same SDF grid and
    offset, seed advanced to the preshape's first global particle)."""
    q = copy.copy(p)
    pre = copy.copy(p.preshapes[u.preshape])
    g = pre.sdf_index
    q.sdf = StackedSdf([p.sdf.grids[g]], p.sdf.epsilon, [p.sdf.offsets[g]])
    pre.sdf_index = 0
    q.preshapes = [pre]
    q.initializations = [p.initializations[u.preshape]]
    q.seed = int(p.seed) + u.first
    q.record_trace = False
    return q


def select(theta, loss, free, conv, preshape):
    """grasp.cpp:283-306: strict < over collision-free particles in global
    order, else the best attempt with kNoGraspFound."""
    best = -1
    for j in range(len(loss)):
        if free[j] and (best < 0 or loss[j] < loss[best]):
            best = j
    status = GraspStatus.kFound
    if best < 0:
        status = GraspStatus.kNoGraspFound
        for j in range(len(loss)):
            if best < 0 or loss[j] < loss[best]:
                best = j
    return dict(status=status, theta=np.asarray(theta[best]), preshape_id=int(preshape[best]),
                final_loss=float(loss[best]), converged=bool(conv[best]), particle_theta=np.asarray(theta),
                particle_loss=np.asarray(loss), particle_collision_free=np.asarray(free),
                particle_converged=np.asarray(conv), particle_preshape=np.asarray(preshape))


def summary(i: int, sol) -> tuple:
    """What a rank contributes for unit i (gathered, then `combine`d)."""
    return (i, np.asarray(sol.particle_theta), np.asarray(sol.particle_loss),
            np.asarray(sol.particle_collision_free), np.asarray(sol.particle_converged))


def solve_local(problems: Sequence[GraspProblem], solve_fn: Callable[[GraspProblem], object], rank: int,
                world: int, partition_fn: Callable[[GraspProblem, Piece], object] | None = None) -> list:
    """Solve `rank`'s pieces (`plan`); returns the particle summaries to
    gather.  A particle-sharded piece is solved by partition_fn(sub, piece),
    which returns the WHOLE unit's summaries on every rank of the partition
    (the solver's final all-gather); its partition rank 0 contributes them.
    Without partition_fn a sharded piece is solved whole by solve_fn (the
    CPU restatement in the tests: same answer, no exchange)."""
    units = units_of(problems)
    mine = []
    for pc in plan(units, world)[rank]:
        u = units[pc.unit]
        sub = subproblem(problems[u.obj], u)
        sol = solve_fn(sub) if pc.world == 1 or partition_fn is None else partition_fn(sub, pc)
        if pc.rank == 0:
            mine.append(summary(pc.unit, sol))
    return mine


def solve_sharded(problems: Sequence[GraspProblem], solve_fn: Callable[[GraspProblem], object], rank: int,
                  world: int, all_gather: Callable[[object], list],
                  partition_fn: Callable[[GraspProblem, Piece], object] | None = None) -> list:
    """Solve `rank`'s pieces, gather the summaries from all ranks and return
    the per-object selections (identical on every rank)."""
    return combine(problems, all_gather(solve_local(problems, solve_fn, rank, world, partition_fn)))


def join_particle_partition(solver, rank: int, world: int, broadcast: Callable[[object], object]) -> bytes:
    """Particle sharding within a population (cfg5): rank 0 makes the NCCL
    unique id, `broadcast` (torch.distributed.broadcast_object_list from rank
    0) hands it to every rank, and every rank joins the communicator with its
    Solver (asicp_set_partition_nccl, collective).  Afterwards each rank
    prepares the SAME full problem; the solver owns the particle slice
    [r J / R, (r + 1) J / R) and returns the full answer on every rank."""
    from .grasp import nccl_unique_id

    uid = nccl_unique_id() if rank == 0 else None
    uid = broadcast(uid)
    solver.set_partition_nccl(rank, world, uid)
    return uid


def particle_slice(J: int, rank: int, world: int) -> tuple:
    """The global particles a rank owns under particle sharding (solver.cu prepare)."""
    return rank * J // world, (rank + 1) * J // world


def combine(problems: Sequence[GraspProblem], gathered: list) -> list:
    """Per-object selection from the gathered unit summaries."""
    units = units_of(problems)
    by_unit = {}
    for part in gathered:
        for rec in part:
            by_unit[rec[0]] = rec[1:]
    results = []
    for o, _ in enumerate(problems):
        idx = [i for i, u in enumerate(units) if u.obj == o and u.count > 0]
        theta = np.concatenate([np.asarray(by_unit[i][0]).reshape(-1, 7) for i in idx])
        loss = np.concatenate([by_unit[i][1] for i in idx])
        free = np.concatenate([by_unit[i][2] for i in idx])
        conv = np.concatenate([by_unit[i][3] for i in idx])
        pre = np.concatenate([np.full(units[i].count, units[i].preshape) for i in idx])
        results.append(select(theta, loss, free, conv, pre))
    return results
