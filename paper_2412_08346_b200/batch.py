"""Device-resident batch of independent solves overlapped on one B200.

A batch entry is an object's problem or one (object, preshape) unit of it
(shard.subproblem).  Each entry gets its own context (device buffers, captured
CUDA graph) and stream; `run` enqueues every solve (asicp_run_async) before
waiting on any (asicp_wait), so the small-population kernels of one entry fill
the SMs the others leave idle.  A 1024-particle unit keeps about 1.5 GB
resident, so the 33 units of the 11-object batch (cfg4) fit one GPU's HBM.

Selection per object is shard.combine's (the reference's rule,
grasp.cpp:283-306); nothing here changes what a solve computes.
"""
from __future__ import annotations

from typing import Callable, List, Sequence

from .grasp import GraspProblem, GraspSolution, Solver


class BatchSolver:
    """`setup(i, solver)`, when given, runs before entry i is prepared (e.g. to
    join a particle partition, shard.plan's shared units)."""

    def __init__(self, problems: Sequence[GraspProblem], device: int = 0, streams: Sequence[int] | None = None,
                 setup: Callable[[int, Solver], None] | None = None, **solver_kw):
        if streams is not None and len(streams) != len(problems):
            raise ValueError("one stream per problem")
        self.solvers: List[Solver] = []
        solver_kw.setdefault("throughput", True)  # the entries share the GPU: split the NN for throughput
        for i, p in enumerate(problems):
            s = Solver(device=device, stream=streams[i] if streams is not None else None, **solver_kw)
            if setup is not None:
                setup(i, s)
            s.prepare(p)
            self.solvers.append(s)

    def launch(self) -> None:
        for s in self.solvers:
            s.run_async()

    def prepare_launch(self, problems: Sequence[GraspProblem]) -> None:
        """Re-prepare every entry from host buffers and launch it at once, so
        entry i's solve runs on the GPU while the host prepares entry i + 1
        (the end-to-end path: asicp_prepare + asicp_run_async per entry)."""
        if len(problems) != len(self.solvers):
            raise ValueError("one problem per entry")
        for s, p in zip(self.solvers, problems):
            s.prepare(p)
            s.run_async()

    def wait(self) -> List[GraspSolution]:
        return [s.wait() for s in self.solvers]

    def run(self) -> List[GraspSolution]:
        self.launch()
        return self.wait()

    def launches(self) -> int:
        return sum(int(s.stats().kernel_launches) for s in self.solvers)

    def close(self) -> None:
        for s in self.solvers:
            s.close()
        self.solvers = []
