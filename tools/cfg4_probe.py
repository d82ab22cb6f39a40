"""cfg4 probe: where the 11-object batch spends its time.

  python tools/cfg4_probe.py times [--objects N]
      every (object, preshape) unit solved alone (graph replay, device time of
      the ctx stream), their sum, and all units launched together as bench.py
      does (wall time around launch + wait).
  python tools/cfg4_probe.py unit [--unit U] [--objects N]
      one warm-up solve of unit U, then one solve between
      cudaProfilerStart/Stop (ncu --profile-from-start off): the launch list of
      exactly one 1024-particle unit.
"""
import argparse
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2412_08346_b200 import Solver, fixtures, shard  # noqa: E402
from paper_2412_08346_b200.batch import BatchSolver  # noqa: E402
from paper_2412_08346_b200 import _lib as L  # noqa: E402
from paper_2412_08346_b200.grasp import CProblem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("mode", choices=["times", "unit", "subset"])
ap.add_argument("--units", type=str, default="4,8,17,33", help="subset: batch sizes (first U units) to time")
ap.add_argument("--objects", type=int, default=11)
ap.add_argument("--unit", type=int, default=0)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--max-chunks", type=int, default=0, help="ASICP_OPT_MAX_CHUNKS of the batch contexts")
ap.add_argument("--latency", action="store_true", help="subset: batch contexts in latency mode (no ASICP_OPT_THROUGHPUT)")
ap.add_argument("--tc", type=int, default=0, help="NN filter on the tensor cores: 0 none, 1 every unit, K >= 2 every K-th")
a = ap.parse_args()


def tc_setup(i, s):
    if a.tc:
        s.lib.asicp_set_option(s.ctx, L.ASICP_OPT_NN_TC, 1 if (a.tc == 1 or i % a.tc == 0) else 0)


problems = [fixtures.config(4, seed=o).problem() for o in range(a.objects)]
units = shard.units_of(problems)
subs = [CProblem(shard.subproblem(problems[u.obj], u)) for u in units]

if a.mode == "unit":
    cudart = ctypes.CDLL("libcudart.so.12") if Path("/usr/local/cuda/lib64/libcudart.so.12").exists() else None
    s = Solver(use_graph=not a.eager)
    s.prepare(subs[a.unit])
    s.run()
    s.run()
    if cudart is None:
        import torch

        torch.cuda.profiler.start()
    else:
        cudart.cudaProfilerStart()
    sol = s.run()
    if cudart is None:
        torch.cuda.profiler.stop()
    else:
        cudart.cudaProfilerStop()
    st = s.stats()
    print(f"unit {a.unit}: solve {st.solve_ms:.3f} ms, {st.kernel_launches} launches, status {int(sol.status)}")
    raw = s.raw_stats()
    nsub = 4 * ((problems[units[a.unit].obj].scene_cloud.shape[0] + 31) // 32)
    print(f"collision sub-clusters left to the point test: {raw[14]} of {raw[13] + 1024} x {nsub} "
          f"({raw[14] / max(1, (raw[13] + 1024) * nsub):.3%})")
    print(f"NN: uncertified windows {raw[0]}, full FP64 rescans {raw[1]} (validation {raw[8]}, ambiguous window "
          f"{raw[9]}, across splits {raw[11]}), queries {raw[2]}")
    ph = raw[240:248]
    if sum(ph):
        names = ["item start", "TMA wait", "hot loop", "top-3", "window epilogue", "sub-chunk barrier", "emit",
                 "exit"]
        print("NN filter phases (warp-cycles): " + ", ".join(f"{n} {v / sum(ph):.1%}" for n, v in zip(names, ph)))
    s.close()
    sys.exit(0)

if a.mode == "subset":
    # Device time of a batch of the first U units (the per-rank share of the
    # cfg4 plan at 8 / 4 / 2 ranks is 4 / 8 / 16 whole units + a slice).
    for u in [int(x) for x in a.units.split(",")]:
        b = BatchSolver(subs[:u], setup=tc_setup, throughput=not a.latency)
        b.run()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            b.run()
            ts.append(1e3 * (time.perf_counter() - t0))
        b.close()
        print(f"{u:3d} units ({u * 1024} particles): {sorted(ts)[2]:.1f} ms (median of 5)", flush=True)
    sys.exit(0)

iso = []
for i, p in enumerate(subs):
    s = Solver()
    s.prepare(p)
    s.run()
    best = min((s.run(), s.stats().solve_ms)[1] for _ in range(3))
    iso.append(best)
    s.close()
print("isolated unit solve ms:", " ".join(f"{t:.2f}" for t in iso))
print(f"sum of isolated unit solves: {sum(iso):.1f} ms  (mean {sum(iso) / len(iso):.2f} ms)")
b = BatchSolver(subs, max_chunks=a.max_chunks, setup=tc_setup)
b.run()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    b.run()
    ts.append(1e3 * (time.perf_counter() - t0))
print("concurrent batch wall ms:", " ".join(f"{t:.1f}" for t in ts))
b.close()
