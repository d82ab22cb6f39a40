"""Run one cfg2 solve (for ncu launch lists / captures).  Usage:
   python tools/profile_once.py [cfg] [--graph] [--runs N]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2412_08346_b200 import Solver, fixtures

cfg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2
runs = int(sys.argv[sys.argv.index("--runs") + 1]) if "--runs" in sys.argv else 1
fx = fixtures.config(cfg, seed=0)
s = Solver(use_graph="--graph" in sys.argv)
s.prepare(fx)
for _ in range(runs):
    sol = s.run()
print("status", sol.status, "loss", sol.final_loss, sol.diagnostics)
raw = s.raw_stats()
nsub = 4 * ((fx.struct.n_scene + 31) // 32)
print(f"collision sub-clusters left to the point test: {raw[14] / max(1, (raw[13] + fx.J) * nsub):.3%}")
if "--iter-stats" in sys.argv:
    import ctypes as C
    n = 4 * 64
    buf = (C.c_uint64 * n)()
    got = s.lib.asicp_dbg_iter_stats(s.ctx, buf, n)
    rows = [list(buf[4 * i:4 * i + 4]) for i in range(got // 4) if any(buf[4 * i:4 * i + 4])]
    print("per-iteration counters [fwd pairs, rev pairs, fwd queries, rev queries]:")
    for i, r in enumerate(rows):
        print(i, r)
