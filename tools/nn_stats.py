"""Print the NN certification counters of one solve (diagnostic).
   python tools/nn_stats.py [cfg] [max_chunks]"""
import ctypes as C, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2412_08346_b200 import Solver, fixtures
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
fx = fixtures.desk(0) if cfg == 0 else fixtures.config(cfg, seed=0)
s = Solver()
if len(sys.argv) > 2:
    s.lib.asicp_set_option(s.ctx, 4, int(sys.argv[2]))
sol = s.optimize(fx)
t = time.time(); sol = s.run(); dt = time.time() - t
raw = (C.c_uint64 * 256)()
s.lib.asicp_dbg_raw_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
s.lib.asicp_dbg_raw_stats(s.ctx, raw)
names = ["fp64_windows", "full_rescans", "queries", "ties", "pairs", "rescan_fwd", "rescan_rev", "rescan_final",
         "why_mode", "why_top3", "why_list", "why_merge"]
print(f"solve {dt*1e3:.1f} ms", {n: int(raw[i]) for i, n in enumerate(names)})
print("per-iteration rescans:", [int(raw[16 + k]) for k in range(fx.k_max + 1)])
import struct
f = lambda u: struct.unpack('<f', struct.pack('<I', int(u) & 0xffffffff))[0]
d = [int(raw[201 + i]) for i in range(14)]
print("first top3 overflow: iter", d[0], "particle", d[1], "q", d[2], "b1 b2 b3 thr", [f(x) for x in d[3:7]], "nc", d[7],
      "s1 s2", d[8] & 0xffff, d[8] >> 16, "q", [f(x) for x in d[9:12]], "margin", f(d[12]), "cbase", d[13])
print("collide status counts: clear", int(raw[240]), "hit", int(raw[241]), "exact", int(raw[242]))
