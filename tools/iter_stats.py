"""Per-iteration NN work of one solve (asicp_dbg_iter_stats), optionally joined
with an ncu launch list to give per-launch FLOP rates.

usage: python tools/iter_stats.py [CFG] [--launches launches.csv] [--json out.json]
"""
import csv
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2412_08346_b200 import Solver, fixtures  # noqa: E402
from paper_2412_08346_b200 import _lib as L  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2
s = Solver()
fx = fixtures.config(cfg, seed=0)
s.prepare(fx)
s.run()
lib = L.load()
lib.asicp_dbg_iter_stats.restype = C.c_int64
lib.asicp_dbg_iter_stats.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
n = lib.asicp_dbg_iter_stats(s.ctx, None, 0)
buf = np.zeros(n, dtype=np.uint64)
lib.asicp_dbg_iter_stats(s.ctx, buf.ctypes.data_as(C.c_void_p), n)
st = buf.reshape(-1, 4)
times = {}
if "--launches" in sys.argv:
    rows = list(csv.reader(open(sys.argv[sys.argv.index("--launches") + 1])))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    ki, vi = rows[h].index("Kernel Name"), rows[h].index("Metric Value")
    for r in rows[h + 1:]:
        if len(r) > vi and "nn_filter_kernel" in r[ki]:
            key = "fwd" if "<8" in r[ki] else "rev"
            times.setdefault(key, []).append(float(r[vi].replace(",", "")) * 1e-3)
out = []
for k, (pf, pr, qf, qr) in enumerate(st):
    rec = dict(k=k, fwd_pairs=int(pf), rev_pairs=int(pr), fwd_queries=int(qf), rev_queries=int(qr))
    out.append(rec)
print(f"{'k':>3} {'fwd Mpairs':>11} {'fwd q':>8} {'rev Mpairs':>11} {'rev q':>7}")
for r in out:
    print(f"{r['k']:3d} {r['fwd_pairs'] / 1e6:11.1f} {r['fwd_queries']:8d} {r['rev_pairs'] / 1e6:11.2f} {r['rev_queries']:7d}")
tot = st.sum(0)
print("total fwd pairs %.3e rev pairs %.3e fwd q %d rev q %d" % (tot[0], tot[1], tot[2], tot[3]))
if "--json" in sys.argv:
    Path(sys.argv[sys.argv.index("--json") + 1]).write_text(json.dumps(out))
