"""Host-side breakdown of an end-to-end optimize (diagnostic, GPU):
prepare (validate + upload) vs run (graph replay + D2H + selection)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2412_08346_b200 import Solver, fixtures  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
fx = fixtures.config(cfg, seed=0)
s = Solver()
for rep in range(6):
    t0 = time.perf_counter()
    s.prepare(fx)
    t1 = time.perf_counter()
    s.run()
    t2 = time.perf_counter()
    st = s.stats()
    print(f"rep {rep}: prepare {1e3 * (t1 - t0):7.2f} ms  run {1e3 * (t2 - t1):7.2f} ms  "
          f"(device solve {st.solve_ms:6.2f} ms)", flush=True)
