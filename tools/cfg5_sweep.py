"""cfg5 object-size sweep on one GPU (diagnostic): one 16384-particle solve per
cloud size, device time and peak memory.  usage: python tools/cfg5_sweep.py 10000 50000 ..."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2412_08346_b200 import Solver, fixtures  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [10000, 50000, 100000, 200000]
for n in sizes:
    fx = fixtures.config(5, seed=0, n_object=n)
    s = Solver()
    try:
        free0, total = torch.cuda.mem_get_info()
        t0 = time.perf_counter()
        s.prepare(fx)
        free1, _ = torch.cuda.mem_get_info()
        sol = s.run()
        t1 = time.perf_counter()
        sol = s.run()
        st = s.stats()
        print(f"n={n:7d} J={fx.J} device {st.solve_ms:9.1f} ms  first call {1e3 * (t1 - t0):9.1f} ms  "
              f"resident {(free0 - free1) / 2**30:6.1f} GiB of {total / 2**30:.0f}  "
              f"pit/s {fx.J * fx.k_max / (st.solve_ms * 1e-3):,.0f}  status {int(sol.status)} loss {sol.final_loss:.4g}",
              flush=True)
    except Exception as e:  # report and continue with the next size
        print(f"n={n:7d} failed: {e}", flush=True)
    s.close()
    torch.cuda.empty_cache()
