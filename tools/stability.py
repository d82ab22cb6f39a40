"""SVGD stability scan of a fixture workload (diagnostic, GPU).

usage: python tools/stability.py [CFG [SEED [PPP,PPP.. [SCALE,SCALE..]]]]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2412_08346_b200 import Solver, fixtures

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ppps = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [64, 128, 256]
scales = [float(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1.0, 0.5, 0.25, 0.1]
s = Solver()
for ppp in ppps:
    for scale in scales:
        fx = fixtures.config(cfg, seed=seed, particles_per_preshape=ppp).set(record_trace=1, step_scale=scale)
        sol = s.optimize(fx)
        com = np.array(fx.struct.com[:])
        d = np.linalg.norm(sol.trace_theta[:, :, :3] - com, axis=2)
        mx = d.max(1)
        ks = sorted({10, fx.struct.k_stein - 1, fx.struct.k_max - 1})
        st = s.stats()
        print(f"cfg{cfg} seed {seed} ppp {ppp} scale {scale}: " +
              " ".join(f"max dist k={k} {mx[k]:.3g}" for k in ks) +
              f" | free {sol.particle_collision_free.mean():.2f} status {int(sol.status)} loss {sol.final_loss:.4g}"
              f" median final dist {np.median(d[-1]):.3g} solve {st.solve_ms:.2f} ms", flush=True)
