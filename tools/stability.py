"""SVGD stability scan of the cfg2 workload (diagnostic)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2412_08346_b200 import Solver, fixtures
s = Solver()
for ppp in [64, 128, 256]:
    for scale in [1.0, 0.5, 0.25, 0.1]:
        fx = fixtures.config(2, seed=0, particles_per_preshape=ppp).set(record_trace=1, step_scale=scale)
        sol = s.optimize(fx)
        com = np.array(fx.struct.com[:])
        d = np.linalg.norm(sol.trace_theta[:, :, :3] - com, axis=2)
        mx = d.max(1)
        print(f"ppp {ppp} scale {scale}: max dist k=10 {mx[10]:.3g} k=20 {mx[20]:.3g} k=37 {mx[37]:.3g} k=99 {mx[99]:.3g} "
              f"| free {sol.particle_collision_free.mean():.2f} status {int(sol.status)} loss {sol.final_loss:.4g} "
              f"median final dist {np.median(d[99]):.3g}", flush=True)
