"""Parity report: B200 path vs the reference oracle on desk seeds / cfg1 (diagnostic)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2412_08346_b200 import Solver, fixtures
from oracle import ref

s = Solver()
for name, fx in [(f"desk{seed}", fixtures.desk(seed)) for seed in range(10)] + \
        [("cfg1", fixtures.config(1, seed=0))]:
    fx.set(record_trace=1)
    t = time.time(); want = ref.optimize_grasp(fx); t_ref = time.time() - t
    s.optimize(fx)
    t = time.time(); got = s.optimize(fx); t_gpu = time.time() - t
    dth = np.abs(got.trace_theta - want.trace_theta).max()
    dl = np.nanmax(np.abs(got.trace_loss - want.trace_loss))
    bit = np.array_equal(got.trace_theta, want.trace_theta) and np.array_equal(got.particle_loss, want.particle_loss)
    d = got.diagnostics
    print(f"{name}: bit_identical={bit} max|dtheta|={dth:.3e} max|dloss|={dl:.3e} "
          f"col_equal={np.array_equal(got.trace_in_collision, want.trace_in_collision)} "
          f"status {got.status}/{want.status} free {got.particle_collision_free.sum()}/{want.particle_collision_free.sum()} "
          f"ref {t_ref*1e3:.0f} ms gpu {t_gpu*1e3:.1f} ms | queries {d['nn_queries']} uncert {d['nn_uncertified']} "
          f"refine {d['nn_full_refines']} ties {d['nn_pool_ties']} pairs {d['nn_pairs']:.3e}", flush=True)

# device exp vs the box's libm
import ctypes as Cc, math
lib = Cc.CDLL(str(Path(__file__).resolve().parent.parent / "paper_2412_08346_b200" / "libasicp.so"))
rng = np.random.default_rng(0)
x = np.concatenate([-rng.uniform(0, 40, 1_000_000), -rng.exponential(3, 500_000)])
y = np.zeros_like(x)
lib.asicp_dbg_exp_device(x.ctypes.data_as(Cc.c_void_p), y.ctypes.data_as(Cc.c_void_p), Cc.c_int64(len(x)))
ref = np.array([math.exp(v) for v in x])
print("device exp mismatches vs libm:", int((y.view(np.uint64) != ref.view(np.uint64)).sum()), "of", len(x))
