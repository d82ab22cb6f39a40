import sys, time
sys.path.insert(0, '/root/repo')
from paper_2412_08346_b200 import Solver, fixtures
ppp, n = int(sys.argv[1]), int(sys.argv[2])
fx = fixtures.config(5, seed=0, particles_per_preshape=ppp, n_object=n).set(k_max=int(sys.argv[3]), k_stein=min(15, int(sys.argv[3]) - 1), anneal_period_total=int(sys.argv[3]))
s = Solver(use_graph=False)
try:
    s.prepare(fx); sol = s.run(); print(ppp, n, "ok", s.stats().solve_ms)
except Exception as e:
    print(ppp, n, "FAIL", str(e)[:150])
