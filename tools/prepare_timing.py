"""Time asicp_prepare (validate + H2D) and asicp_run repeatedly on cfg2 to
separate host-side noise from the device solve (diagnostics)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2412_08346_b200 import Solver, fixtures  # noqa: E402

torch.cuda.set_device(0)
fx = fixtures.config(2, seed=0)
s = Solver(stream=torch.cuda.current_stream().cuda_stream)
s.prepare(fx)
s.run()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(16):
    if i >= 8:  # second half: the bench's L2 flush before each step
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.prepare(fx)
    t1 = time.perf_counter()
    s.run()
    t2 = time.perf_counter()
    print(f"prepare {1e3 * (t1 - t0):7.2f} ms   run {1e3 * (t2 - t1):7.2f} ms")
