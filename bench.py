#!/usr/bin/env python
"""B200 AS-ICP bench: particle-iterations/s and per-grasp solve latency.

Default workload (BASELINE.json configs[3], SURVEY.md §8(d) cfg4 — the largest
single-GPU configuration and the north star's multi-object batch): 11
synthetic objects (cylinders / boxes / spheres / blobs, 10k points each, each
on its own table scene) x 3 KG3 preshapes x 1024 particles, k_max = 40 (15
annealed Stein + 25 SGD iterations).  One step = all 11 objects solved and
selected: 33,792 particles x 40 = 1,351,680 particle-iterations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload cfg2|cfg3|cfg4|cfg5|reg] [--n-object N] [--reg-batch B]

--gpus N > 1 without torchrun in the environment re-launches this script under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL);
under torchrun, WORLD_SIZE must equal N.

cfg4 is sharded by shard.plan: whole (object, preshape) units go to the ranks
while they fit the mean load, the leftover units are particle-sharded over all
ranks (NCCL all-gather of the population per Stein iteration, captured in the
solve's CUDA graph), so every rank carries the same particle count; each rank
keeps its pieces device-resident and overlaps them on one GPU (batch.py); the
per-object answers are gathered and selected after the solves.  Total work is
fixed, so the scaling is strong.

cfg2 / cfg3 at N > 1: each rank solves its own object instance (object
sharding, no data-path collective): weak scaling.  cfg5 (configs[4]) is one
population of 16384 particles against an n-point cylinder (--n-object, default
10k), particle-sharded over the ranks (strong scaling).  reg (SURVEY.md §8(f)
rank 4) is a batch of register_sgd_icp problems; metric registrations/s.

The reference arm (--impl reference) times the unmodified reference
optimize_grasp (oracle/_ref) on the host cores, one bounded sample of the
workload per step (cfg4: one (object, preshape) unit — a whole 1024-particle
Stein population — cycling over the 33 units), with inputs built by the
oracle-side fixture library, so that arm maps no product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "particle-iterations/sec"
UNIT = "particle-iterations/s"
PAPER_LATENCY_S = 0.926  # a different metric (latency), not vs_baseline
WORKLOADS = {
    "cfg2": (2, "cfg2: 3 KG3 preshapes x 256 particles vs 10k-pt cylinder, 64^3 SDF, 100 iters (38 Stein)"),
    "cfg3": (3, "cfg3: noisy 40%-occluded single-view 20k-pt scan, 3 KG3 preshapes x 1024 particles, 40 iters "
                "(15 Stein), SDF collision on"),
    "cfg4": (4, "cfg4: 11-object batch (cylinders/boxes/spheres/blobs, 10k pts) x 3 KG3 preshapes x 1024 "
                "particles, 40 iters (15 Stein), (object, preshape) units sharded over ranks"),
    "cfg5": (5, "cfg5: one KG3 preshape x 16384 particles (one Stein population) vs an n-pt cylinder, 40 iters "
                "(15 Stein), particles sharded over ranks with an NCCL allgather per Stein iteration"),
}
CFG5_CPU_SAMPLE_PARTICLES = 2048
N_BATCH_OBJECTS = 11


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS) + ["reg"])
    ap.add_argument("--reg-batch", type=int, default=1184, help="reg: problems per GPU (default 8 per SM)")
    ap.add_argument("--n-object", type=int, default=0, help="cfg5 object cloud size (default 10000)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic capture of the NN kernel")
    ap.add_argument("--cpu-1worker", action="store_true",
                    help="also time the reference with workers = 1 on the cpu_baseline sample")
    ap.add_argument("--dry-run", action="store_true",
                    help="start the ranks (gloo), report them and exit: checks the --gpus launch without a GPU")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_under_torchrun(args) -> int | None:
    """--gpus N > 1 outside torchrun: re-run this script as N ranks (one per
    GPU) under torch.distributed.run on 127.0.0.1; returns its exit code.
    Under torchrun (or N = 1) returns None and the caller proceeds."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus and not (args.gpus == 1 and world > 1 and "--gpus" not in sys.argv):
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return None
    if args.gpus <= 1:
        return None
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def dry_run(args) -> int:
    """Rank plumbing only (gloo, no GPU): every rank reports in, rank 0
    prints one JSON line."""
    rank, world, _ = dist_env()
    ranks = [rank]
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        ranks = [None] * world
        dist.all_gather_object(ranks, rank)
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_arg": args.gpus, "ranks": ranks}), flush=True)
    return 0


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and not s[2 + i].startswith("Not")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def problem_bytes(view) -> int:
    """Host->device bytes asicp_prepare uploads for this problem."""
    v = view.struct
    b = 24 * (v.n_object + v.n_scene) + 32 * v.n_object  # FP64 clouds + FP32 candidates (two layouts)
    for i in range(v.n_preshapes):
        b += 24 * v.preshapes[i].n_surface + 24 + 4 + 4
    for i in range(v.n_sdf_grids):
        g = v.sdf_grids[i]
        b += 4 * g.dims[0] * g.dims[1] * g.dims[2] + 96
    J = view.J
    b += J * (7 * 8 + 4 + 4 + 8) + 7 * 8 * J  # particle tables + init poses
    return int(b)


def solution_bytes(J: int) -> int:
    return J * (7 * 8 + 8 + 4 + 4) + 64


def cpu_reference(fixture, threads: int):
    """Reference optimize_grasp (oracle/_ref) on the host cores, full workload."""
    from oracle import ref

    fixture.struct.workers = threads  # fixtures and CProblem (cfg4 units) both hold an asicp_problem
    t0 = time.perf_counter()
    sol = ref.optimize_grasp(fixture)
    dt = time.perf_counter() - t0
    fixture.struct.workers = 0
    return dt, sol


def sample_fixture(workload: str, n_object: int = 0, seed: int = 0, reference: bool = False):
    """The workload's fixture for object `seed` (cfg5: 2048 of the 16384
    particles — a smaller population makes the reference's O(K^2) Stein step
    cheaper per particle, so the sampled rate flatters the CPU).  reference:
    built by the oracle-side fixture library (the reference arm maps no
    product library)."""
    if reference:
        from oracle import ref

        make = ref.fixture_config
    else:
        from paper_2412_08346_b200 import fixtures

        make = fixtures.config
    if workload == "cfg5":
        return make(5, seed=seed, particles_per_preshape=CFG5_CPU_SAMPLE_PARTICLES, n_object=n_object)
    return make(WORKLOADS[workload][0], seed=seed)


def reference_samples(workload: str, n_object: int, count: int):
    """Per-step samples of the reference arm.  cfg4: the (object, preshape)
    units in order (one whole 1024-particle Stein population each, solved
    exactly as the sharded GPU path solves it, shard.subproblem); others: the
    whole object-0 solve."""
    if workload != "cfg4":
        fx = sample_fixture(workload, n_object, reference=True)
        return [fx] * count, f"full {workload} solve of object 0 ({fx.J * fx.k_max} particle-iterations) per step"
    from paper_2412_08346_b200 import shard
    from paper_2412_08346_b200.grasp import CProblem

    n_units = 3 * N_BATCH_OBJECTS
    objs = {}
    out = []
    for k in range(count):
        u = k % n_units
        o = u // 3
        if o not in objs:
            objs[o] = sample_fixture(workload, seed=o, reference=True).problem()
        unit = shard.units_of([objs[o]])[u % 3]
        out.append(CProblem(shard.subproblem(objs[o], unit)))
    return out, ("one cfg4 (object, preshape) unit per step (1024 particles x 40 iterations = 40960 "
                 "particle-iterations, a whole Stein population), cycling over the 33 units")


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle)"}))
        return 0
    threads = os.cpu_count() or 1
    samples, what = reference_samples(args.workload, args.n_object, args.warmup + args.steps)
    for fx in samples[:args.warmup]:
        cpu_reference(fx, threads)
    times, pits = [], []
    for fx in samples[args.warmup:]:
        dt, _ = cpu_reference(fx, threads)
        times.append(dt)
        pits.append(fx.J * fx.k_max)
    ms = 1e3 * float(np.mean(times))
    value = float(np.sum(pits)) / float(np.sum(times))
    sample = f"{what}, graspmatch::optimize_grasp workers={threads}"
    cfg_fx = sample_fixture(args.workload, args.n_object, reference=True)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if args.workload in ("cfg4", "cfg5") else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args.workload, cfg_fx, world),
        "solve_latency_ms": ms,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(workload, fx, world):
    v = fx.struct
    d = {"workload": WORKLOADS[workload][1],
         "particles": fx.J, "k_max": fx.k_max, "k_stein": fx.k_stein, "n_object": int(v.n_object),
         "n_scene": int(v.n_scene), "n_surface": int(v.preshapes[0].n_surface),
         "sdf_dims": list(v.sdf_grids[0].dims),
         "l2": "flushed (256 MiB write) before every timed step"}
    if workload == "cfg5":
        d.update({"parallelism": f"particle-shard x{world} (NCCL allgather of [theta, drift] per Stein iteration)"
                                 if world > 1 else "1 GPU",
                  "step": "one full optimize_grasp solve of the 16384-particle population"})
    elif workload == "cfg4":
        d.update({"objects": N_BATCH_OBJECTS, "units": 3 * N_BATCH_OBJECTS, "particles": 3 * N_BATCH_OBJECTS * 1024,
                  "particles_per_object": fx.J,
                  "parallelism": (f"shard.plan over {world} GPU(s): whole (object, preshape) units up to the mean "
                                  "load, leftover units particle-sharded over all GPUs (NCCL allgather per Stein "
                                  "iteration); pieces overlapped on streams per GPU"),
                  "step": "all 11 objects solved (33 units) + per-object selection"})
    else:
        d.update({"parallelism": f"object-shard x{world}" if world > 1 else "1 GPU",
                  "step": "one full optimize_grasp solve"})
    return d


class Timer:
    """Device time of a region spanning several streams: a start event on the
    main stream that every worker stream waits on, and an end event recorded
    after the main stream has waited on every worker."""

    def __init__(self, torch, main, workers):
        self.torch, self.main, self.workers = torch, main, workers
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def start(self):
        self.a.record(self.main)
        for s in self.workers:
            s.wait_event(self.a)

    def stop(self):
        for s in self.workers:
            e = self.torch.cuda.Event()
            e.record(s)
            self.main.wait_event(e)
        self.b.record(self.main)

    def ms(self):
        return self.a.elapsed_time(self.b)


REG_METRIC = "registrations/sec"
REG_UNIT = "registrations/s"
REG_DESC = ("reg: SURVEY.md §8(f) rank 4 — register_sgd_icp batch, acceptance C2 problems (500-pt box-surface "
            "clouds displaced <= 0.2 m / 30 deg, Gauss-Newton rotation preconditioner, minibatch 100, 500 iterations)")


def reg_problems(n: int):
    """Problem i = C2 trial i % 20 (test_acceptance.cpp:256-282) with seed 1000 + i."""
    from paper_2412_08346_b200 import fixtures

    trials = [fixtures.c2_trial(t) for t in range(20)]
    srcs = [trials[i % 20][0] for i in range(n)]
    refs = [trials[i % 20][1] for i in range(n)]
    inits = np.tile([0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0], (n, 1))
    seeds = [1000 + i for i in range(n)]
    return srcs, refs, inits, seeds


def reg_cpu(srcs, refs, inits, seeds, cfg, threads: int):
    """Reference register_sgd_icp (oracle/_ref) over the problems, `threads`
    host threads (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import ref

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        out = list(ex.map(lambda i: ref.register_sgd_icp(srcs[i], refs[i], inits[i], cfg, seeds[i]),
                          range(len(srcs))))
    return time.perf_counter() - t0, out


def reg_config(n: int, world: int):
    return {"workload": REG_DESC, "problems_per_gpu": n, "n_source": 500, "n_reference": 500, "minibatch": 100,
            "max_iterations": 500, "preconditioner": "kGaussNewtonRotation",
            "parallelism": f"problem-shard x{world}" if world > 1 else "1 GPU",
            "step": "one batched solve of every problem (one CTA per problem)",
            "l2": "flushed (256 MiB write) before every timed step"}


def run_registration(args):
    """The §8(f) rank-4 row: batched SGD-ICP registration (csrc/register.cu)."""
    rank, world, local = dist_env()
    sys.path.insert(0, str(ROOT / "tests"))
    from paper_2412_08346_b200 import PreconditionerMode, SgdConfig

    cfg = SgdConfig(preconditioner_mode=PreconditionerMode.kGaussNewtonRotation, minibatch_size=100,
                    max_iterations=500)
    n = args.reg_batch
    sample_n = min(n, 64)
    threads = os.cpu_count() or 1
    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import ref

        if not ref.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle)"}))
            return 0
        srcs, refs, inits, seeds = reg_problems(sample_n)
        for _ in range(args.warmup):
            reg_cpu(srcs, refs, inits, seeds, cfg, threads)
        times = [reg_cpu(srcs, refs, inits, seeds, cfg, threads)[0] for _ in range(args.steps)]
        ms = 1e3 * float(np.mean(times))
        value = sample_n / (ms * 1e-3)
        sample = f"{sample_n} C2 registrations per step, graspmatch::register_sgd_icp on {threads} threads"
        print(json.dumps({
            "impl": "reference", "metric": REG_METRIC, "value": value, "unit": REG_UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": reg_config(sample_n, world),
            "cpu_baseline": {"value": value, "unit": REG_UNIT, "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": REG_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
            flush=True)
        return 0

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2412_08346_b200 import RegistrationBatch, Solver, register_sgd_icp_batch
    from paper_2412_08346_b200 import _lib as L
    import ctypes as C

    main_stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    srcs, refs, inits, seeds = reg_problems(n)
    seeds = [s + rank * n for s in seeds]  # each rank its own problems (problem sharding, weak scaling)
    solver = Solver(device=local, stream=main_stream.cuda_stream)
    batch = RegistrationBatch(solver, srcs, refs, inits, seeds, cfg)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def all_max(x: float) -> float:
        t = torch.tensor([x], device="cuda")
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        result = batch.run()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kern_ms = []
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            ev[k][0].record(main_stream)
            result = batch.run()
            ev[k][1].record(main_stream)
            kern_ms.append(solver.stats().solve_ms)
        barrier()
    ms_max = all_max(float(np.mean([a.elapsed_time(b) for a, b in ev])))
    value = world * n / (ms_max * 1e-3)

    for _ in range(args.warmup):  # untimed end-to-end warm-ups (host allocator first touch)
        register_sgd_icp_batch(srcs, refs, inits, cfg, seeds, solver=solver)
    e2e_ms = []
    for k in range(max(1, args.steps)):
        barrier()
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_res = register_sgd_icp_batch(srcs, refs, inits, cfg, seeds, solver=solver)
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_max = all_max(float(np.median(e2e_ms)))  # median: see the grasp workloads below
    e2e_mean = all_max(float(np.mean(e2e_ms)))
    same_e2e = all(np.array_equal(a.theta, b.theta) for a, b in zip(result, e2e_res))

    lib = L.load()
    lib.asicp_dbg_dfma_tflops.restype = C.c_double
    peak = float(lib.asicp_dbg_dfma_tflops(4000))
    iters = sum(r.iterations for r in result)
    pairs = float(iters) * 100 * 500  # (query, reference point) pairs of the brute-force NN
    kms = float(np.mean(kern_ms))
    achieved = 8.0 * pairs / (kms * 1e-3) / 1e12

    if rank == 0:
        line = {
            "metric": REG_METRIC, "value": value, "unit": REG_UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": reg_config(n, world),
            "registration_iterations_per_s": world * iters / (ms_max * 1e-3),
            "e2e": {"value": world * n / (e2e_max * 1e-3), "unit": REG_UNIT,
                    "h2d_bytes_per_step": batch.input_bytes, "d2h_bytes_per_step": batch.output_bytes,
                    "latency_ms": e2e_max, "stat": "median of the K steps (max over ranks)",
                    "mean_latency_ms": e2e_mean, "mean_value": world * n / (e2e_mean * 1e-3),
                    "steps_ms": e2e_ms, "bit_identical_to_resident": same_e2e},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "roofline": {"bound": "fp64", "kernel": "register_kernel", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak > 0 else None,
                         "peak_source": "DFMA microbenchmark on this GPU (asicp_dbg_dfma_tflops); the NN "
                                        "cannot contract (bit-exactness), so 0.5 is its ceiling",
                         "traffic": None, "kernel_ms": kms,
                         "algorithmic": "8 FP64 FLOP x (batch point, reference point) pairs: "
                                        "iterations x 100 x 500 per problem"},
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                from oracle import ref

                if ref.available():
                    dt, rs = reg_cpu(srcs[:sample_n], refs[:sample_n], inits[:sample_n], seeds[:sample_n], cfg,
                                     threads)
                    same = all(np.array_equal(a.theta, b.theta) and a.final_loss == b.final_loss
                               and a.iterations == b.iterations for a, b in zip(rs, result[:sample_n]))
                    line["cpu_baseline"] = {
                        "value": sample_n / dt, "unit": REG_UNIT, "cores": threads, "kind": "reference",
                        "sample": f"the first {sample_n} problems, oracle/_ref graspmatch::register_sgd_icp on "
                                  f"{threads} threads", "bit_identical": same}
            except Exception as e:  # reported, never required
                line["cpu_baseline"] = {"error": repr(e)}
        print(json.dumps(line), flush=True)
    solver.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_baseline(args, result, batch: bool) -> dict:
    """The reference (oracle/_ref) on this box's host cores, on a bounded
    sample of the workload, with the bit-identity of the sample's answer.
    cfg4: object 0 solved whole (3 preshapes x 1024 particles) vs the GPU's
    object-0 answer (its units' summaries combined)."""
    try:
        from oracle import ref

        if not ref.available():
            return {"error": "oracle/_ref not built"}
        threads = os.cpu_count() or 1
        sfx = sample_fixture(args.workload, args.n_object, reference=True)
        spits = sfx.J * sfx.k_max
        dt, rs = cpu_reference(sfx, threads)
        if args.workload == "cfg5":
            same = None  # the sample is a smaller population than the bench's
        elif batch:
            r0 = result[0]
            same = bool(rs.final_loss == r0["final_loss"] and np.array_equal(rs.theta, r0["theta"])
                        and np.array_equal(rs.particle_theta, r0["particle_theta"])
                        and np.array_equal(rs.particle_loss, r0["particle_loss"]))
        else:
            same = bool(np.array_equal(rs.particle_theta, result.particle_theta)
                        and rs.final_loss == result.final_loss)
        out = {
            "value": spits / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"one full {args.workload} solve of object 0 ({sfx.J} particles, {spits} particle-iterations), "
                      f"oracle/_ref graspmatch::optimize_grasp workers={threads}"
                      + (" (extrapolated per particle-iteration to the 11-object batch)" if batch else ""),
            "latency_ms": dt * 1e3,
            "bit_identical": same,
        }
        if args.cpu_1worker:
            dt1, _ = cpu_reference(sfx, 1)
            out["workers_1"] = {"value": spits / dt1, "latency_ms": dt1 * 1e3, "cores": 1}
        return out
    except Exception as e:  # the baseline is reported, never required
        return {"error": repr(e)}


def traffic_child(workload: str, n_object: int) -> None:
    """Run under ncu by measure_traffic: one profiled (eager) solve of the
    workload's NN roofline problem (cfg4: unit 0)."""
    from paper_2412_08346_b200 import Solver, fixtures, shard
    from paper_2412_08346_b200.grasp import CProblem

    if workload == "cfg4":
        p = fixtures.config(4, seed=0).problem()
        prob = CProblem(shard.subproblem(p, shard.units_of([p])[0]))
    elif workload == "cfg5":
        prob = fixtures.config(5, seed=0, n_object=n_object)
    else:
        prob = fixtures.config(WORKLOADS[workload][0], seed=0)
    s = Solver(device=0, profile=True)
    s.prepare(prob)
    s.run()
    s.close()


def measure_traffic(args, timeout_s: int = 300) -> dict | None:
    """roofline.traffic: DRAM bytes (read + write) per launch of the NN filter
    kernel, from one ncu capture (two DRAM counters only) of one profiled solve
    of the same problem the roofline times.  ncu's timings are not used."""
    import csv
    import shutil
    import tempfile

    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).exists():
        return {"error": "ncu not found"}
    with tempfile.TemporaryDirectory() as td:
        log = Path(td) / "traffic.csv"
        code = f"import sys; sys.path.insert(0, {str(ROOT)!r}); import bench; bench.traffic_child({args.workload!r}, {args.n_object})"
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--print-units", "base",
               "-k", "regex:nn_filter_kernel", "--csv", "--log-file", str(log), sys.executable, "-c", code]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, cwd=str(ROOT))
        except subprocess.TimeoutExpired:
            return {"error": f"ncu timed out after {timeout_s} s"}
        if r.returncode != 0 or not log.exists():
            return {"error": f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-300:]}"}
        per = {}
        with open(log) as f:
            rows = [ln for ln in f if ln.startswith('"')]
        for row in csv.DictReader(rows):
            name = row.get("Metric Name", "")
            if name.startswith("dram__bytes_"):
                v = float(str(row.get("Metric Value", "0")).replace(",", ""))
                per[row["ID"]] = per.get(row["ID"], 0.0) + v
        if not per:
            return {"error": "no nn_filter_kernel launches captured"}
        vals = list(per.values())
        return {"bytes_per_launch": float(np.mean(vals)), "launches": len(vals), "max_bytes": float(max(vals)),
                "total_bytes": float(sum(vals)),
                "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every nn_filter_kernel "
                          "launch of one profiled solve (cfg4: unit 0), measured inside this bench run"}


def main():
    args = parse()
    rc = relaunch_under_torchrun(args)
    if rc is not None:
        return rc
    if args.dry_run:
        return dry_run(args)
    if args.workload == "reg":
        return run_registration(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    rank, world, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2412_08346_b200 import Solver, fixtures, shard
    from paper_2412_08346_b200 import _lib as L
    from paper_2412_08346_b200.batch import BatchSolver
    from paper_2412_08346_b200.grasp import CProblem, nccl_unique_id
    import ctypes as C

    main_stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def all_max(x: float) -> float:
        t = torch.tensor([x], device="cuda")
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def all_gather(obj):
        if dist is None:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def all_sum(x: int) -> int:
        return int(sum(all_gather(x)))

    def broadcast(obj):
        box = [obj]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    batch = args.workload == "cfg4"
    e2e_split = []  # (prepare ms, run ms) per e2e step (single-problem workloads)
    if batch:
        problems = [fixtures.config(4, seed=o).problem() for o in range(N_BATCH_OBJECTS)]
        units = shard.units_of(problems)
        pieces = shard.plan(units, world)[rank]
        subs = [CProblem(shard.subproblem(problems[units[pc.unit].obj], units[pc.unit])) for pc in pieces]
        k_max = problems[0].k_max
        pits_total = sum(u.count for u in units) * k_max
        streams = [torch.cuda.Stream() for _ in subs]

        def join(i, solver):
            # A unit shared by all ranks: one NCCL communicator per unit (ids
            # made by rank 0 and broadcast in the same unit order everywhere).
            pc = pieces[i]
            if pc.world > 1:
                solver.set_partition_nccl(pc.rank, pc.world, broadcast(nccl_unique_id() if rank == 0 else None))

        runner = BatchSolver(subs, device=local, streams=[s.cuda_stream for s in streams], setup=join)
        fx = fixtures.config(4, seed=0)  # config description / CPU sample (object 0)

        def solve_resident():
            runner.launch()

        def finish():
            sols = runner.wait()
            parts = all_gather([shard.summary(pc.unit, s) for pc, s in zip(pieces, sols) if pc.rank == 0])
            return shard.combine(problems, parts)

        def solve_e2e():
            # asicp_prepare (H2D of the unit's host buffers) then asicp_run_async,
            # unit by unit: the GPU solves unit i while the host prepares i + 1.
            runner.prepare_launch(subs)
            return finish()

        worker_streams = streams
        h2d = sum(problem_bytes(cp) for cp in subs)
        d2h = sum(solution_bytes(cp.J) for cp in subs)
        launches_of = runner.launches
    else:
        cfg = WORKLOADS[args.workload][0]
        solver = Solver(device=local, stream=main_stream.cuda_stream)
        if args.workload == "cfg5":
            # One population sharded by particle: every rank prepares the same problem.
            fx = fixtures.config(5, seed=0, n_object=args.n_object)
            pits_total = fx.J * fx.k_max
            if world > 1:
                shard.join_particle_partition(solver, rank, world, broadcast)
        else:
            fx = fixtures.config(cfg, seed=rank)  # object instance per rank (object sharding)
            pits_total = world * fx.J * fx.k_max
        solver.prepare(fx)
        holder = {}

        def solve_resident():
            holder["sol"] = solver.run()

        def finish():
            return holder["sol"]

        def solve_e2e():
            # asicp_optimize_grasp = asicp_prepare (validate + H2D) + asicp_run
            # (solve + D2H + selection); the split is recorded for diagnosis.
            t0 = time.perf_counter()
            solver.prepare(fx)
            t1 = time.perf_counter()
            sol = solver.run()
            e2e_split.append((1e3 * (t1 - t0), 1e3 * (time.perf_counter() - t1)))
            return sol

        worker_streams = []
        h2d = problem_bytes(fx)
        d2h = solution_bytes(fx.J)
        launches_of = lambda: solver.stats().kernel_launches  # noqa: E731

    # ---- device-resident timing (value): inputs already in HBM ----
    for _ in range(args.warmup):
        solve_resident()
        result = finish()
    barrier()
    timers = [Timer(torch, main_stream, worker_streams) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            timers[k].start()
            solve_resident()
            timers[k].stop()
            if batch:
                result = finish()
        barrier()
    if not batch:
        result = finish()
    ms_max = all_max(float(np.mean([t.ms() for t in timers])))
    value = pits_total / (ms_max * 1e-3)
    launches = launches_of()

    # ---- end-to-end through the public API with host buffers ----
    # W untimed end-to-end warm-ups first: the first few host-side prepares
    # run into fresh-page faults of the host allocator (tools/prepare_timing.py).
    for _ in range(args.warmup):
        barrier()
        solve_e2e()
    e2e_split.clear()
    e2e_ms, e2e_dev_ms = [], []
    for k in range(max(1, args.steps)):
        barrier()
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        result = solve_e2e()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
        if not batch:
            e2e_dev_ms.append(solver.stats().solve_ms)
    # Median over the K end-to-end steps: the host side of a step (validate +
    # pageable H2D) sees sporadic multi-ms stalls on these boxes that are not
    # the library's (tools/prepare_timing.py); the mean is reported beside it.
    e2e_max = all_max(float(np.median(e2e_ms)))
    e2e_mean = all_max(float(np.mean(e2e_ms)))
    e2e_value = pits_total / (e2e_max * 1e-3)

    # ---- roofline of the dominant kernel (NN filter), profiled run on one problem ----
    prof = Solver(device=local, stream=main_stream.cuda_stream, profile=True)
    prof.prepare(subs[0] if batch else fx)
    prof.run()
    st = prof.stats()
    prof.close()
    nn_ms_per_launch = st.nn_ms / max(st.nn_launches, 1)
    nn_flops = 8.0 * st.nn_pairs  # 8 algorithmic FLOP per (query, candidate) pair
    achieved = nn_flops / (st.nn_ms * 1e-3) / 1e12 if st.nn_ms > 0 else None
    lib = L.load()
    lib.asicp_dbg_ffma_tflops.restype = C.c_double
    peak = float(lib.asicp_dbg_ffma_tflops(20000))
    active_evals = sum(int(x) for x in ([s.raw_stats()[13] for s in runner.solvers] if batch
                                         else [solver.raw_stats()[13]]))
    active_total = all_sum(active_evals)  # particle evaluations that were not SGD-frozen
    traffic = None
    if rank == 0 and world == 1 and not args.no_traffic:
        traffic = measure_traffic(args)

    if rank == 0:
        best = result[0] if batch else result
        status = int(best["status"]) if batch else int(best.status)
        final_loss = best["final_loss"] if batch else best.final_loss
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if args.workload in ("cfg4", "cfg5") else "weak",
            "vs_baseline": None, "dtype": "f64 (FP32-certified NN filter)", "data": "synthetic",
            "config": config_dict(args.workload, fx, world),
            "solve_latency_ms": ms_max,
            "paper_latency_ms": PAPER_LATENCY_S * 1e3,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "latency_ms": e2e_max, "stat": "median of the K steps (max over ranks)",
                    "mean_latency_ms": e2e_mean, "mean_value": pits_total / (e2e_mean * 1e-3),
                    "steps_ms": e2e_ms, "device_solve_ms": e2e_dev_ms,
                    "prepare_run_ms": e2e_split},
            "gpu_launches": int(launches) * args.steps,
            "clocks": clk.summary(),
            "roofline": {"bound": "fp32", "kernel": "nn_filter_kernel",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if (achieved and peak > 0) else None,
                         "peak_source": "FFMA microbenchmark on this GPU (asicp_dbg_ffma_tflops)",
                         "traffic": traffic.get("bytes_per_launch") if traffic else None,
                         "traffic_detail": traffic, "nn_ms_per_launch": nn_ms_per_launch,
                         "nn_launches": int(st.nn_launches), "nn_share_of_step": st.nn_ms / st.solve_ms,
                         "algorithmic": "8 FLOP x (query, candidate) pairs; pairs counted by the kernel"},
            "status": status, "final_loss": final_loss,
            "active_particle_iterations_per_step": active_total,
            "stage_ms_profiled_unit": {"nn_filter": st.nn_ms, "collide": st.collide_ms,
                                       "minibatch": st.minibatch_ms, "cost": st.cost_ms, "stein": st.svgd_ms,
                                       "solve": st.solve_ms},
        }
        if batch:
            line["objects_found"] = int(sum(int(r["status"]) == 0 for r in result))
        else:
            line["nn"] = result.diagnostics
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args, result, batch)
        print(json.dumps(line), flush=True)
    if batch:
        runner.close()
    else:
        solver.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
