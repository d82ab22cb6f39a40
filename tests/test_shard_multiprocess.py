"""Multi-process (world_size 2, gloo, CPU) test of the object/preshape sharding.

Two ranks split the (object, preshape) units of a 2-object batch (3 KG3
preshapes each, cfg2 shape reduced), solve their units with the CPU
restatement (oracle port — the GPU path is the same host logic around the
B200 Solver), all-gather the particle summaries over gloo and select per
object.  The sharded answers must equal the unsharded solve bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ref

pytestmark = pytest.mark.skipif(not ref.port_available(), reason="oracle port not built (make -C oracle port)")


def _problems():
    from paper_2412_08346_b200 import fixtures

    out = []
    for seed in (0, 1):
        fx = fixtures.config(2, seed=seed, particles_per_preshape=3)
        fx.set(k_max=4, k_stein=2, anneal_period_total=4)
        out.append(fx.problem())
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2412_08346_b200.shard import solve_sharded

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    res = solve_sharded(_problems(), ref.port_optimize_grasp, rank, world, gather)
    q.put((rank, [(int(r["status"]), r["theta"], r["final_loss"], r["particle_loss"]) for r in res]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_solve_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [ref.port_optimize_grasp(p) for p in _problems()]
    for rank in (0, 1):
        for (status, theta, loss, ploss), w in zip(outs[rank], want):
            assert status == int(w.status)
            assert np.array_equal(theta, w.theta)
            assert loss == w.final_loss
            assert np.array_equal(ploss, w.particle_loss)


def test_assignment_is_balanced_and_deterministic():
    from paper_2412_08346_b200.shard import Unit, assign

    units = [Unit(o, p, 0, 1024) for o in range(11) for p in range(3)]
    owner = assign(units, 8)
    assert owner == assign(units, 8)
    loads = np.bincount(owner, minlength=8)
    assert loads.max() - loads.min() <= 1  # 33 equal units on 8 ranks -> 5/4 split


class _RecordingSolver:
    def set_partition_nccl(self, rank, world, uid):
        self.args = (rank, world, uid)


def _partition_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2412_08346_b200.shard import join_particle_partition

    def broadcast(obj):
        box = [obj]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    s = _RecordingSolver()
    join_particle_partition(s, rank, world, broadcast)
    q.put((rank, s.args))
    dist.barrier()
    dist.destroy_process_group()


def test_particle_partition_join_shares_one_nccl_id():
    """cfg5 plumbing over gloo: rank 0's NCCL unique id reaches every rank and
    each rank joins with its own (rank, world)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_partition_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[0][:2] == (0, 2) and outs[1][:2] == (1, 2)
    assert len(outs[0][2]) == 128 and outs[0][2] == outs[1][2]


def test_particle_slices_cover_the_population():
    from paper_2412_08346_b200.shard import particle_slice

    for J in (1, 7, 21, 100, 16384):
        for world in (1, 2, 3, 8):
            if J < world:
                continue
            cuts = [particle_slice(J, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == J
            assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
            sizes = [hi - lo for lo, hi in cuts]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
