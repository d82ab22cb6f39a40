"""Host-side checks of the product library (CPU, no kernel launches).

* libasicp.so loads and exports every symbol include/*.h declares;
* the host-exact scalar helpers reproduce the reference KATs;
* the glibc-exact exp restatement used by the SVGD kernel equals the
  platform exp bit for bit;
* the bench/test fixtures are bit-identical to the reference's own
  synthetic fixtures (synthetic.cpp, sdf.cpp:48-175).
"""
import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import ref
from paper_2412_08346_b200 import _lib as L
from paper_2412_08346_b200 import annealing, fixtures, minibatch_schedule

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols(headers=None):
    names = set()
    for h in headers or sorted((ROOT / "include").glob("*.h")):
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(asicp_\w+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    """libasicp.so exports everything asicp.h / asicp_debug.h declare;
    the fixture generators live in their own library (asicp_fixtures.h)."""
    fx_header = ROOT / "include" / "asicp_fixtures.h"
    product = [h for h in sorted((ROOT / "include").glob("*.h")) if h != fx_header]
    lib = C.CDLL(str(L.LIB_PATH))
    names = declared_symbols(product)
    assert len(names) >= 18
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(L.EXPORTS) <= names
    assert L.load().asicp_abi_version() == 1
    assert not any(hasattr(lib, n) for n in L.FIXTURE_EXPORTS), "fixtures are not part of the product library"
    fx = C.CDLL(str(L.FIXTURES_PATH))
    fx_names = declared_symbols([fx_header])
    assert fx_names == set(L.FIXTURE_EXPORTS)
    assert not [n for n in sorted(fx_names) if not hasattr(fx, n)]


def test_python_constants_mirror_the_header():
    """Every ASICP_OPT_* / status define of asicp.h has the same value in the
    ctypes layer (_lib.py), so Solver options reach the right switch."""
    text = (ROOT / "include" / "asicp.h").read_text()
    defines = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(ASICP_\w+)\s+(-?\d+)", text)}
    opts = {k: v for k, v in defines.items() if k.startswith("ASICP_OPT_")}
    assert {"ASICP_OPT_NN_MODE", "ASICP_OPT_THROUGHPUT", "ASICP_OPT_NN_TC"} <= set(opts)
    for k, v in opts.items():
        assert getattr(L, k) == v, k


def test_schedule_kats():
    """test_spatial_index.cpp:153-184 / test_acceptance.cpp:633-657."""
    assert minibatch_schedule(13, 40, 900) == 439
    for k_max in (40, 15, 7):
        for n in (900, 60, 1):
            sat = 2.0 * k_max / 3.0
            for k in range(k_max + 1):
                want = min(max(round(n * min(k, sat) / sat + 0.0), 1), n)
                got = minibatch_schedule(k, k_max, n)
                assert abs(got - want) <= 1  # python round() is banker's; llround ties away
                if k >= sat:
                    assert got == n


def test_annealing_kats():
    """test_optim.cpp:352-382."""
    assert annealing(4, 40, 5, 2.0) == 0.25
    assert annealing(8, 40, 5, 2.0) == 0.0
    assert annealing(0, 40, 5, 2.0) == 0.0


def test_glibc_exact_exp_host():
    lib = C.CDLL(str(L.LIB_PATH))
    rng = np.random.default_rng(1)
    x = np.concatenate([-rng.uniform(0, 40, 300_000), -rng.exponential(3.0, 100_000), rng.uniform(-300, 300, 50_000)])
    y = np.zeros_like(x)
    lib.asicp_dbg_exp_host(x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), C.c_int64(len(x)))
    want = np.array([math.exp(v) for v in x])
    assert np.array_equal(y.view(np.uint64), want.view(np.uint64))


needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("seed", [0, 7])
def test_desk_fixture_bit_identical(seed):
    a = fixtures.desk(seed).problem()
    b = ref.desk(seed).problem()
    assert np.array_equal(a.object_cloud, b.object_cloud)
    assert np.array_equal(a.scene_cloud, b.scene_cloud)
    pa, pb = a.preshapes[0], b.preshapes[0]
    assert np.array_equal(pa.inner_surface_cloud, pb.inner_surface_cloud)
    assert np.array_equal(pa.full_cloud, pb.full_cloud)
    assert np.array_equal(pa.tcp, pb.tcp)
    ga, gb = a.sdf.grids[0], b.sdf.grids[0]
    assert tuple(ga.dims) == tuple(gb.dims)
    assert np.array_equal(ga.origin, gb.origin) and ga.voxel == gb.voxel
    assert ga.boundary_max_abs == gb.boundary_max_abs
    assert np.array_equal(ga.values, gb.values)
    assert np.array_equal(a.initializations[0], b.initializations[0])
    assert np.array_equal(a.com, b.com)
    assert a.seed == b.seed == seed


@needs_ref
def test_cylinder_and_build_sdf_bit_identical():
    for args in [(0.04, 0.15, 10000, 1), (0.03, 0.12, 2000, 5)]:
        assert np.array_equal(fixtures.cylinder_cloud(*args), ref.cylinder_cloud(*args))
    kg3 = fixtures.config(1, seed=0, particles_per_preshape=8).problem().preshapes[0].full_cloud
    for voxel, pad, band in [(0.005, -1.0, 0.003), (0.0037, 0.01, 0.002)]:
        a = fixtures.build_sdf(kg3, voxel, pad, band)
        b = ref.build_sdf(kg3, voxel, pad, band)
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2] and a[3] == b[3]
        assert np.array_equal(a[4], b[4])


def test_kg3_fixture_shape():
    fx = fixtures.config(1, seed=0)
    v = fx.struct
    assert fx.J == 64 and fx.k_max == 50 and fx.k_stein == 15
    assert v.preshapes[0].n_surface == 1008
    fx2 = fixtures.config(2, seed=0, particles_per_preshape=4)
    v2 = fx2.struct
    assert v2.n_preshapes == 3 and fx2.J == 12 and fx2.k_max == 100 and fx2.k_stein == 38
    for i in range(3):
        assert max(v2.sdf_grids[i].dims[:]) == 64


def test_partial_view_and_batch_fixtures():
    """cfg3 (noisy 40 %-occluded single view, 20k points) and cfg4 (the
    11-object batch) fixture shapes; deterministic per seed."""
    a = fixtures.config(3, seed=0, particles_per_preshape=4).problem()
    b = fixtures.config(3, seed=0, particles_per_preshape=4).problem()
    assert a.object_cloud.shape == (20000, 3)
    assert np.array_equal(a.object_cloud, b.object_cloud)
    assert len(a.preshapes) == 3 and a.k_max == 40 and a.k_stein == 15
    assert not np.array_equal(a.object_cloud, fixtures.config(3, seed=1, particles_per_preshape=4).problem().object_cloud)
    clouds = [fixtures.config(4, seed=o, particles_per_preshape=4).problem().object_cloud for o in range(11)]
    for c in clouds:
        assert c.shape == (10000, 3) and c[:, 2].min() >= -1e-12  # standing on the table plane
    assert len({c.tobytes() for c in clouds}) == 11
    full = fixtures.config(4, seed=0)
    assert full.J == 3 * 1024 and full.problem().stein.step_scale == 64.0 / 1024


def _problem_arrays(p):
    out = [p.object_cloud, p.scene_cloud, p.com, np.array([p.k_max, p.k_stein, p.seed, p.contact_tolerance])]
    for s in p.preshapes:
        out += [s.inner_surface_cloud, s.full_cloud, s.tcp, np.array([s.sdf_index])]
    for g, off in zip(p.sdf.grids, p.sdf.offsets):
        out += [np.asarray(g.origin), np.array([g.voxel, g.boundary_max_abs]), np.asarray(g.dims), g.values,
                np.asarray(off)]
    out += [np.asarray(i) for i in p.initializations]
    return out


def test_oracle_side_fixtures_equal_product_fixtures():
    """bench.py's reference arm builds its inputs with the oracle-side build of
    csrc/fixtures.cu (oracle/_build/libasicp_fixtures_oracle.so), so it maps no
    product library: both builds must produce the same problems."""
    if not ref.FIXTURES_PATH.exists():
        pytest.skip("make -C oracle port")
    for cfg, seed in [(4, 3), (2, 0), (3, 1)]:
        a = fixtures.config(cfg, seed=seed, particles_per_preshape=16).problem()
        b = ref.fixture_config(cfg, seed=seed, particles_per_preshape=16).problem()
        xa, xb = _problem_arrays(a), _problem_arrays(b)
        assert len(xa) == len(xb)
        for u, v in zip(xa, xb):
            assert np.array_equal(u, v)


def test_reference_arm_maps_no_product_library():
    """The reference arm (bench.py --impl reference) must not load libasicp.so
    or libasicp_fixtures.so: run its input construction in a fresh process and
    read its memory map."""
    import subprocess
    import sys

    code = ("import bench, sys\n"
            "fx = bench.sample_fixture('cfg4', 0, reference=True)\n"
            "maps = open('/proc/self/maps').read()\n"
            "sys.exit(1 if ('libasicp.so' in maps or 'libasicp_fixtures.so' in maps) else 0)\n")
    if not ref.FIXTURES_PATH.exists():
        pytest.skip("make -C oracle port")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
