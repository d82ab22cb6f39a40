"""graspmatch::build_sdf on the GPU against the
reference field: bit-identical values, dims, origin and boundary maximum.

The CPU restatement fixtures.build_sdf is itself pinned to oracle/_ref by
tests/test_fixtures_capi.py::test_cylinder_and_build_sdf_bit_identical; when
oracle/_ref is present the GPU field is also compared with it directly.
"""
import numpy as np
import pytest

from paper_2412_08346_b200 import InvalidArgument, Solver, fixtures

pytestmark = pytest.mark.gpu


def clouds():
    kg3 = fixtures.config(1, seed=0, particles_per_preshape=4).problem().preshapes[0].full_cloud
    cyl = fixtures.cylinder_cloud(0.04, 0.15, 4000, 3)
    rng = np.random.default_rng(5)
    half = np.array([0.05, 0.03, 0.02])
    box = rng.uniform(-1, 1, (3000, 3)) * half  # box surface: one coordinate pinned to a face
    axis = rng.integers(0, 3, 3000)
    box[np.arange(3000), axis] = np.sign(rng.uniform(-1, 1, 3000)) * half[axis]
    return [("kg3", kg3, 0.005, -1.0, 0.003), ("kg3_fine", kg3, 0.0037, 0.01, 0.002),
            ("cylinder", cyl, 0.004, -1.0, 0.003), ("box", box, 0.006, 0.02, 0.004)]


@pytest.mark.parametrize("case", range(4))
def test_build_sdf_matches_reference_field(case):
    name, cloud, voxel, pad, band = clouds()[case]
    s = Solver()
    got = s.build_sdf(cloud, voxel, pad, band)
    s.close()
    dims, origin, vox, bmax, values = fixtures.build_sdf(cloud, voxel, pad, band)
    assert tuple(got.dims) == tuple(dims), name
    assert np.array_equal(got.origin, origin) and got.voxel == vox, name
    assert np.array_equal(got.values.view(np.uint32), np.asarray(values, dtype=np.float32).view(np.uint32)), name
    assert got.boundary_max_abs == bmax, name
    assert (got.values > 0).any() and (got.values < 0).any(), name  # an interior and an exterior


def test_build_sdf_matches_oracle_ref():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    name, cloud, voxel, pad, band = clouds()[0]
    s = Solver()
    got = s.build_sdf(cloud, voxel, pad, band)
    s.close()
    want = ref.build_sdf(cloud, voxel, pad, band)
    assert tuple(got.dims) == tuple(want[0])
    assert np.array_equal(got.values.view(np.uint32), np.asarray(want[4], dtype=np.float32).view(np.uint32))
    assert got.boundary_max_abs == want[3]


def test_build_sdf_invalid_arguments():
    s = Solver()
    kg3 = clouds()[0][1]
    with pytest.raises(InvalidArgument, match="voxel must be positive"):
        s.build_sdf(kg3, 0.0)
    with pytest.raises(InvalidArgument, match="need >= 4 non-coplanar points"):
        s.build_sdf(kg3[:3], 0.005)
    plane = np.c_[np.random.default_rng(1).uniform(-1, 1, (50, 2)), np.zeros(50)]
    with pytest.raises(InvalidArgument, match="need >= 4 non-coplanar points"):
        s.build_sdf(plane, 0.05)
    s.close()
