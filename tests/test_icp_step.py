"""icp_closed_form_step oracle pinning (CPU only): the plain-C restatement
(oracle/port) equals the reference (oracle/_ref, optim.cpp:51-90 with the
Eigen shim's JacobiSVD) and the committed golden vectors, on cases reaching
every SVD / Kabsch / Shepperd branch and every error path."""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent))
import reg_cases  # noqa: E402

from oracle import ref  # noqa: E402
from paper_2412_08346_b200 import InvalidArgument  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden" / "icp_step.npz"


@pytest.fixture(scope="module")
def golden():
    g = np.load(GOLDEN)
    return {str(n): (g["theta"][i], bool(g["degenerate"][i])) for i, n in enumerate(g["names"])}


@pytest.mark.skipif(not ref.port_available(), reason="oracle port not built")
@pytest.mark.parametrize("case", reg_cases.icp_cases(), ids=lambda c: c[0])
def test_port_matches_golden(case, golden):
    name, src, rf, th = case
    r = ref.port_icp_closed_form_step(src, rf, th)
    assert np.array_equal(r.theta, golden[name][0]) and r.degenerate == golden[name][1]


def test_golden_covers_every_branch(golden):
    assert golden["single_point"][1] and golden["collinear"][1] and golden["two_points"][1]
    assert not golden["planar"][1] and not golden["aligned"][1]
    # Shepperd: the 150-degree cases have negative traces (the other branches).
    for ax in range(3):
        q = golden[f"rot150_axis{ax}"][0][3:]
        assert abs(q[0]) < 0.3 and abs(q[1 + ax]) > 0.9


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_port_errors_match_reference():
    src = np.zeros((5, 3))
    bad = reg_cases.IDENTITY.copy()
    bad[3] = 1.2
    for args in [(np.zeros((0, 3)), src, reg_cases.IDENTITY), (src, src + 1.0, bad)]:
        msgs = []
        for fn in (ref.icp_closed_form_step, ref.port_icp_closed_form_step):
            with pytest.raises(InvalidArgument) as e:
                fn(*args)
            msgs.append(str(e.value))
        assert msgs[0] == msgs[1]
