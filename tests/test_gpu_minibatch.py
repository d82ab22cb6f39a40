"""Device minibatch sampler (mt19937_64 + Lemire + partial Fisher-Yates,
rng.hpp:16-44 / spatial_index.cpp:111-123) against the reference draws.

Covers every path: the counting-sort kernel (clouds of <= 49152 points, any
m; 16-bit shared arena, 32-bit shared arena, shared counters + global
arrays), the radix-sort kernel at its three sizes (m <= 4096, 12288, 20480)
for larger clouds, the all-global counting sort beyond that (cfg5's 200k-point
clouds), and the serial swap kernel (parallel disabled), over consecutive
calls on one engine stream.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2412_08346_b200 import _lib as L

pytestmark = pytest.mark.gpu

CASES = [(208, 10000, [1, 150, 300, 450, 2400, 4500, 5250, 10000]), (5, 1500, [844, 1500, 1500]),
         (7, 30000, [3000, 12000, 16000, 20000, 24000]), (9, 50000, [30000]), (3, 64, [64, 64]),
         (11, 60000, [3000, 9000, 15000, 22000]), (13, 200000, [20000, 60000, 150000])]


def draws(seed, n, ms, parallel):
    lib = L.load()
    lib.asicp_dbg_minibatch.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_int64), C.c_int64, C.c_int32,
                                        C.POINTER(C.c_int32)]
    arr = (C.c_int64 * len(ms))(*ms)
    out = np.zeros(sum(ms), dtype=np.int32)
    assert lib.asicp_dbg_minibatch(seed, n, arr, len(ms), parallel, out.ctypes.data_as(C.POINTER(C.c_int32))) == 0
    return out


@pytest.mark.parametrize("case", range(len(CASES)))
def test_parallel_and_serial_draws_match_reference(case):
    from oracle import ref

    seed, n, ms = CASES[case]
    par, ser = draws(seed, n, ms, 1), draws(seed, n, ms, 0)
    assert np.array_equal(par, ser)
    if not ref.available():
        pytest.skip("oracle/_ref not built: parallel == serial checked only")
    o = skip = 0
    for m in ms:
        assert np.array_equal(par[o:o + m], ref.sample_minibatch_indices(seed, n, m, skip)), (n, m)
        o += m
        skip += m
