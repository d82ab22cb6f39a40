"""Device minibatch sampler vs the reference sample_minibatch_indices (diagnostic)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402
from paper_2412_08346_b200 import _lib as L  # noqa: E402

lib = L.load()
lib.asicp_dbg_minibatch.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_int64), C.c_int64, C.c_int32,
                                    C.POINTER(C.c_int32)]
ok_all = True
for par in (1, 0):
    for seed, n, ms in [(208, 10000, [1, 150, 300, 450, 2400, 4500, 5250, 10000]), (5, 1500, [844, 1500, 1500]),
                        (9, 50000, [30000]), (3, 64, [64, 64])]:
        arr = (C.c_int64 * len(ms))(*ms)
        out = np.zeros(sum(ms), dtype=np.int32)
        rc = lib.asicp_dbg_minibatch(seed, n, arr, len(ms), par, out.ctypes.data_as(C.POINTER(C.c_int32)))
        o = skip = 0
        for m in ms:
            want = ref.sample_minibatch_indices(seed, n, m, skip)
            same = np.array_equal(out[o:o + m], want)
            ok_all &= same
            print(f"parallel={par} seed {seed} n {n} m {m}: equal={same}")
            o += m
            skip += m
print("ALL EQUAL" if ok_all else "MISMATCH")
