import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2412_08346_b200 import _lib as L
from oracle import ref
lib = L.load()
lib.asicp_dbg_minibatch.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_int32)]
for seed, n, ms in [(208, 10000, [1, 150, 300, 450, 2400, 4500, 5250]), (5, 1500, [844, 1500, 1500]), (9, 50000, [30000])]:
    arr = (C.c_int64 * len(ms))(*ms)
    out = np.zeros(sum(ms), dtype=np.int32)
    rc = lib.asicp_dbg_minibatch(seed, n, arr, len(ms), out.ctypes.data_as(C.POINTER(C.c_int32)))
    o = 0; skip = 0; ok = True
    for m in ms:
        want = ref.sample_minibatch_indices(seed, n, m, skip)
        got = out[o:o + m]
        same = np.array_equal(got, want)
        ok &= same
        print(f"seed {seed} n {n} m {m}: equal={same} unique={len(np.unique(got))}")
        o += m; skip += m
