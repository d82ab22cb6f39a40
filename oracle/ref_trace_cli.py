"""Reference trace file of the desk scenario — TEST INFRASTRUCTURE ONLY.

    python oracle/ref_trace_cli.py SEED N_INIT N_TOP K_MAX K_STEIN ANNEAL_TOTAL PATH

Runs graspmatch::optimize_grasp with record_trace and graspmatch::export_trace
(io.cpp:691-710) from oracle/_ref in a process that loads nothing else: the
library carries a static libstdc++ whose iostreams crash when another
libstdc++ (numpy's) is already loaded, so tests call this in a subprocess.
"""
import ctypes
import sys
from pathlib import Path

lib = ctypes.CDLL(str(Path(__file__).resolve().parent / "_ref" / "libgraspmatch_ref.so"))
lib.ref_desk_export_trace.argtypes = [ctypes.c_uint64] + [ctypes.c_int64] * 5 + [ctypes.c_char_p]
seed, n_init, n_top, k_max, k_stein, anneal = (int(a) for a in sys.argv[1:7])
sys.exit(lib.ref_desk_export_trace(seed, n_init, n_top, k_max, k_stein, anneal, sys.argv[7].encode()))
