# NN filter phase accounting (diagnostic): rebuild the library with
# -DASICP_NN_PHASES, run one cfg4 unit, print the per-phase warp-cycle shares.
set -e
ASICP_NVCC_EXTRA=-DASICP_NN_PHASES python -c "from paper_2412_08346_b200 import build; build.build(force=True)"
python tools/cfg4_probe.py unit --eager
