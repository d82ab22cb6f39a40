# Quick GPU loop: parity (reduced + full-size cfg3/cfg4), the cfg4 unit probe
# (isolated + concurrent batch timings), the ncu launch list of one unit, and
# the NN phase accounting.  Outputs land in gpurun_out/q_*.
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_fullsize.py -m gpu -x -q -k "not cfg5" > gpurun_out/q_test.log 2>&1
timeout 300 python tools/cfg4_probe.py times > gpurun_out/q_times.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/q_launches.csv python tools/cfg4_probe.py unit > gpurun_out/q_unit.log 2>&1
