# Tensor-core NN filter (ASICP_NN_TC=1): one solve, parity tests, cfg2/cfg4 bench, launch list.
set -x
ASICP_NN_TC=1 timeout 90 python tools/profile_once.py 2 > gpurun_out/t_once.log 2>&1 || exit 1
ASICP_NN_TC=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_test.log 2>&1
ASICP_NN_TC=1 timeout 120 python bench.py --workload cfg2 --steps 10 --warmup 3 --no-traffic --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/t_cfg2.json
ASICP_NN_TC=1 timeout 180 python bench.py --steps 5 --warmup 3 --no-traffic --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/t_cfg4.json
ASICP_NN_TC=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t_launches.csv python tools/profile_once.py 2 > gpurun_out/t_ncu.log 2>&1
