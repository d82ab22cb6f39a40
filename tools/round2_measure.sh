# Round-2 measurement set (one GPU): the GPU test suite, every bench
# workload, the reference arm, ncu launch lists and full captures of the
# dominant kernels.  Outputs in gpurun_out/m2_*.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m2_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/m2_gputest.log 2>&1
timeout 900 python bench.py > gpurun_out/m2_bench_cfg4.log 2>&1
timeout 900 python bench.py --workload cfg2 --cpu-1worker > gpurun_out/m2_bench_cfg2.log 2>&1
timeout 600 python bench.py --workload cfg3 > gpurun_out/m2_bench_cfg3.log 2>&1
timeout 900 python bench.py --workload cfg5 > gpurun_out/m2_bench_cfg5.log 2>&1
timeout 600 python bench.py --workload reg > gpurun_out/m2_bench_reg.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/m2_bench_ref_cfg4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/m2_cfg4_unit_launches.csv python tools/cfg4_probe.py unit > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m2_cfg2_launches.csv python tools/profile_once.py 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:nn_filter -s 30 -c 1 -o gpurun_out/m2_nn_filter python tools/cfg4_probe.py unit > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:nn_filter -s 40 -c 1 -o gpurun_out/m2_nn_final python tools/cfg4_probe.py unit > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:collide -s 20 -c 1 -o gpurun_out/m2_collide python tools/cfg4_probe.py unit > /dev/null 2>&1
timeout 300 python tools/cfg4_probe.py times > gpurun_out/m2_cfg4_times.log 2>&1
