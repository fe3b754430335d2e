python __graft_entry__.py >/dev/null 2>&1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_eig.py -q -p no:hypothesispytest 2>&1 | tail -2
for c in c1 c5; do timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t8_launch_$c.csv python profiles/run_step.py $c 1 > /dev/null 2>&1; done
