python __graft_entry__.py >/dev/null 2>&1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_eig.py -q -p no:hypothesispytest 2>&1 | tail -2
for c in c5 c1 c3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/t7_$c.json 2>gpurun_out/t7_$c.err; python -c "import json;d=json.load(open(\"gpurun_out/t7_$c.json\"));print(\"$c\", round(d[\"ms_per_step\"],2), [(s[\"eig_method\"], s[\"gram_ms\"], s[\"eig_ms\"], s[\"ttm_ms\"]) for s in d[\"stages\"]])"; done
for c in c1 c5; do timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t7_launch_$c.csv python profiles/run_step.py $c 1 > /dev/null 2>&1; done
