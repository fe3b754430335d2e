python __graft_entry__.py >/dev/null 2>&1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tridiag.py tests/test_gpu_eig.py tests/test_gpu_dist.py -q -p no:hypothesispytest 2>&1 | tail -3
for o in "-1" "0"; do timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --opt eig_method=$o > gpurun_out/t6_c2_$o.json 2>gpurun_out/t6_c2_$o.err; python -c "import json;d=json.load(open(\"gpurun_out/t6_c2_$o.json\"));print(\"c2 eig_method=$o\", round(d[\"ms_per_step\"],2), [(s[\"eig_method\"], s[\"gram_ms\"], s[\"eig_ms\"], s[\"ttm_ms\"], s[\"als_ms\"]) for s in d[\"stages\"]])"; done
ATK_TRACE=1 timeout 300 python profiles/run_step.py c2 2 > gpurun_out/t6_trace_c2.log 2>&1
