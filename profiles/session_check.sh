python __graft_entry__.py >/dev/null 2>&1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reference_suite.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py -q -x -p no:hypothesispytest 2>&1 | tail -3
for c in c3 c1; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"$c\", round(d[\"ms_per_step\"],2), [(s[\"gram_ms\"], s[\"eig_ms\"], s[\"ttm_ms\"]) for s in d[\"stages\"]])"; done
