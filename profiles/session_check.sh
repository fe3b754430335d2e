# Quick GPU check used between commits: parity suites + C2/C3/C1 bench lines.
python __graft_entry__.py >/dev/null 2>&1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reference_suite.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_als_fused.py tests/test_gpu_dist.py -q -x -p no:hypothesispytest > gpurun_out/session_tests.log 2>&1
ATK_TRACE=1 timeout 300 python profiles/als_probe.py 3 2>&1 | grep -E "rep|it=4\]" | tail -6
for o in 1 0; do timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --opt als_fused=$o 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"c2 als_fused=$o\", round(d[\"ms_per_step\"],2), [(s[\"gram_ms\"], s[\"eig_ms\"], s[\"ttm_ms\"], s[\"als_ms\"]) for s in d[\"stages\"]])"; done
echo "tests: $(tail -1 gpurun_out/session_tests.log)"
