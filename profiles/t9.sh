python __graft_entry__.py >/dev/null 2>&1; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eig.py tests/test_gpu_tridiag.py -q -x -p no:hypothesispytest 2>&1 | tail -3
for o in 1 0; do timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --opt cheb_fused=$o 2>gpurun_out/t9_c2_$o.err | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"c2 cheb_fused=$o\", round(d[\"ms_per_step\"],2), [(s[\"eig_ms\"], s[\"als_ms\"]) for s in d[\"stages\"]])"; done
ATK_TRACE=1 timeout 300 python profiles/run_step.py c2 1 2>&1 | grep -E "filter|done" | head -12
