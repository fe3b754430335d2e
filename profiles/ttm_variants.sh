#!/bin/bash
# C5 step stage times under TTM variants (split off / wide single MMA / two MMAs).
TAG=${1:-tv}; mkdir -p gpurun_out
run() { timeout 300 env $2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 $3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"$1\", round(d[\"ms_per_step\"],2), [(s[\"gram_ms\"], s[\"eig_ms\"], s[\"ttm_ms\"]) for s in d[\"stages\"]])"; }
run split_wide "" ""
run split_two "ATK_TTM_SPLIT2=1" ""
run nosplit "" "--opt ttm_split=0"
