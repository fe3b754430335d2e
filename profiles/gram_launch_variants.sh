#!/bin/bash
# C5 step under different Gram K-launch sizes (option gram_launch_kb; the wide units use half).
for kb in 4096 2048 1024 8192; do
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 --opt gram_launch_kb=$kb 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"launch_kb=$kb\", round(d[\"ms_per_step\"],2), [s[\"gram_ms\"] for s in d[\"stages\"]], d[\"clocks\"][\"sm_mhz\"])"
done
