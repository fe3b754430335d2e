#!/bin/bash
# Quick GPU check after an engine change: the GPU suite, C5 / C2 / C5u bench lines, a C5 step timeline.
TAG=${1:-q}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > gpurun_out/${TAG}_tests.log 2>&1
echo "tests=$? $(tail -1 gpurun_out/${TAG}_tests.log)"; grep -E "^FAILED|^ERROR|Error" gpurun_out/${TAG}_tests.log | head
for c in c5 c2 c5u; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c=$?"
done
python - <<PY
import json
for c in ["c5","c2","c5u"]:
    try:
        d=json.load(open(f"gpurun_out/${TAG}_bench_{c}.json"))
        print(c, round(d["ms_per_step"],3), round(d["value"]), [(s["gram_ms"], s["eig_ms"], s["ttm_ms"], s["als_ms"]) for s in d["stages"]], d.get("clocks",{}).get("sm_mhz"))
    except Exception as e: print(c, "ERR", e)
PY
ATK_CFG=c5 timeout 300 python profiles/timeline_probe.py step gpurun_out/${TAG}_tl_step.json full > gpurun_out/${TAG}_gap_step.txt 2>&1; echo "step=$?"; head -3 gpurun_out/${TAG}_gap_step.txt | tail -1
