#!/bin/bash
# One consolidated measurement session (round 2): tests, every config's bench line, the C5
# launch list, the Gram traffic and one ncu --set full capture of the Gram + TTM kernels.
TAG=${1:-r2f}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:hypothesispytest > gpurun_out/${TAG}_tests.log 2>&1
echo "tests=$? $(tail -1 gpurun_out/${TAG}_tests.log)"; grep -E "^FAILED|^ERROR" gpurun_out/${TAG}_tests.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$? $(tail -1 gpurun_out/${TAG}_smoke.log)"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err; echo "bench c5=$?"
for c in c1 c2 c3 c4 c5u; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c=$?"
done
python - <<PY
import json
for c in ["c5","c1","c2","c3","c4","c5u"]:
    try:
        d=json.load(open(f"gpurun_out/${TAG}_bench_{c}.json"))
        print(c, round(d["ms_per_step"],3), round(d["value"]), "e2e", round(d.get("e2e",{}).get("value",0)), [(s["gram_ms"], s["eig_ms"], s["ttm_ms"], s["als_ms"]) for s in d["stages"]], d.get("roofline",{}).get("frac"))
    except Exception as e: print(c, "ERR", e)
PY
ATK_PROFILE_NONCOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c5.csv python profiles/run_step.py c5 1 > /dev/null 2>&1; echo "launches=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"gram_tf32_2cta|gram2_reduce" --csv --log-file gpurun_out/${TAG}_gramtraffic.csv python profiles/run_step.py c5 1 > /dev/null 2>&1; echo "traffic=$?"
python profiles/make_traffic.py gpurun_out/${TAG}_gramtraffic.csv gpurun_out/${TAG}_gram_traffic.json | head -c 300; echo
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_tf32_2cta|ttm_tf32" -c 2 -o gpurun_out/${TAG}_full python profiles/run_step.py c5 1 > /dev/null 2>&1; echo "ncu=$?"
