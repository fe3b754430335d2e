#!/bin/bash
# Gram K-launch size vs DRAM traffic (ncu) and step time (bench): gram_launch_kb 4096 (default) / 2048 / 1024 / 512
mkdir -p gpurun_out
for kb in 4096 2048 1024 512; do
  n=$((16 * 4096 / kb))
  ATK_OPTS=gram_launch_kb=$kb timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"gram_tf32_2cta|gram2_reduce" --csv --log-file gpurun_out/kb_$kb.csv python profiles/run_step.py c5 1 > /dev/null 2>&1
  python profiles/make_traffic.py gpurun_out/kb_$kb.csv gpurun_out/kb_$kb.json $n > /dev/null 2>&1
  timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --opt gram_launch_kb=$kb > gpurun_out/kbb_$kb.json 2>/dev/null
  python -c "import json;t=json.load(open('gpurun_out/kb_$kb.json'));d=json.load(open('gpurun_out/kbb_$kb.json'));print('kb=$kb', 'dram GB %.1f' % (t['dram_bytes_per_launch']/1e9), 'step', round(d['ms_per_step'],3), 'gram', d['stages'][0]['gram_ms'], d['clocks']['sm_mhz'])"
done
