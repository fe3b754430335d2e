#!/bin/bash
# bisect_kernel warps per CTA x Sturm chains per lane (ATK_BIS_WPB / ATK_BIS_C probe knobs)
for w in 8 2 1; do for c in 1 2 4; do
  echo "wpb=$w C=$c $(ATK_BIS_WPB=$w ATK_BIS_C=$c timeout 120 python profiles/timeline_probe.py eig gpurun_out/bs.json 2>&1 | grep -E ' bisect' | head -1) $(ATK_BIS_WPB=$w ATK_BIS_C=$c timeout 120 python profiles/bigeig_timeline.py 2048 3 2>&1 | grep -E ' bisect' | head -1)"
done; done
