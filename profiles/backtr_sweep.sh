#!/bin/bash
# backtr_kernel vectors (warps) per CTA (ATK_BACKTR_BW probe knob), C5's Rayleigh-Ritz block
for b in 32 16 8 4 2; do
  echo "bw=$b $(ATK_BACKTR_BW=$b timeout 120 python profiles/timeline_probe.py eig gpurun_out/bt.json 2>&1 | grep -E ' backtr' | head -1)"
done
