#!/bin/bash
# ChFSI skinny DMMA GEMMs under different minimum split-K chunks (ATK_DGEMM_MIN_CHUNK probe knob)
for c in 32 64 128 256 512; do
  echo "min_chunk=$c $(ATK_DGEMM_MIN_CHUNK=$c timeout 120 python profiles/timeline_probe.py eig gpurun_out/dc.json 2>&1 | grep -E 'span|dgemm' | tr '\n' ' ')"
done
