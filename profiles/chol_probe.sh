#!/bin/bash
# chol_inv_kernel launch times vs CTA size (ATK_CHOL_THREADS) on ChFSI runs at k = 48 and k = 80
# usage: bash profiles/chol_probe.sh TAG [threads ...]
TAG=$1; shift
mkdir -p gpurun_out
for th in ${@:-256 512 1024}; do
  for nr in "1024 32" "2048 64"; do
    env ATK_CHOL_THREADS=$th ATK_PROFILE_NONCOOP=1 ${CHOL_ENV:-} ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      -k regex:chol_ --log-file gpurun_out/${TAG}_chol_${th}_${nr/ /_}.csv python profiles/cheb_probe.py $nr 1 > /dev/null 2>&1
    echo "threads=$th n,r=$nr: $(python profiles/launch_summary.py gpurun_out/${TAG}_chol_${th}_${nr/ /_}.csv | grep chol_)"
  done
done
