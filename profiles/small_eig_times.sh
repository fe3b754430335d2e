#!/bin/bash
# ncu launch times of the dense tridiagonal eig kernels for the given n (default 32 48 64 128)
# usage: bash profiles/small_eig_times.sh TAG [n ...]
TAG=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"trd|bisect|invit|backtr" --log-file gpurun_out/${TAG}_small_eig.csv \
    python profiles/trd_probe.py ${@:-32 48 64 128} > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/${TAG}_small_eig.csv
