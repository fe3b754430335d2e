#!/bin/bash
# Where the C5 eigensolve's time goes between kernels: CUPTI timeline of one eig (full listing)
# and of one C5 step, plus the CholeskyQR orthogonality defect entering each pass.
mkdir -p gpurun_out
timeout 300 python profiles/timeline_probe.py eig gpurun_out/tl_eig.json full > gpurun_out/gap_eig.txt 2>&1; echo "eig=$?"
ATK_TRACE_QR=1 timeout 300 python profiles/timeline_probe.py eig gpurun_out/tl_eig2.json > gpurun_out/gap_qr.txt 2>&1; echo "qr=$?"
ATK_CFG=c5 timeout 300 python profiles/timeline_probe.py step gpurun_out/tl_step.json full > gpurun_out/gap_step.txt 2>&1; echo "step=$?"
