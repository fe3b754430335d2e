"""Measure the roofline denominators the bench needs but MEASURED_PEAKS.json lacks.

python profiles/measure_peaks.py OUT.json

* tf32: torch.matmul fp32 8192^3 with TF32 tensor cores allowed (cuBLAS), 2 N^3 flop;
* fp64: torch.matmul fp64 8192^3 (cuBLAS DGEMM on DMMA);
* hbm: b.copy_(a) over 1 Gi fp32 elements (read + write bytes).
Each is measured as a burst (best of 10, CUDA events) and sustained (back to back for 4 s,
mean), the same recipe as the driver's MEASURED_PEAKS.json.  Clocks are sampled with
nvidia-smi during the sustained loops.
"""
from __future__ import annotations

import json
import subprocess
import sys
import time

import torch


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def measure(fn, work, sustain_s=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    burst = max(work / timed(fn, 1) for _ in range(10))
    # sustained: back to back for ~sustain_s seconds
    t1 = timed(fn, 1)
    reps = max(1, int(sustain_s / t1))
    q = "clocks.sm,power.draw,clocks_event_reasons.sw_power_cap"
    p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    time.sleep(0.2)
    sus = work / timed(fn, reps)
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    mhz = sorted(float(r.split(",")[0]) for r in out if r.split(",")[0].strip().replace(".", "").isdigit())
    return burst, sus, (mhz[len(mhz) // 2] if mhz else None)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "peaks.json"
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    res = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    bu, su, mhz = measure(lambda: torch.matmul(a, b, out=c), 2 * n ** 3)
    res["tf32_tflops"], res["tf32_tflops_sustained"], res["tf32_sm_mhz"] = bu / 1e12, su / 1e12, mhz
    del a, b, c
    a = torch.randn(n, n, device="cuda", dtype=torch.float64)
    b = torch.randn(n, n, device="cuda", dtype=torch.float64)
    c = torch.empty(n, n, device="cuda", dtype=torch.float64)
    bu, su, mhz = measure(lambda: torch.matmul(a, b, out=c), 2 * n ** 3)
    res["fp64_tflops"], res["fp64_tflops_sustained"], res["fp64_sm_mhz"] = bu / 1e12, su / 1e12, mhz
    del a, b, c
    m = 1 << 30
    a = torch.empty(m, device="cuda")
    b = torch.empty(m, device="cuda")
    a.fill_(1.0)
    bu, su, mhz = measure(lambda: b.copy_(a), 8 * m, sustain_s=2.0)
    res["hbm_gbs"], res["hbm_gbs_sustained"] = bu / 1e9, su / 1e9
    res["how"] = ("torch.matmul 8192^3 fp32 with allow_tf32 (cuBLAS tf32) and fp64 (cuBLAS DGEMM), 2N^3 flop; "
                  "copy_ of 1 Gi fp32 (read+write bytes); burst = best of 10 single launches, sustained = "
                  "back to back for 4 s (2 s for the copy), CUDA events")
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
