#!/bin/bash
# One GPU session: tests, bench, reference arm, launch list, ncu captures.
# Usage: bash profiles/gpu_round.sh TAG [parts...]  (parts: tests bench ref launches ncu)
TAG=$1; shift
PARTS=${@:-tests bench ref launches ncu}
mkdir -p gpurun_out
python __graft_entry__.py >/dev/null 2>&1 || true
for p in $PARTS; do
  case $p in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q -p no:hypothesispytest > gpurun_out/${TAG}_tests.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_tests.log)";;
    slow) timeout 1500 python -m pytest tests -m "gpu and slow" -x -q -s -p no:hypothesispytest > gpurun_out/${TAG}_slow.log 2>&1; echo "slow=$? $(tail -1 gpurun_out/${TAG}_slow.log)";;
    probe) ATK_TRACE=1 timeout 600 python tests/eig_probe.py 2048 > gpurun_out/${TAG}_probe.log 2>&1; echo "probe=$?"; grep -vE "^\[atk eig n=2048" gpurun_out/${TAG}_probe.log | tail -12;;
    trace) ATK_TRACE=1 timeout 300 python profiles/run_step.py c5 2 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace=$?"; tail -40 gpurun_out/${TAG}_trace.log;;
    eigt) timeout 300 python -m pytest tests/test_gpu_eig.py -x -q -p no:hypothesispytest > gpurun_out/${TAG}_eigt.log 2>&1; echo "eigt=$? $(tail -1 gpurun_out/${TAG}_eigt.log)";;
    ncujac) timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi1s -c 1 -o gpurun_out/${TAG}_jac python profiles/jacobi_probe.py 96 > gpurun_out/${TAG}_ncujac.log 2>&1; echo "ncujac=$?";;
    allcfg) for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c=$?"; head -c 300 gpurun_out/${TAG}_bench_$c.json; echo; done;;
    tracecfg) for c in c1 c2; do ATK_TRACE=1 timeout 300 python profiles/run_step.py $c 1 > gpurun_out/${TAG}_trace_$c.log 2>&1; echo "trace $c=$?"; done;;
    c5u) timeout 600 python bench.py --config c5u --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c5u.json 2> gpurun_out/${TAG}_bench_c5u.err; echo "c5u=$?";;
    peaks) timeout 300 python profiles/measure_peaks.py gpurun_out/${TAG}_peaks.json > gpurun_out/${TAG}_peaks.log 2>&1; echo "peaks=$?"; tail -c 600 gpurun_out/${TAG}_peaks.json; echo;;
    bigeig) ATK_TRD_PROFILE=1 timeout 600 python profiles/eig_big_probe.py > gpurun_out/${TAG}_bigeig.log 2>&1; echo "bigeig=$?"; grep -E "dense eig|trd n|method=|Error|error" gpurun_out/${TAG}_bigeig.log | tail -30;;
    bigeigt) timeout 900 python -m pytest tests/test_gpu_eig_big.py -x -q -p no:hypothesispytest > gpurun_out/${TAG}_bigeigt.log 2>&1; echo "bigeigt=$? $(tail -1 gpurun_out/${TAG}_bigeigt.log)"; grep -E "Error|assert|FAIL" gpurun_out/${TAG}_bigeigt.log | head -20;;
    c5ueig) ATK_TRACE=1 timeout 600 python profiles/c5u_eig_probe.py > gpurun_out/${TAG}_c5ueig.log 2>&1; echo "c5ueig=$?"; grep -E "^method|hand|dense|passes" gpurun_out/${TAG}_c5ueig.log | tail -30;;
    dist) timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -p no:hypothesispytest > gpurun_out/${TAG}_dist.log 2>&1; echo "dist=$? $(tail -1 gpurun_out/${TAG}_dist.log)"; grep -E "Error|assert" gpurun_out/${TAG}_dist.log | head -20;;
    cpp) timeout 600 python -m pytest tests/test_gpu_cpp.py tests/test_cpp_types.py -x -q -p no:hypothesispytest > gpurun_out/${TAG}_cpp.log 2>&1; echo "cpp=$? $(tail -1 gpurun_out/${TAG}_cpp.log)";;
    eigall) timeout 1200 python -m pytest tests/test_gpu_eig.py tests/test_gpu_eig_big.py tests/test_gpu_tridiag.py tests/test_gpu_svd.py -q -p no:hypothesispytest > gpurun_out/${TAG}_eigall.log 2>&1; echo "eigall=$? $(tail -1 gpurun_out/${TAG}_eigall.log)"; grep -E "^FAILED|Error" gpurun_out/${TAG}_eigall.log | head -20;;
    full) timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:hypothesispytest > gpurun_out/${TAG}_full.log 2>&1; echo "full=$? $(tail -1 gpurun_out/${TAG}_full.log)"; grep -E "full:|FAILED" gpurun_out/${TAG}_full.log;;
    eigc5) timeout 600 python profiles/eig_c5_probe.py > gpurun_out/${TAG}_eigc5.log 2>&1; echo "eigc5=$?"; tail -30 gpurun_out/${TAG}_eigc5.log;;
    eigtrace) timeout 600 python profiles/eig_c5_trace.py > gpurun_out/${TAG}_eigtrace.log 2>&1; echo "eigtrace=$?"; tail -40 gpurun_out/${TAG}_eigtrace.log;;
    fast) timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:hypothesispytest > gpurun_out/${TAG}_tests.log 2>&1; echo "fast=$? $(tail -1 gpurun_out/${TAG}_tests.log)";;
    bench) timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench=$?"; head -c 400 gpurun_out/${TAG}_bench.json; echo;;
    ref) timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref=$?"; head -c 300 gpurun_out/${TAG}_ref.json; echo;;
    launches) ATK_PROFILE_NONCOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python profiles/run_step.py ${CFG:-c5} 1 > gpurun_out/${TAG}_launches.log 2>&1; echo "launches=$?";;
    traffic) timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"gram_tf32_2cta|gram2_reduce" --csv --log-file gpurun_out/${TAG}_gramtraffic.csv python profiles/run_step.py c5 1 > gpurun_out/${TAG}_traffic.log 2>&1; echo "traffic=$?"; python profiles/make_traffic.py gpurun_out/${TAG}_gramtraffic.csv gpurun_out/${TAG}_gram_traffic.json | head -c 300; echo;;
    ncueig) timeout 600 ncu --set full --clock-control none --import-source on -k regex:"trd_|invit_kernel|bisect_kernel|backtr_kernel|dgemm_tile|chol_inv" -c 8 -o gpurun_out/${TAG}_eig python profiles/run_step.py c5 1 > gpurun_out/${TAG}_ncueig.log 2>&1; echo "ncueig=$?";;
    ncucheb) ATK_PROFILE_NONCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cheb_" -c 2 -o gpurun_out/${TAG}_cheb python profiles/run_step.py c2 1 > gpurun_out/${TAG}_ncucheb.log 2>&1; echo "ncucheb=$?";;
    ncu) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_tf32_2cta|ttm_tf32" -c 2 -o gpurun_out/${TAG}_full python profiles/run_step.py c5 1 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu=$?";;
  esac
done
