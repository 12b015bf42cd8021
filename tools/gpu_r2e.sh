# round 2: new GPU tests + full default bench
set -x
D=gpurun_out/r2e; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_reference_driver.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_dropin.py -x -q > $D/tests.log 2>&1; echo tests_rc=$? >> $D/tests.log
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; echo bench_rc=$? >> $D/bench.err
tail -15 $D/tests.log; tail -3 $D/bench.err; cat $D/bench.json
