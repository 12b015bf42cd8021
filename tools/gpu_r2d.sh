# round 2: newton breakdown, drop-in + multirank tests
set -x
D=gpurun_out/r2d; mkdir -p $D
timeout 300 python tools/vc_time.py --counts 2048 2048 --newton > $D/time.log 2>&1
UC_SGS_PERCOLOR=1 timeout 300 python tools/vc_time.py --counts 2048 2048 --newton >> $D/time.log 2>&1
timeout 600 python -m pytest tests/test_dropin.py tests/test_gpu_multirank.py -x -q > $D/tests.log 2>&1; echo tests_rc=$? >> $D/tests.log
cat $D/time.log; tail -30 $D/tests.log
