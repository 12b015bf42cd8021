# round 2: parity-run smoother (compile-time tiles): bits, timing, launch lists, ncu
set -x
D=gpurun_out/${RUN:-r2c}; mkdir -p $D
UC_SGS_PERCOLOR=1 python tools/pc_bits.py save $D/pc.npz > $D/bits.log 2>&1
python tools/pc_bits.py compare $D/pc.npz >> $D/bits.log 2>&1; echo bits_rc=$? >> $D/bits.log
for c in "2048 2048" "256 256 256"; do
  timeout 300 python tools/vc_time.py --counts $c --newton >> $D/time.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_2d.csv python tools/vc_time.py --counts 2048 2048 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_3d.csv python tools/vc_time.py --counts 256 256 256 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgs_run -s 0 -c 6 -o $D/prof_run2d python tools/vc_time.py --counts 2048 2048 --reps 1 > $D/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgs_run -s 0 -c 6 -o $D/prof_run3d python tools/vc_time.py --counts 256 256 256 --reps 1 > $D/ncu3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "precond or slab or lex or vcycle or multirank" > $D/tests.log 2>&1; echo tests_rc=$? >> $D/tests.log
cat $D/bits.log $D/time.log; tail -3 $D/tests.log
