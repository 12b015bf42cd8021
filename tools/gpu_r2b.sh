# round 2: parity-run smoother timing + launch list + ncu of the run kernels
set -x
D=gpurun_out/r2b; mkdir -p $D
python tools/pc_bits.py compare gpurun_out/r2a/pc.npz > $D/bits.log 2>&1; echo bits_rc=$? >> $D/bits.log
for c in "2048 2048" "256 256 256"; do
  timeout 300 python tools/vc_time.py --counts $c >> $D/time.log 2>&1
done
UC_SGS_PERCOLOR=1 timeout 300 python tools/vc_time.py --counts 2048 2048 >> $D/time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_2d.csv python tools/vc_time.py --counts 2048 2048 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_3d.csv python tools/vc_time.py --counts 256 256 256 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgs_run -s 0 -c 6 -o $D/prof_run2d python tools/vc_time.py --counts 2048 2048 --reps 1 > $D/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgs_run -s 0 -c 6 -o $D/prof_run3d python tools/vc_time.py --counts 256 256 256 --reps 1 > $D/ncu3.log 2>&1
cat $D/bits.log $D/time.log
