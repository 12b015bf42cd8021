set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > gpurun_out/plain_fill.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fill.csv python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > /dev/null 2>&1; echo l1=$?
python tools/newton_step.py --reps 1 > gpurun_out/plain_newton.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_newton.csv python tools/newton_step.py --reps 1 > /dev/null 2>&1; echo l2=$?
ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o gpurun_out/prof_residual python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > gpurun_out/ncu_res.log 2>&1; echo p1=$?
ncu --set full --clock-control none --import-source on -k regex:k_sgs_color -s 64 -c 4 -o gpurun_out/prof_sgs python tools/newton_step.py --reps 1 > gpurun_out/ncu_sgs.log 2>&1; echo p2=$?
