python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench4.log 2>&1; tail -1 gpurun_out/bench4.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['clocks'],d['newton'])"
python tools/newton_step.py --reps 1 > gpurun_out/plain_newton4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_newton4.csv python tools/newton_step.py --reps 1 > /dev/null 2>&1; echo l=$?
ncu --set full --clock-control none --import-source on -k regex:k_sgs_color -s 2000 -c 4 -o gpurun_out/prof_sgs4 python tools/newton_step.py --reps 1 > gpurun_out/ncu_sgs4.log 2>&1; echo p=$?
