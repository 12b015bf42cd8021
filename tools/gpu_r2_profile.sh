# round 2 profile refresh (one GPU): bench lines, launch lists, ncu --set full of the
# top kernels, instruction mix, smoke, reference arm, GPU test suite.  Outputs in gpurun_out/r2p.
set -x
D=gpurun_out/r2p; mkdir -p $D
python tools/kernel_mix.py > /dev/null 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum \
    --clock-control none --csv -k regex:k_residual --log-file $D/kernel_mix_ncu.csv python tools/kernel_mix.py > /dev/null 2>&1
python tools/dp_mix.py $D/kernel_mix_ncu.csv > $D/dp_inst_per_element.json && cp $D/dp_inst_per_element.json profiles/dp_inst_per_element.json
python bench.py > $D/bench.json 2> $D/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline --no-extra > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_newton_2d.csv \
    python tools/newton_step.py --counts 2048 2048 --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_newton_3d.csv \
    python tools/newton_step.py --counts 256 256 256 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o $D/prof_residual \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline --no-extra > $D/ncu_res.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgs_run -s 0 -c 6 -o $D/prof_run2d python tools/vc_time.py --counts 2048 2048 --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgs_run -s 0 -c 6 -o $D/prof_run3d python tools/vc_time.py --counts 256 256 256 --reps 1 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.json 2> $D/bench_ref.err
python -m pytest tests -m gpu -q -x > $D/gputests.log 2>&1; echo tests_rc=$? >> $D/gputests.log
tail -2 $D/gputests.log; cat $D/bench.json | head -c 600; echo; cat $D/bench_ref.json | head -c 400
