# Round-1 final refresh (one GPU): bench lines, instruction mix, launch lists, ncu captures
set -x
mkdir -p gpurun_out/r1c
python bench.py --steps 20 --warmup 5 > gpurun_out/r1c/bench.log 2>&1
python bench.py --workload al2d_4096 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1c/bench_al.log 2>&1
python bench.py --workload fg3d_256 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1c/bench_3d.log 2>&1
python tools/kernel_mix.py > /dev/null 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum \
    --clock-control none --csv -k regex:k_residual --log-file gpurun_out/r1c/mix.csv python tools/kernel_mix.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > /dev/null 2>&1
python tools/newton_step.py --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c/launches_newton.csv \
    python tools/newton_step.py --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o gpurun_out/r1c/prof_residual \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > gpurun_out/r1c/ncu_res.log 2>&1
