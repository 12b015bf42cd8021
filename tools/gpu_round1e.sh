# Round-1 closing refresh after the flux/heat-weight folding (one GPU): instruction mix
# (regenerates profiles/dp_inst_per_element.json on the box before the bench lines read it),
# bench lines at every workload, fill launch list, one ncu --set full of k_residual NEW.
set -x
mkdir -p gpurun_out/r1e
python tools/kernel_mix.py > /dev/null 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum \
    --clock-control none --csv -k regex:k_residual --log-file gpurun_out/r1e/kernel_mix_ncu.csv python tools/kernel_mix.py > /dev/null 2>&1
python tools/dp_mix.py gpurun_out/r1e/kernel_mix_ncu.csv > gpurun_out/r1e/dp_inst_per_element.json && \
    cp gpurun_out/r1e/dp_inst_per_element.json profiles/dp_inst_per_element.json
python bench.py > gpurun_out/r1e/bench.json 2> gpurun_out/r1e/bench.err
python bench.py --workload al2d_4096 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1e/bench_al.json 2> gpurun_out/r1e/bench_al.err
python bench.py --workload fg3d_256 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1e/bench_3d.json 2> gpurun_out/r1e/bench_3d.err
python bench.py --workload fg3d_512 --steps 5 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1e/bench_3d512.json 2> gpurun_out/r1e/bench_3d512.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1e/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o gpurun_out/r1e/prof_residual \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > gpurun_out/r1e/ncu_res.log 2>&1
