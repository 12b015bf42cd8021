# Round-1 closing refresh after the 2D value-weight folding (r0w) (one GPU): instruction mix
# (regenerates profiles/dp_inst_per_element.json on the box before the bench lines read it),
# bench lines at every workload, fill launch list, one ncu --set full of k_residual NEW.
set -x
mkdir -p gpurun_out/r1f
python tools/kernel_mix.py > /dev/null 2>&1 && \
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,gpu__time_duration.sum \
    --clock-control none --csv -k regex:k_residual --log-file gpurun_out/r1f/kernel_mix_ncu.csv python tools/kernel_mix.py > /dev/null 2>&1
python tools/dp_mix.py gpurun_out/r1f/kernel_mix_ncu.csv > gpurun_out/r1f/dp_inst_per_element.json && \
    cp gpurun_out/r1f/dp_inst_per_element.json profiles/dp_inst_per_element.json
python bench.py > gpurun_out/r1f/bench.json 2> gpurun_out/r1f/bench.err
python bench.py --workload al2d_4096 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1f/bench_al.json 2> gpurun_out/r1f/bench_al.err
python bench.py --workload fg3d_256 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1f/bench_3d.json 2> gpurun_out/r1f/bench_3d.err
python bench.py --workload fg3d_512 --steps 5 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1f/bench_3d512.json 2> gpurun_out/r1f/bench_3d512.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1f/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o gpurun_out/r1f/prof_residual \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > gpurun_out/r1f/ncu_res.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1f/smoke.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1f/bench_ref.json 2> gpurun_out/r1f/bench_ref.err
python -m pytest tests -m gpu -q -x > gpurun_out/r1f/gputests.log 2>&1; echo tests_rc=$?
