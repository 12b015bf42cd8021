# Round-1 refresh: bench line, launch lists, ncu captures (run under gpurun, one GPU)
set -x
mkdir -p gpurun_out/r1b
python bench.py --steps 20 --warmup 5 > gpurun_out/r1b/bench.log 2>&1
python bench.py --workload al2d_4096 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1b/bench_al.log 2>&1
python bench.py --workload fg3d_256 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1b/bench_3d.log 2>&1
# launch lists (cold, serialised) of the same commands
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > gpurun_out/r1b/ncu_fill.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b/launches_newton.csv \
    python tools/newton_step.py --reps 1 > gpurun_out/r1b/ncu_newton.log 2>&1
# full captures of the dominant kernels
ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o gpurun_out/r1b/prof_residual \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > gpurun_out/r1b/ncu_res.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sgs_color -s 64 -c 4 -o gpurun_out/r1b/prof_sgs \
    python tools/newton_step.py --reps 1 > gpurun_out/r1b/ncu_sgs.log 2>&1
