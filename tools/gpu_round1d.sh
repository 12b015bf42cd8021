# Round-1 closing refresh (one GPU): bench lines at every workload + the reference arm
set -x
mkdir -p gpurun_out/r1d
python bench.py > gpurun_out/r1d/bench.json 2> gpurun_out/r1d/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1d/bench_ref.json 2> gpurun_out/r1d/bench_ref.err
python bench.py --workload al2d_4096 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1d/bench_al.json 2> gpurun_out/r1d/bench_al.err
python bench.py --workload fg3d_256 --steps 10 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1d/bench_3d.json 2> gpurun_out/r1d/bench_3d.err
python bench.py --workload fg3d_512 --steps 5 --warmup 3 --no-cpu-baseline --no-lex > gpurun_out/r1d/bench_3d512.json 2> gpurun_out/r1d/bench_3d512.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline > /dev/null 2>&1
