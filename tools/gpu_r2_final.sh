#!/bin/bash
# Round-2 closing refresh on one GPU: bench lines (default + reference arm),
# launch lists of the fill and of 2D/3D Newton solves, ncu --set full of the top
# kernels (residual tile, 2D/3D line runs), smoke, GPU test suite.
# Outputs in gpurun_out/r2f (copied to profiles/r02 by hand).
D=gpurun_out/r2f; mkdir -p $D
python -c "import sys; sys.path.insert(0,'.'); from paper_2006_16764_b200 import build; build.build()"
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.json 2> $D/bench_ref.err; echo ref_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline --no-extra > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_newton_2d.csv \
    python tools/newton_step.py --counts 2048 2048 --reps 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_newton_3d.csv \
    python tools/newton_step.py --counts 256 256 256 --reps 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_vc2d.csv \
    python tools/vc_time.py --reps 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_vc3d.csv \
    python tools/vc_time.py --counts 256 256 256 --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o $D/prof_residual \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline --no-extra > $D/ncu_res.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line -s 0 -c 4 -o $D/prof_line2d \
    python tools/vc_time.py --counts 2048 2048 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line -s 0 -c 4 -o $D/prof_line3d \
    python tools/vc_time.py --counts 256 256 256 --reps 1 > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $D/gputests.log 2>&1; echo tests_rc=$? >> $D/gputests.log
tail -2 $D/gputests.log; head -c 400 $D/bench.json; echo; head -c 300 $D/bench_ref.json
