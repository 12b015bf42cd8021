cd "$(dirname "$0")/.."
D=gpurun_out/r2g; mkdir -p $D
python -c "import sys; sys.path.insert(0,'.'); from paper_2006_16764_b200 import build; build.build()"
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; echo bench_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_residual -s 4 -c 2 -o $D/prof_residual \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline --no-extra > $D/ncu_res.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_fill.csv \
    python bench.py --steps 2 --warmup 3 --no-newton --no-cpu-baseline --no-extra > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $D/gputests.log 2>&1; echo tests_rc=$? >> $D/gputests.log
tail -2 $D/gputests.log; head -c 300 $D/bench.json
