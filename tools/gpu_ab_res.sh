#!/bin/bash
# A/B compile flags on the residual/Jv fill: [BENCH_ARGS=...] tools/gpu_ab_res.sh "-DA=1 -DB=2" [...]
for variant in "" "$@"; do
  python -c "from paper_2006_16764_b200.build import build; import sys; build(True, extra=sys.argv[1:])" $variant || exit 1
  echo "variant: ${variant:-default}"
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -x 2>&1 | tail -1
  python bench.py --steps 10 --warmup 3 --no-newton --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['kernels'])"
done
