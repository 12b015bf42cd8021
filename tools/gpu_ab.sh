#!/bin/bash
# A/B a compile flag on the V-cycle timings: tools/gpu_ab.sh -DFLAG [...]
for variant in "" "$@"; do
  python -c "from paper_2006_16764_b200.build import build; import sys; build(True, extra=sys.argv[1:])" $variant || exit 1
  echo "variant: ${variant:-default}"
  python tools/vcycle_time.py --counts 256 256 256 --reps 10 --builds 2 | tail -1
  python tools/vcycle_time.py --counts 2048 2048 --reps 20 --builds 2 | tail -1
done
