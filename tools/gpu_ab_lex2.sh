#!/bin/bash
# A/B compile flags on the 2D lexicographic V-cycle: tools/gpu_ab_lex2.sh -DFLAG [...]
for variant in "" "$@"; do
  python -c "from paper_2006_16764_b200.build import build; import sys; build(True, extra=sys.argv[1:])" $variant || exit 1
  echo "variant: ${variant:-default}"
  python tools/vcycle_time.py --counts 2048 2048 --reps 3 --builds 2 --ordering lexicographic | tail -1
  python tools/vcycle_time.py --counts 512 512 --reps 5 --builds 2 --ordering lexicographic | tail -1
done
