#!/bin/bash
# A/B compile flags on the lexicographic V-cycle: tools/gpu_ab_lex.sh -DFLAG [...]
for variant in "" "$@"; do
  python -c "from paper_2006_16764_b200.build import build; import sys; build(True, extra=sys.argv[1:])" $variant || exit 1
  echo "variant: ${variant:-default}"
  python tools/vcycle_time.py --counts 128 128 128 --reps 3 --builds 1 --ordering lexicographic | tail -1
  python tools/vcycle_time.py --counts 256 256 256 --reps 2 --builds 1 --ordering lexicographic | tail -1
done
