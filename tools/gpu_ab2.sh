#!/bin/bash
# A/B compile variants on the V-cycle apply time: tools/gpu_ab2.sh "counts" "-DA=1" "-DB=2" ...
counts="$1"; shift
for variant in "$@"; do
  python -c "from paper_2006_16764_b200.build import build; import sys; build(True, extra=sys.argv[1:])" $variant || exit 1
  echo "variant: ${variant:-default} $(python tools/vc_time.py --counts $counts --reps 20 | tail -1)"
done
python -c "from paper_2006_16764_b200.build import build; build(True)"
