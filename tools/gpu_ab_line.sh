#!/bin/bash
# A/B of compile-time variants of the line-run kernels: V-cycle apply times
# (2D 2048^2, 3D 256^3) per variant; rebuilds the default library at the end.
cd "$(dirname "$0")/.."
for flags in "$@"; do
  python -c "
import sys; sys.path.insert(0,'.')
from paper_2006_16764_b200 import build
build.build(force=True, extra='$flags'.split())" || exit 1
  echo "== $flags"
  timeout 120 python tools/vc_time.py --reps 20
  timeout 120 python tools/vc_time.py --counts 256 256 256 --reps 10
done
python -c "
import sys; sys.path.insert(0,'.')
from paper_2006_16764_b200 import build
build.build(force=True)"
