#!/bin/bash
# A/B of compile-time variants of the residual / Jv tiles: bench fill throughput
# (2D 2048^2, alloy 4096^2, 3D 256^3) per variant; rebuilds the default at the end.
cd "$(dirname "$0")/.."
for flags in "$@"; do
  python -c "
import sys; sys.path.insert(0,'.')
from paper_2006_16764_b200 import build
build.build(force=True, extra='$flags'.split())" || exit 1
  for wl in fg2d_2048 al2d_4096 fg3d_256; do
    r=$(timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-newton --no-cpu-baseline --no-extra 2>/dev/null | tail -1)
    python -c "
import json,sys; d=json.loads(sys.argv[1]); k=d.get('kernels',{})
print('$flags', '$wl', d['value'], k.get('residual_ms'), k.get('jv_ms'))" "$r"
  done
done
python -c "
import sys; sys.path.insert(0,'.')
from paper_2006_16764_b200 import build
build.build(force=True)"
