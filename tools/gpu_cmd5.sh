for flags in "" "-DUC_SGS_PARTIAL" "-DUC_SGS_MINB=4" "-DUC_SGS_PARTIAL -DUC_SGS_MINB=4" "-DUC_SGS_MINB=3"; do
python -c "
from paper_2006_16764_b200 import build as B
B.build(force=True, extra='$flags'.split())"
echo "== $flags"; python tools/vcycle_time.py --reps 10 | tail -1; python tools/vcycle_time.py --counts 256 256 256 --reps 3 | tail -1
done
