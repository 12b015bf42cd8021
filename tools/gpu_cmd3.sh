for mb in 4 3 2; do
python -c "
from paper_2006_16764_b200 import build as B
B.build(force=True, extra=['-DUC_RES2D_MINB=$mb'])"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-newton 2>&1 | tail -1 > gpurun_out/b2d_$mb.json; python -c "import json;d=json.load(open('gpurun_out/b2d_$mb.json'));print('2D minb $mb',d['value'],d['kernels'])"
python bench.py --workload al2d_4096 --steps 10 --warmup 3 --no-cpu-baseline --no-newton 2>&1 | tail -1 > gpurun_out/ba_$mb.json; python -c "import json;d=json.load(open('gpurun_out/ba_$mb.json'));print('alloy minb $mb',d['value'],d['kernels'])"
done
