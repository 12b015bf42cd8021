timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b2d.json; python -c "import json;d=json.load(open('gpurun_out/b2d.json'));print('2D',d['value'],d['kernels'],d['newton']['sec_per_newton_iteration'],d['newton']['vcycle_apply_ms'])"
python bench.py --workload fg3d_256 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b3d.json; python -c "import json;d=json.load(open('gpurun_out/b3d.json'));print('3D minb2',d['value'],d['kernels'],d['newton'])"
python -c "
from paper_2006_16764_b200 import build as B
B.build(force=True, extra=['-DUC_RES3D_MINB=1'])"
python bench.py --workload fg3d_256 --steps 10 --warmup 3 --no-cpu-baseline --no-newton 2>&1 | tail -1 > gpurun_out/b3d1.json; python -c "import json;d=json.load(open('gpurun_out/b3d1.json'));print('3D minb1',d['value'],d['kernels'])"
