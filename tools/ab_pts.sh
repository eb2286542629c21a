# A/B of the dense-grid pass variants: points per thread x CTAs per SM
FR_GRID_PTS=3 python -m pytest tests/test_gpu_register.py -m gpu -x -q 2>&1 | tail -1
for v in "2 2" "3 2" "2 2" "3 2"; do set -- $v
  FR_GRID_PTS=$1 FR_GRID_MINB=$2 python bench.py --no-cpu-baseline --no-e2e --steps 400 > gpurun_out/v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('pts=$1 minb=$2', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
