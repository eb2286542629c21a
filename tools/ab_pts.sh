# A/B: points per thread per ring stage of the dense-grid pass
python -m pytest tests/test_gpu_register.py -m gpu -x -q 2>&1 | tail -1
FR_GRID_PTS=2 python -m pytest tests/test_gpu_register.py -m gpu -x -q 2>&1 | tail -1
for p in 1 2 1 2; do FR_GRID_PTS=$p python bench.py --no-cpu-baseline --no-e2e --steps 400 > gpurun_out/pts_$p.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/pts_$p.log').read().strip().splitlines()[-1]); print('pts=$p', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
