# A/B of the dense-grid pass kernels (FR_GRID_KERNEL=3: cp.async ring, 3 pts/thread;
# 4: quarter-scale clamped pass, 4 consecutive points/thread from 16-byte loads)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_register.py tests/test_gpu_behaviour.py tests/test_gpu_batch.py -m gpu -x -q 2>&1 | tail -2
for v in 3 4 3 4; do
  FR_GRID_KERNEL=$v python bench.py --no-cpu-baseline --no-e2e --steps 400 > gpurun_out/v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('kernel=$v', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
