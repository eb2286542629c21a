# A/B of dense-grid pass variants (FR_GRID_KERNEL=3: cp.async ring, 3 pts/thread;
# 4: grid4, shared-memory constants; 5: grid4 with constant-bank constants;
# FR_GRID_TILES=0: device loop without the centred tiled copy of the points)
mkdir -p gpurun_out
for v in "5 1" "5 0" "5 1" "5 0"; do set -- $v
  FR_GRID_TILES=$2 FR_GRID_KERNEL=$1 python bench.py --no-cpu-baseline --no-e2e --steps 400 > gpurun_out/v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('kernel=$1 tiles=$2', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" || tail -3 gpurun_out/v.log; done
