# A/B of the tiled pass: 4 points per trip at 2 CTAs/SM (default) vs two
# points at a time at 3 CTAs/SM (FR_TILES_HALVES=1)
mkdir -p gpurun_out
for v in "0" "1" "0" "1"; do set -- $v
  if [ "$1" = 1 ]; then export FR_TILES_HALVES=1; else unset FR_TILES_HALVES; fi
  python bench.py --no-cpu-baseline --no-e2e --steps 400 > gpurun_out/v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('halves=$1', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" || tail -3 gpurun_out/v.log; done
unset FR_TILES_HALVES
FR_TILES_HALVES=1 python -m pytest tests/test_gpu_tiled_loop.py -m gpu -x -q 2>&1 | tail -1
