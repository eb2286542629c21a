# A/B of the tiled pass fold interval (FR_FOLD64=1: warp fold every 64 points per thread)
mkdir -p gpurun_out
for v in 0 1 0 1 0 1; do
  if [ "$v" = 1 ]; then export FR_FOLD64=1; else unset FR_FOLD64; fi
  python bench.py --no-cpu-baseline --no-e2e --steps 400 > gpurun_out/v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('fold64=$v', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" || tail -3 gpurun_out/v.log; done
unset FR_FOLD64
FR_FOLD64=1 python -m pytest tests/test_gpu_tiled_loop.py tests/test_gpu_register.py -m gpu -x -q 2>&1 | tail -1
