# A/B of the device-loop iteration: FR_EM_FUSED=0 (tiled pass + separate solver
# kernel) vs the fused tail (last block reduces and solves)
mkdir -p gpurun_out
for v in "1" "0" "1" "0"; do set -- $v
  FR_EM_FUSED=$1 python bench.py --no-cpu-baseline --no-e2e --steps 400 > gpurun_out/v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('fused=$1', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" || tail -3 gpurun_out/v.log; done
