# one-CTA persistent EM (FR_EM_CLUSTER=0) vs the 8-CTA cluster EM, C1 end to end and the batch protocol
mkdir -p gpurun_out
python -m pytest tests/test_gpu_register.py tests/test_gpu_batch.py tests/test_gpu_behaviour.py -m gpu -x -q 2>&1 | tail -1
for v in 0 1 0 1; do
  FR_EM_CLUSTER=$v python tools/configs_timing.py 2>&1 | grep '^C1' | python -c "import json,sys; l=sys.stdin.read(); d=json.loads(l[3:]); print('cluster=$v C1', d['wall_s'], d['iterations'], d['speedup_wall'])"
  FR_EM_CLUSTER=$v python bench.py --mode batch 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cluster=$v batch', d['batched_s'], d['sequential_s'], d['identical_to_sequential'])"
done
