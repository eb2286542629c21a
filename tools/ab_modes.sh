# sigma / batch modes: this tree vs the tree under _old (previous commit)
mkdir -p gpurun_out
for t in . _old . _old; do
  (cd $t && python bench.py --mode batch --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t batch', d['batched_s'], d['sequential_s'])")
  (cd $t && python bench.py --mode sigma --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t sigma', d['ms_per_step'], d['e_step_ms_per_iter'], d['m_step_ms_per_iter'])")
done
