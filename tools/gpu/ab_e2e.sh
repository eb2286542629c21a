# A/B of register() fixed overhead and the 1M e2e between ab/libA.so and the in-tree build
mkdir -p gpurun_out; rm -f gpurun_out/ab_e2e.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo tests=$? >> gpurun_out/ab_tests.log
for r in 1 2; do for L in ab/libA.so paper_1811_10136_b200/libfilterreg_b200.so; do
  echo "== $L" >> gpurun_out/ab_e2e.log
  FR_LIB=$L timeout 300 python tools/register_overhead_probe.py 2>&1 | grep "register:" >> gpurun_out/ab_e2e.log
  FR_LIB=$L timeout 300 python tools/e2e_pinned_probe.py 10500 105000 1000000 >> gpurun_out/ab_e2e.log 2>&1
done; done
tail -2 gpurun_out/ab_tests.log
