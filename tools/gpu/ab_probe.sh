mkdir -p gpurun_out; rm -f gpurun_out/ab_probe.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo tests=$? >> gpurun_out/ab_tests.log
for r in 1 2; do for L in ab/libA.so paper_1811_10136_b200/libfilterreg_b200.so; do echo "== $L" >> gpurun_out/ab_probe.log; FR_LIB=$L FR_EM64_PROFILE=1 timeout 300 python tools/em64_probe.py 1000000 100000 10500 >> gpurun_out/ab_probe.log 2>&1; done; done
tail -2 gpurun_out/ab_tests.log
