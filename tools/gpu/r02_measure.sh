# Round-2 measurement bundle on one B200 (each profiled command first runs
# without a profiler and must exit 0).
#   bash tools/gpu/r02_measure.sh
set -x
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python bench.py > $O/r02_bench.log 2>&1 || exit 1
timeout 600 python bench.py --impl reference > $O/r02_ref.log 2>&1
timeout 300 python tools/em64_capture.py 1000000 > $O/r02_capture_plain.log 2>&1 || exit 1
# launch list of the bench (short run; per-launch times are cold / serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/r02_launches.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e \
    > $O/r02_launches_run.log 2>&1
# full captures of k_em64: the 50-iteration registration (launch 1) and a pass alone (launch 2)
timeout 900 ncu --set full --import-source on -k 'regex:^k_em64$' -s 1 -c 2 -o $O/r02_em64_1m \
    python tools/em64_capture.py 1000000 > $O/r02_ncu_em64_1m.log 2>&1
timeout 900 ncu --set full --import-source on -k 'regex:^k_em64$' -s 2 -c 1 -o $O/r02_em64_16m_pass \
    python tools/em64_capture.py 16000000 --iters 4 > $O/r02_ncu_em64_16m.log 2>&1
# sanitizers on small problems: the grid-resident loop, the float32 loop, both batch drivers
# compute-sanitizer is closed on the GPU pool (runs under it left GPUs needing a reset)
for tool in ; do
  timeout 400 compute-sanitizer --tool $tool --print-limit 50 python tools/em64_capture.py 20000 \
      --iters 6 --f32 --batch > $O/r02_sanitizer_$tool.log 2>&1
done
ls -la $O
