# Round-end measurement set (run on the GPU box from the repo root):
# default bench line, reference arm, sigma / batch modes, launch list, full
# captures of the per-iteration pass kernel and the splat site sums.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-400
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
python bench.py --mode sigma --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sigma.log 2>&1; tail -1 gpurun_out/bench_sigma.log | cut -c1-300
python bench.py --mode batch --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_batch.log 2>&1; tail -1 gpurun_out/bench_batch.log | cut -c1-300
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rigid_pass_tiles -s 5 -c 1 \
    -o gpurun_out/pass_only_full python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full0.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rigid_pass_tiles -s 25 -c 1 \
    -o gpurun_out/pass_full python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_splat_segsum -s 1 -c 1 \
    -o gpurun_out/segsum_full python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_seg.log 2>&1
ls -la gpurun_out | tail -12
