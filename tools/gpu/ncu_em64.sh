# ncu capture of one pass launch of the float64 EM kernel (k_em64) at the given size
# usage: bash tools/gpu/ncu_em64.sh <points> <tag> [variant]
set -x
export FR_EM64_VARIANT=${3:-2}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on -k regex:k_em64 -s 3 -c 1 -o gpurun_out/em64_$2 python tools/em64_probe.py $1 > gpurun_out/ncu_em64_$2.log 2>&1
