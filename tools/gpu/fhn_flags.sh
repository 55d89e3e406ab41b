#!/bin/bash
# FH-N lattice kernel variants by kernel flag:
#   gpurun -- 'bash tools/gpu/fhn_flags.sh TAG "0 8 0 8" [ncu-flag]'
set -u
mkdir -p gpurun_out/prof
TAG=${1:-x}; FLAGS=${2:-"0"}
L=gpurun_out/fhn_flags_$TAG.log
timeout 900 python -m pytest tests/test_gpu_noise.py -q -p no:cacheprovider -x -k "fhn" > $L 2>&1
echo "pytest rc=$?" >> $L
for f in $FLAGS; do
  echo "== kernel-flags $f" >> $L
  timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --profile --kernel-flags $f >> $L 2>&1
done
if [ -n "${3:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fhn_cm" -s 2 -c 1 -o gpurun_out/prof/fhn_$TAG -f \
    python bench.py --config cfg4 --steps 2 --warmup 2 --no-cpu-baseline --profile --kernel-flags $3 > gpurun_out/prof/fhn_$TAG.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/fhn_$TAG.ncu-rep > gpurun_out/prof/fhn_$TAG.txt 2>&1
fi
