#!/bin/bash
# Packed-fp32 (FFMA2) FH-N lattice kernel vs its scalar-issue form:
#   gpurun -- 'bash tools/gpu/x2_fhn.sh TAG [ncu]'
set -u
mkdir -p gpurun_out/prof
TAG=${1:-x}
L=gpurun_out/x2_fhn_$TAG.log
(cd tools/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe pipe_probe.cu && /tmp/pipe_probe) > gpurun_out/pipe_probe_$TAG.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_noise.py -q -p no:cacheprovider -x -k "fhn" > $L 2>&1
echo "pytest rc=$?" >> $L
for f in 0 4 0 4; do
  echo "== kernel-flags $f" >> $L
  timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --profile --kernel-flags $f >> $L 2>&1
done
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --profile >> $L 2>&1
if [ "${2:-}" = "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fhn_cm" -s 2 -c 1 -o gpurun_out/prof/fhn_$TAG -f \
    python bench.py --config cfg4 --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/fhn_$TAG.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/fhn_$TAG.ncu-rep > gpurun_out/prof/fhn_$TAG.txt 2>&1
fi
