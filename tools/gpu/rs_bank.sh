#!/bin/bash
# cfg1b bank resampler timing (sigma 1 / 10) per PF_RS flag set, 2 repeats:
#   gpurun -- 'bash tools/gpu/rs_bank.sh TAG "0 16"'
set -u
TAG=${1:-x}; FLAGS=${2:-0}; L=gpurun_out/rs_bank_$TAG.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bank or multinomial or cfg1 or pipelined" > $L 2>&1
echo "pytest rc=$?" >> $L
for i in 1 2; do for f in $FLAGS; do for sg in 1 10; do
  timeout 300 python bench.py --config cfg1b --sigma $sg --steps 20 --warmup 3 --no-cpu-baseline --kernel-flags $f 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('flags $f sigma $sg', json.dumps({'ms':d['ms_per_step'],'frac':d['roofline']['frac']}))" >> $L
done; done; done
if [ -n "${3:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:resample_bank" -s 2 -c 1 -o gpurun_out/prof/rsb_$TAG -f python bench.py --config cfg1b --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/rsb_$TAG.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/rsb_$TAG.ncu-rep > gpurun_out/prof/rsb_$TAG.txt 2>&1
fi
