#!/bin/bash
# cfg1b bank resampler timing (sigma 1 / 10), 3 repeats:  gpurun -- 'bash tools/gpu/rs_bank.sh TAG'
set -u
TAG=${1:-x}; L=gpurun_out/rs_bank_$TAG.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bank or multinomial or cfg1" > $L 2>&1
echo "pytest rc=$?" >> $L
for i in 1 2; do for sg in 1 10; do
  timeout 300 python bench.py --config cfg1b --sigma $sg --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('sigma $sg', json.dumps({'ms':d['ms_per_step'],'frac':d['roofline']['frac']}))" >> $L
done; done
