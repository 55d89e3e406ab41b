#!/bin/bash
# Compact-CDF wide resampler (wide4) vs the materialised CDF (PF_RS_WIDE_MATERIALISE=8):
#   gpurun -- 'bash tools/gpu/w4.sh TAG [ncu]'
set -u
mkdir -p gpurun_out/prof
TAG=${1:-x}
L=gpurun_out/w4_$TAG.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "wide or production or chunked or cfg1 or collapse" > $L 2>&1
echo "pytest rc=$?" >> $L
for sg in 1 10; do for f in 0 8 0 8; do
  echo "== sigma $sg flags $f" >> $L
  timeout 600 python bench.py --config cfg1c --sigma $sg --steps 10 --warmup 3 --no-cpu-baseline --kernel-flags $f 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(json.dumps({'ms':d['ms_per_step'],'frac':d['roofline']['frac'],'e2e':d['e2e']['value']}))
    else: print(l.rstrip())" >> $L
done; done
if [ "${2:-}" = "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/w4_launches_$TAG.csv python bench.py --config cfg1c --steps 3 --warmup 3 --no-cpu-baseline --profile > gpurun_out/prof/w4_launches_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:wide4_merge" -s 2 -c 1 -o gpurun_out/prof/w4m_$TAG -f python bench.py --config cfg1c --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/w4m_$TAG.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/w4m_$TAG.ncu-rep > gpurun_out/prof/w4m_$TAG.txt 2>&1
fi
