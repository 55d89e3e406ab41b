#!/bin/bash
# One GPU-box pass of everything the driver runs at round end, plus the
# pipe probe:  gpurun -- 'bash tools/gpu/full_check.sh'
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
(cd tools/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe pipe_probe.cu && /tmp/pipe_probe) > gpurun_out/pipe_probe.txt 2>&1
