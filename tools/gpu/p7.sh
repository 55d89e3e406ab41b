#!/bin/bash
# Philox rounds experiment: lib_var/p10 (production, 10 rounds) against lib_var/p7
# (-DPF_PHILOX_ROUNDS=7) on the two propagate workloads, then the noise-law and
# statistical-parity tests on the 7-round build (the known-answer tests fail on it by
# design and are not run).
set -u
bash tools/gpu/ab_lib.sh cfg4 p10 p7
bash tools/gpu/ab_lib.sh cfg2 p10 p7
cp paper_1407_8071_b200/lib/libpfbank.so /tmp/libpfbank.keep.so
cp lib_var/p7/libpfbank.so paper_1407_8071_b200/lib/libpfbank.so
python -m pytest tests/test_gpu_noise.py tests/test_gpu_stats.py -m gpu -q -p no:cacheprovider > gpurun_out/p7_tests.log 2>&1
echo "rc=$?" >> gpurun_out/p7_tests.log
cp /tmp/libpfbank.keep.so paper_1407_8071_b200/lib/libpfbank.so
for f in gpurun_out/ab_cfg*_p*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"].get("kernel_ms"))')"; done
tail -3 gpurun_out/p7_tests.log
