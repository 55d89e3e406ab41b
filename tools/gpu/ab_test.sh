#!/bin/bash
# A/B of lib_var/<variant> against lib_var/p10 on one workload, then the FH-N parity and
# noise tests on the variant:  bash tools/gpu/ab_test.sh cfg4 split
set -u
cfg=$1; v=$2
bash tools/gpu/ab_lib.sh $cfg p10 $v
cp paper_1407_8071_b200/lib/libpfbank.so /tmp/libpfbank.keep.so
cp lib_var/$v/libpfbank.so paper_1407_8071_b200/lib/libpfbank.so
timeout 900 python -m pytest tests/test_gpu_noise.py tests/test_gpu_guard.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${v}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${v}_tests.log
cp /tmp/libpfbank.keep.so paper_1407_8071_b200/lib/libpfbank.so
for f in gpurun_out/ab_${cfg}_*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"].get("kernel_ms"))')"; done
tail -4 gpurun_out/${v}_tests.log
