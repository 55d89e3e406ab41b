set -u
mkdir -p gpurun_out/prof
timeout 2400 python -m pytest tests/test_gpu_graph.py tests/test_gpu_noise.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_apf.py tests/test_gpu_fhnnet.py tests/test_gpu_small.py tests/test_gpu_verify.py tests/test_gpu_data.py -q -p no:cacheprovider -rs -s -x > gpurun_out/r2_gputest4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest4.log
for c in cfg4 cfg0 cfg3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench4_$c.log 2>&1
  echo "bench rc=$?" >> gpurun_out/r2_bench4_$c.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fhn_ws_kernel" -s 2 -c 1 -o gpurun_out/prof/fhn_ws_r2a -f \
    python bench.py --config cfg4 --steps 2 --warmup 2 --no-cpu-baseline --profile > gpurun_out/prof/fhn_ws_r2a.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof/fhn_ws_r2a.log
timeout 1500 python -m pytest tests/test_gpu_sanitize.py -q -p no:cacheprovider -rs > gpurun_out/r2_sanitize.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_sanitize.log
