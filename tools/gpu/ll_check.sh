set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_noise.py tests/test_gpu_parity.py tests/test_gpu_stats.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/t1.log 2>&1; echo "rc=$?" >> gpurun_out/t1.log
for i in 1 2; do python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/b4_$i.log 2>&1; done
python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/b3.log 2>&1
