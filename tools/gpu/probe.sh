set -u
mkdir -p gpurun_out
cd tools/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe pipe_probe.cu && /tmp/pipe_probe > ../../gpurun_out/pipe_probe.txt 2>&1
cat ../../gpurun_out/pipe_probe.txt
