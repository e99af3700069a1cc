nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/scratch/stream_probe.cu && /tmp/stream_probe > gpurun_out/stream_probe.txt 2>&1
cat gpurun_out/stream_probe.txt
