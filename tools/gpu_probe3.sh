mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mma_rate_probe tools/mma_rate_probe.cu && timeout 120 /tmp/mma_rate_probe > gpurun_out/mma_rate_probe2.txt 2>&1
echo "probe rc $?" >> gpurun_out/mma_rate_probe2.txt
