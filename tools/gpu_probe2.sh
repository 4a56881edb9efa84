mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/i8mma_probe tools/i8mma_probe.cu && timeout 120 /tmp/i8mma_probe > gpurun_out/i8mma_probe2.txt 2>&1
echo "probe rc $?" >> gpurun_out/i8mma_probe2.txt
timeout 300 python tools/det_check.py > gpurun_out/det_check.txt 2>&1
