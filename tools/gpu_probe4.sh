mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/issue_probe tools/issue_probe.cu && timeout 120 /tmp/issue_probe > gpurun_out/issue_probe.txt 2>&1
echo "rc $?" >> gpurun_out/issue_probe.txt
