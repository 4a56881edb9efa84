mkdir -p gpurun_out
python tools/tc_ab.py 2 > gpurun_out/tc_ab.log 2>&1; echo "rc $?" >> gpurun_out/tc_ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tcgen05 or store_steps" -p no:cacheprovider > gpurun_out/tc_parity.log 2>&1; echo "rc $?" >> gpurun_out/tc_parity.log
