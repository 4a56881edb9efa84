mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_smem.py tests/test_gpu_c_abi.py -q -p no:cacheprovider > gpurun_out/q2_tests.log 2>&1
echo "rc $?" >> gpurun_out/q2_tests.log
python tools/oz_prof.py > gpurun_out/oz_prof.log 2>&1
timeout 900 python tools/bench_configs.py C1 C2 > gpurun_out/q2_configs.jsonl 2> gpurun_out/q2_configs.err
