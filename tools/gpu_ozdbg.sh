mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_ab_switches.py tests/test_gpu_fp64.py -q -p no:cacheprovider > gpurun_out/oz_tests.log 2>&1
echo "rc $?" >> gpurun_out/oz_tests.log
python tools/oz_prof.py > gpurun_out/oz_prof.log 2>&1
