mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/pass_bench.json 2> gpurun_out/pass_bench.err
echo "bench rc $?" >> gpurun_out/pass_bench.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/pass_tests.log 2>&1
echo "rc $?" >> gpurun_out/pass_tests.log
