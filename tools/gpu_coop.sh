mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coop.py -x -q -p no:cacheprovider > gpurun_out/coop_tests.log 2>&1
echo "rc $?" >> gpurun_out/coop_tests.log
timeout 600 python tools/bench_configs.py C2 > gpurun_out/coop_configs.jsonl 2> gpurun_out/coop_configs.err
