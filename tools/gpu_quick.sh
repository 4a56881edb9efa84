timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py tests/test_gpu_smem.py -q -p no:cacheprovider -k "tcgen05 or shards or smem or C4_analogue or nccl" > gpurun_out/q_tests.log 2>&1; echo "rc $?" >> gpurun_out/q_tests.log
timeout 900 python tools/bench_configs.py C3 C4 auto > gpurun_out/q_configs.jsonl 2>&1
