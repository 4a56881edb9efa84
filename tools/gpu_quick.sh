timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "tcgen05" > gpurun_out/q_tests.log 2>&1; echo "rc $?" >> gpurun_out/q_tests.log
python bench.py --no-cpu --no-e2e > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
