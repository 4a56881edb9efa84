mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc $?" >> gpurun_out/bench_r02.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_l.log 2>&1
echo "ncu list rc $?" >> gpurun_out/ncu_l.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c_abi.py tests/test_gpu_shards.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_sub.log 2>&1; echo "rc $?" >> gpurun_out/gpu_tests_sub.log
