# int8 (Ozaki) fp64 engine: parity tests, a short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider > gpurun_out/oz_tests.log 2>&1
echo "rc $?" >> gpurun_out/oz_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/oz_bench.json 2> gpurun_out/oz_bench.err
echo "bench rc $?" >> gpurun_out/oz_bench.err
