mkdir -p gpurun_out
MPID_LIB=libmpid_base.so python tools/oz_prof.py > gpurun_out/oz_prof_base.log 2>&1
python tools/oz_prof.py > gpurun_out/oz_prof_new.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider > gpurun_out/oz_tests.log 2>&1; echo "rc $?" >> gpurun_out/oz_tests.log
