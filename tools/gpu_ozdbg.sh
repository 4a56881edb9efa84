mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_oz_tn$|k_oz_tn\(|k_oz_err" --csv --log-file gpurun_out/oz_dbg_0.csv python tools/oz_prof.py 524288 > gpurun_out/oz_dbg_0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider > gpurun_out/oz_tests.log 2>&1
echo "rc $?" >> gpurun_out/oz_tests.log
python tools/oz_prof.py > gpurun_out/oz_prof.log 2>&1
