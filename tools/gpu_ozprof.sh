mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -p no:cacheprovider > gpurun_out/oz_tests.log 2>&1
echo "rc $?" >> gpurun_out/oz_tests.log
python tools/oz_prof.py > gpurun_out/oz_prof.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_oz|k_err|k_dgemm|k_gather|k_trsm|k_chol|k_sum|k_assemble|k_eye|k_R_to|k_pack|k_diag" --csv --log-file gpurun_out/oz_launches.csv python tools/oz_prof.py > gpurun_out/oz_ncu.log 2>&1
echo "rc $?" >> gpurun_out/oz_ncu.log
