mkdir -p gpurun_out
python tools/pass_tune.py 16 > gpurun_out/pass_tune.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 130 -c 1 -f -o gpurun_out/pass_tc_src python tools/pass_tune.py 16 > gpurun_out/pass_src_ncu.log 2>&1
echo "rc $?" >> gpurun_out/pass_src_ncu.log
