mkdir -p gpurun_out
timeout 2700 python tools/bench_configs.py > gpurun_out/configs_r02.jsonl 2> gpurun_out/configs_r02.err
echo "rc $?" >> gpurun_out/configs_r02.err
python tools/oz_prof.py 262144 > gpurun_out/oz_prof_small.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_oz_err" -c 1 -o gpurun_out/oz_err_full python tools/oz_prof.py 262144 > gpurun_out/oz_ncu_full.log 2>&1
