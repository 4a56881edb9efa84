bash tools/gpu_all.sh
ncu --set full --clock-control none --import-source on -k regex:k_err_ws -c 1 -o gpurun_out/errws_full python tools/bench_configs.py C4 gram > gpurun_out/ncu_errws.log 2>&1
