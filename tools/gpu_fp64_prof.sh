# ncu --set full of one launch each of the fp64 stage kernels at C4 (error + TN GEMM)
ncu --set full --clock-control none --import-source on -k regex:k_err_persist -c 1 -o gpurun_out/err_full python tools/bench_configs.py C4 > gpurun_out/ncu_err.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dgemm_tn_async -s 1 -c 1 -o gpurun_out/tn_full python tools/bench_configs.py C4 > gpurun_out/ncu_tn.log 2>&1
