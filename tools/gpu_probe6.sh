# Latency kernels (warp-per-column TRSM, one-barrier Cholesky, fewer-barrier shared-memory QRCP):
# parity tests, C1 / C2 timings against the previous kernels (env A/B), the C4 bench, launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_smem.py tests/test_gpu_parity.py tests/test_gpu_fp64.py tests/test_gpu_ozaki.py tests/test_gpu_c_abi.py -q -p no:cacheprovider > gpurun_out/p6_tests.log 2>&1; echo "rc $?" >> gpurun_out/p6_tests.log
timeout 600 python tools/bench_configs.py C1 C2 > gpurun_out/c12_cfg_new.jsonl 2> gpurun_out/c12_cfg.err
MPID_TRSM_BLOCK=1 MPID_CHOL_3BAR=1 timeout 600 python tools/bench_configs.py C1 C2 > gpurun_out/c12_cfg_old.jsonl 2>> gpurun_out/c12_cfg.err
timeout 600 python bench.py > gpurun_out/bench_p6.json 2> gpurun_out/bench_p6.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c12_launches_new.csv python tools/bench_configs.py C1 C2 > gpurun_out/c12_launch_new.log 2>&1; echo "rc $?" >> gpurun_out/c12_launch_new.log
