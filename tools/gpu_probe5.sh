# Round-2 probes: the one-launch C1 coefficient kernel (tests + A/B timing), the C4 pass's time
# vs SM clock / power, an ncu source-level capture of the one-launch shared-memory QRCP on C1,
# and the C1 / C2 launch lists.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coef_small.py tests/test_gpu_parity.py tests/test_gpu_smem.py -q -x -p no:cacheprovider > gpurun_out/p5_tests.log 2>&1; echo "rc $?" >> gpurun_out/p5_tests.log
timeout 300 python tools/bench_configs.py C1 > gpurun_out/c1_cfg.jsonl 2> gpurun_out/c1_cfg.err
MPID_COEF_SMALL=0 timeout 300 python tools/bench_configs.py C1 > gpurun_out/c1_cfg_graph.jsonl 2>> gpurun_out/c1_cfg.err
timeout 600 python tools/pass_power.py 8 > gpurun_out/pass_power.log 2>&1; echo "rc $?" >> gpurun_out/pass_power.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qrcp_smem -s 2 -c 1 -o gpurun_out/c1_smem_full python tools/bench_configs.py C1 > gpurun_out/c1_ncu.log 2>&1; echo "rc $?" >> gpurun_out/c1_ncu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c12_launches.csv python tools/bench_configs.py C1 C2 > gpurun_out/c12_launch.log 2>&1; echo "rc $?" >> gpurun_out/c12_launch.log
