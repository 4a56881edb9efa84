# Full round-end validation: GPU tests, smoke, bench (+ reference arm, launch list), every
# config through tools/bench_configs.py, and an ncu --set full capture of the W GEMM.
bash tools/gpu_all.sh
timeout 1200 python tools/bench_configs.py > gpurun_out/configs_v9.jsonl 2> gpurun_out/configs_v9.err
ncu --set full --clock-control none --import-source on -k regex:k_dgemm_tn_pipe8 -s 1 -c 1 -o gpurun_out/tnpipe8_full_v18 python tools/bench_configs.py C4 gram > gpurun_out/ncu_tnpipe.log 2>&1
