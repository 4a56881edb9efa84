bash tools/gpu_all.sh
timeout 1200 python tools/bench_configs.py > gpurun_out/configs_v6.jsonl 2> gpurun_out/configs_v6.err
