python tools/bench_configs.py gram > gpurun_out/configs_gram.jsonl 2> gpurun_out/configs_gram.err
ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -c 1 -o gpurun_out/gram_full python tools/bench_configs.py C4 gram > gpurun_out/ncu_gram.log 2>&1
