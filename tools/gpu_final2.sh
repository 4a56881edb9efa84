mkdir -p gpurun_out
python tools/c5shard_pass.py 64 > gpurun_out/c5pass.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_pass_tc" -s 40 -c 2 -o gpurun_out/c5_pass_full python tools/c5shard_pass.py 64 > gpurun_out/c5pass_ncu.log 2>&1
echo "rc $?" >> gpurun_out/c5pass_ncu.log
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc $?" >> gpurun_out/bench_r02.err
