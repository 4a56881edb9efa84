# Round-2 measurement: bench line, launch list, full ncu capture of the dominant kernel.
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc $?" >> gpurun_out/bench_r02.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2500 --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
echo "ncu list rc $?" >> gpurun_out/ncu_l.log
ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 1 -c 1 -o gpurun_out/pass_tc_r02 \
    python tools/prof_tc2.py 16 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 15 -c 1 -o gpurun_out/pass_tc_store_r02 \
    python tools/prof_tc2.py 16 >> gpurun_out/ncu_full.log 2>&1
echo "ncu full rc $?" >> gpurun_out/ncu_full.log
