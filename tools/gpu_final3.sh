# Round-2 final validation (after the pass's issue-loop fixes): GPU tests, smoke, bench line,
# reference arm, launch list, ncu --set full of the tcgen05 pass (a non-store and a store launch).
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "rc $?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc $?" >> gpurun_out/bench_r02.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_l.log 2>&1
echo "ncu list rc $?" >> gpurun_out/ncu_l.log
ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 125 -c 6 -f -o gpurun_out/pass_tc_v8 python tools/pass_tune.py 16 > gpurun_out/pass_v8_ncu.log 2>&1
echo "ncu full rc $?" >> gpurun_out/pass_v8_ncu.log
