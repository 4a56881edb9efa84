mkdir -p gpurun_out
rm -f gpurun_out/c2_sweep.txt
for c in 0 96 64 32 16; do
  echo "cap $c" >> gpurun_out/c2_sweep.txt
  MPID_PASS_MAXCTAS=$c timeout 300 python tools/bench_configs.py C2 >> gpurun_out/c2_sweep.txt 2>/dev/null
done
