mkdir -p gpurun_out
python tools/oz_prof.py 262144 > gpurun_out/oz_prof_small.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_oz_err" -c 1 -o gpurun_out/oz_err_full python tools/oz_prof.py 262144 > gpurun_out/oz_ncu_full.log 2>&1
echo "rc $?" >> gpurun_out/oz_ncu_full.log
