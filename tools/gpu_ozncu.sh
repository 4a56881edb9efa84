mkdir -p gpurun_out
python tools/oz_prof.py > gpurun_out/oz_prof.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_oz_tn$|k_oz_tn\(|k_oz_err" -c 2 -f -o gpurun_out/oz_final_full python tools/oz_prof.py > gpurun_out/oz_ncu_full.log 2>&1
echo "rc $?" >> gpurun_out/oz_ncu_full.log
