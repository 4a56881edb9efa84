mkdir -p gpurun_out
python tools/c2_prof.py > gpurun_out/c2_prof.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python tools/c2_prof.py > gpurun_out/c2_ncu.log 2>&1
