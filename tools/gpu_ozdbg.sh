mkdir -p gpurun_out
for d in 0 1 2 3; do
  MPID_OZ_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_oz_tn$|k_oz_tn\(" --csv --log-file gpurun_out/oz_dbg_$d.csv python tools/oz_prof.py 524288 > gpurun_out/oz_dbg_$d.log 2>&1
done
