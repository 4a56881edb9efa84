# Warp-state sampling of the tcgen05 pass before (libmpid_base.so = a build of commit db951ab,
# copied beside libmpid.so by hand) and after the issue-loop fixes, and of the int8 fp64 kernels.
mkdir -p gpurun_out
MPID_LIB=libmpid_base.so ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 130 -c 1 -f -o gpurun_out/pass_src_base python tools/pass_tune.py 16 > gpurun_out/pass_src_base.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass_tc -s 130 -c 1 -f -o gpurun_out/pass_src_new python tools/pass_tune.py 16 > gpurun_out/pass_src_new.log 2>&1
bash tools/gpu_ozncu.sh
