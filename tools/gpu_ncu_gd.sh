cd /root/repo; mkdir -p gpurun_out
for L in 8 3 1; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gs_pieces -c 1 -o gpurun_out/prof_gd_L$L -f python tools/profile_kernel.py 2 $L > gpurun_out/ncu_gd_L$L.log 2>&1
done
