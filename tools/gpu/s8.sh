mkdir -p gpurun_out/s8
timeout 300 python tools/c1_stall.py > gpurun_out/s8/c1_stall.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plane2_kernel -s 2 -c 1 -o gpurun_out/s8/plane2 python tools/apply_time.py C4 15 plane_fuse=2 > gpurun_out/s8/ncu_plane2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xex_kernel -s 2 -c 1 -o gpurun_out/s8/xex python tools/apply_time.py C4 15 > gpurun_out/s8/ncu_xex.log 2>&1
