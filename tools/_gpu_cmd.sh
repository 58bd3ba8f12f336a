mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_tl_tile' -s 2 -c 2 -o $O/tl_full python tools/sweep_ncu.py 4 > $O/tl_full.log 2>&1
