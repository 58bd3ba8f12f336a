mkdir -p gpurun_out/it
O=gpurun_out/it
python tools/sweep_ncu.py 5 > $O/sw5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_tl_tile|k_ad_tile' -s 2 -c 2 -o $O/sw5_full python tools/sweep_ncu.py 5 > $O/sw5_full.log 2>&1
