mkdir -p gpurun_out/r2full
O=gpurun_out/r2full
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:'k_ad_tile|k_tl_tile|k_lmp_nn|k_lmp_tn|k_circ_os' -s 60 -c 8 -o $O/cfg4_top python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --per-config "" > $O/ncu.log 2>&1
echo rc=$? >> $O/ncu.log
