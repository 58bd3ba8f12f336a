mkdir -p gpurun_out
CFG=4 python tools/circ_ncu.py > gpurun_out/c4.log 2>&1 && CFG=4 ncu --set full --import-source on --clock-control none -k regex:k_circ_os -s 2 -c 1 -o gpurun_out/r2_circ_os4 python tools/circ_ncu.py > gpurun_out/ncu_c4.log 2>&1
CFG=5 MEMBERS=128 python tools/circ_ncu.py > gpurun_out/c5.log 2>&1 && CFG=5 MEMBERS=128 ncu --set full --import-source on --clock-control none -k regex:k_circ_os -s 2 -c 1 -o gpurun_out/r2_circ_os5 python tools/circ_ncu.py > gpurun_out/ncu_c5.log 2>&1
echo rc=$?
