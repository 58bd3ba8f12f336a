mkdir -p gpurun_out/it
O=gpurun_out/it
python -m pytest tests/test_gpu_operator.py -m gpu -q -x -p no:cacheprovider -k "overlap" > $O/os.log 2>&1; echo rc=$? >> $O/os.log
CFG=4 REPS=5 python tools/ab_pass.py "" "EDAK_CIRC_OS16=0" "EDAK_CIRC_OS16_MINB10=4" "EDAK_CIRC_OS16_MINB10=8" > $O/ab4e.txt 2>&1
CFG=5 REPS=3 python tools/ab_pass.py "" "EDAK_CIRC_OS16_MINB=3" > $O/ab5e.txt 2>&1
CFG=4 MEMBERS=100 timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_circ_os' -s 2 -c 1 -o $O/os16_10 python tools/circ_ncu.py > $O/os16_10.log 2>&1
EDAK_CIRC_OS16=0 CFG=4 MEMBERS=100 timeout 600 ncu --set full --clock-control none -k regex:'k_circ_os' -s 2 -c 1 -o $O/os_old10 python tools/circ_ncu.py > $O/os_old10.log 2>&1
