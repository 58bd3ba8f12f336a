mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=4 python tools/ab_knobs.py "EDAK_X2=0" "EDAK_X2=2" "EDAK_X2=3" > $O/ab_x2_4.txt 2>&1
CFG=5 python tools/ab_knobs.py "EDAK_X2=0" "EDAK_X2=2" > $O/ab_x2_5.txt 2>&1
