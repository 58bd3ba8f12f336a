mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=4 REPS=5 python tools/ab_pass.py "" "EDAK_PCG_SPLIT=1" "EDAK_PCG_GRAPH=0" "EDAK_PCG_GRAPH=0+EDAK_PCG_SPLIT=1" > $O/ab_split4.txt 2>&1
CFG=5 REPS=3 python tools/ab_pass.py "" "EDAK_PCG_SPLIT=1" > $O/ab_split5.txt 2>&1
