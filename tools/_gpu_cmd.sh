mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=5 REPS=3 python tools/ab_pass.py "" "EDAK_PCG_GRAPH=1" "EDAK_PCG_GROUPS=2+EDAK_PCG_GRAPH=1" > $O/ab_g5.txt 2>&1
