mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=3 python tools/ab_knobs.py "" "EDAK_PERIODIC_FAMILY=4,256" "EDAK_PERIODIC_FAMILY=2,512" > $O/ab_pf3.txt 2>&1
CFG=3 REPS=10 python tools/ab_pass.py "" "EDAK_PERIODIC_FAMILY=4,256" "EDAK_PERIODIC_FAMILY=2,512" > $O/abp_pf3.txt 2>&1
