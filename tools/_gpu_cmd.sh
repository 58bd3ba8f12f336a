mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=4 python tools/ab_knobs.py "" "EDAK_SWEEP_LEGACY=1" > $O/ab_pro4.txt 2>&1
CFG=5 python tools/ab_knobs.py "" > $O/ab_pro5.txt 2>&1
CFG=4 REPS=5 python tools/ab_pass.py "" > $O/abp_pro4.txt 2>&1
CFG=5 REPS=3 python tools/ab_pass.py "" > $O/abp_pro5.txt 2>&1
