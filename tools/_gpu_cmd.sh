mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=4 PHASE=pass python tools/kernel_profile.py > $O/kp4.txt 2>&1
CFG=4 REPS=5 python tools/ab_pass.py "" > $O/abp4.txt 2>&1
