mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=5 REPS=3 python tools/ab_pass.py "" "EDAK_LMP_TN=0" "EDAK_LMP_GEMM=0" > $O/ab5c.txt 2>&1
CFG=5 PHASE=pass python tools/kernel_profile.py > $O/kp5_pass.txt 2>&1
