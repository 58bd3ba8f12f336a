mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
CFG=4 PHASE=pass python tools/kernel_profile.py > $O/kp4.txt 2>&1
CFG=4 REPS=5 python tools/ab_pass.py "" > $O/abp4.txt 2>&1
