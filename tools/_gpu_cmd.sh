mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_configs.py tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider > $O/op.log 2>&1; echo rc=$? >> $O/op.log
CFG=4 python tools/ab_knobs.py "" > $O/ab_s4.txt 2>&1
CFG=5 python tools/ab_knobs.py "" > $O/ab_s5.txt 2>&1
CFG=4 REPS=5 python tools/ab_pass.py "" > $O/abp_s4.txt 2>&1
CFG=5 REPS=3 python tools/ab_pass.py "" > $O/abp_s5.txt 2>&1
