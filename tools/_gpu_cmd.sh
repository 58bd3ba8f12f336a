mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 600 python -m pytest tests/test_gpu_operator.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider > $O/op.log 2>&1; echo rc=$? >> $O/op.log
CFG=4 python tools/ab_knobs.py "" "EDAK_SWEEP_LEGACY=1" > $O/ab_v4.txt 2>&1
CFG=5 python tools/ab_knobs.py "" > $O/ab_v5.txt 2>&1
CFG=4 REPS=5 python tools/ab_pass.py "" > $O/abp_v4.txt 2>&1
CFG=5 REPS=3 python tools/ab_pass.py "" > $O/abp_v5.txt 2>&1
