mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_configs.py tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
CFG=3 python tools/ab_knobs.py "" > $O/ab3.txt 2>&1
CFG=4 python tools/ab_knobs.py "" "EDAK_SWEEP_LEGACY=1" > $O/ab4.txt 2>&1
CFG=3 REPS=10 python tools/ab_pass.py "" > $O/abp3.txt 2>&1
for c in 1 2; do CFG=$c REPS=10 python tools/ab_pass.py "" > $O/abp$c.txt 2>&1; done
