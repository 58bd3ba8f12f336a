mkdir -p gpurun_out
V="EDAK_SWEEP_LEGACY=1 EDAK_SWEEP_LEGACY=0 EDAK_AD_TDEPTH=1"
CFG=4 python tools/ab_knobs.py $V > gpurun_out/ab_tma4.txt 2>&1
CFG=5 python tools/ab_knobs.py $V > gpurun_out/ab_tma5.txt 2>&1
python -m pytest tests/test_gpu_operator.py -q -x -p no:cacheprovider > gpurun_out/pytest_op.log 2>&1; echo rc=$? >> gpurun_out/pytest_op.log
