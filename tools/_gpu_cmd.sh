mkdir -p gpurun_out
python -m pytest tests/test_gpu_operator.py -q -x -p no:cacheprovider > gpurun_out/pytest_op.log 2>&1; echo rc=$? >> gpurun_out/pytest_op.log
CFG=4 python tools/ab_knobs.py "EDAK_SWEEP_LEGACY=1" "EDAK_SWEEP_TMA_AD=0" "EDAK_AD_TDEPTH=1" "EDAK_AD_TDEPTH=2" > gpurun_out/ab_ad4.txt 2>&1
CFG=5 MEMBERS=128 python tools/ab_knobs.py "EDAK_SWEEP_LEGACY=1" "EDAK_SWEEP_TMA_AD=0" "EDAK_AD_TDEPTH=1" "EDAK_AD_TDEPTH=2" > gpurun_out/ab_ad5.txt 2>&1
