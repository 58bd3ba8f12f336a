mkdir -p gpurun_out
python -m pytest tests/test_gpu_operator.py -q -x -p no:cacheprovider > gpurun_out/pytest_op.log 2>&1; echo rc=$? >> gpurun_out/pytest_op.log
CFG=4 MEMBERS=100 python tools/ab_knobs.py "EDAK_CIRC_WF=0" "EDAK_CIRC_WF_MINB=2" "EDAK_CIRC_WF_MINB=3" > gpurun_out/ab_wf4.txt 2>&1
CFG=5 MEMBERS=128 python tools/ab_knobs.py "EDAK_CIRC_WF=0" "EDAK_CIRC_WF_MINB=2" "EDAK_CIRC_WF_MINB=3" > gpurun_out/ab_wf5.txt 2>&1
