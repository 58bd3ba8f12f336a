mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider > $O/t1.log 2>&1; echo rc=$? >> $O/t1.log
CFG=5 python tools/pass_breakdown.py > $O/brk5.txt 2>&1
CFG=4 python tools/pass_breakdown.py > $O/brk4.txt 2>&1
