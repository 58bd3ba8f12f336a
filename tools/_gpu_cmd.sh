mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_edge_cases.py tests/test_harness.py -m gpu -q -x -p no:cacheprovider > $O/solv.log 2>&1; echo rc=$? >> $O/solv.log
CFG=4 python tools/pass_breakdown.py > $O/brk4.txt 2>&1
CFG=5 python tools/pass_breakdown.py > $O/brk5.txt 2>&1
CFG=4 PHASE=nystrom python tools/kernel_profile.py > $O/kp4_nys.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider > $O/bp.log 2>&1; echo rc=$? >> $O/bp.log
