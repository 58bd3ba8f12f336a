mkdir -p gpurun_out
python -m pytest tests/test_gpu_solvers.py -q -x -p no:cacheprovider -k "chol or nystrom or svd" > gpurun_out/pytest_ch.log 2>&1; echo rc=$? >> gpurun_out/pytest_ch.log
CFG=5 REPS=1 PHASE=nystrom python tools/kernel_profile.py > gpurun_out/kprof5n.txt 2>&1
python -m pytest tests/test_gpu_bench_path.py -q -x -p no:cacheprovider -k "cfg5" > gpurun_out/pytest_c5.log 2>&1; echo rc=$? >> gpurun_out/pytest_c5.log
