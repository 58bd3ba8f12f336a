mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 600 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider -k "shifted_cholesky or nystrom or potrf" > $O/sc.log 2>&1; echo rc=$? >> $O/sc.log
