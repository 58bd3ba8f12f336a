mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider -k "cholqr_lazy or blocked_gram or nystrom" > $O/newtests.log 2>&1; echo rc=$? >> $O/newtests.log
