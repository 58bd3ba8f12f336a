mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 600 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider -k "svd_jacobi or nystrom" > $O/jac.log 2>&1; echo rc=$? >> $O/jac.log
CFG=4 python tools/jacobi_t_probe.py > $O/jt4.txt 2>&1
CFG=5 python tools/jacobi_t_probe.py > $O/jt5.txt 2>&1
