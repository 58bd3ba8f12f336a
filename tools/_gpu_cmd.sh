mkdir -p gpurun_out
python -m pytest tests/test_gpu_solvers.py -q -x -p no:cacheprovider -k "lanczos" > gpurun_out/pytest_lz.log 2>&1; echo rc=$? >> gpurun_out/pytest_lz.log
python -m pytest tests/test_harness.py -q -x -p no:cacheprovider -k "eig" > gpurun_out/pytest_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_h.log
