mkdir -p gpurun_out
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_bench_path.py -q -x -p no:cacheprovider -k "multirank or shape or eager" > gpurun_out/pytest_mr.log 2>&1; echo rc=$? >> gpurun_out/pytest_mr.log
python -m pytest tests/test_gpu_solvers.py -q -x -p no:cacheprovider -k "pcg" > gpurun_out/pytest_pcg.log 2>&1; echo rc=$? >> gpurun_out/pytest_pcg.log
