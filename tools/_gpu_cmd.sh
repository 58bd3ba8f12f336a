mkdir -p gpurun_out
python -m pytest tests/test_gpu_solvers.py tests/test_gpu_bench_path.py -q -x -p no:cacheprovider > gpurun_out/pytest_sol.log 2>&1; echo rc=$? >> gpurun_out/pytest_sol.log
python bench.py --no-cpu --per-config 5 --steps 5 > gpurun_out/bench_lg.json 2> gpurun_out/bench_lg.err
