mkdir -p gpurun_out
python -m pytest tests/test_gpu_operator.py tests/test_gpu_bench_path.py -q -x -p no:cacheprovider -k "not member_traces" > gpurun_out/pytest_fam.log 2>&1; echo rc=$? >> gpurun_out/pytest_fam.log
python bench.py --no-cpu --no-e2e --per-config 5 --steps 5 > gpurun_out/bench_fam.json 2> gpurun_out/bench_fam.err
