mkdir -p gpurun_out
python -m pytest tests/test_gpu_operator.py tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/pytest_pdl.log 2>&1; echo rc=$? >> gpurun_out/pytest_pdl.log
python -m pytest tests/test_gpu_bench_path.py -q -x -p no:cacheprovider -k "shape or eager" >> gpurun_out/pytest_pdl.log 2>&1; echo rc=$? >> gpurun_out/pytest_pdl.log
CFG=4 python tools/ab_knobs.py "EDAK_PDL=0" "EDAK_PDL=1" > gpurun_out/ab_pdl.txt 2>&1
EDAK_PDL=0 python bench.py --no-cpu --no-e2e --per-config 5 --steps 5 > gpurun_out/bench_pdl0.json 2> gpurun_out/bench_pdl0.err
python bench.py --no-cpu --no-e2e --per-config 5 --steps 5 > gpurun_out/bench_pdl1.json 2> gpurun_out/bench_pdl1.err
