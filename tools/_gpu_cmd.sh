mkdir -p gpurun_out/s4
O=gpurun_out/s4
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python tools/lmp_step_bench.py > $O/ls0.txt 2>&1
