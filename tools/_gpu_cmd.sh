mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "integrate or refresh or stream or model or ensemble or config" > $O/int.log 2>&1; echo rc=$? >> $O/int.log
python bench.py --steps 5 --warmup 3 --no-cpu --per-config "" > $O/b.json 2> $O/b.err
