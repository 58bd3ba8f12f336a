mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 600 python -m pytest tests/test_gpu_operator.py -m gpu -q -x -p no:cacheprovider -k "dropins" > $O/dropins.log 2>&1; echo rc=$? >> $O/dropins.log
