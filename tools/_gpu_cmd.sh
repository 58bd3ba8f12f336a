mkdir -p gpurun_out
python -m pytest tests/test_harness.py -q -x -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_h.log
