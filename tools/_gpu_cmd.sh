mkdir -p gpurun_out/it
O=gpurun_out/it
python tools/lmp_step_bench.py > $O/lmpstep.txt 2>&1
