mkdir -p gpurun_out/it
O=gpurun_out/it
timeout 900 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -p no:cacheprovider -k "lmp or pcg or gemm" > $O/t.log 2>&1; echo rc=$? >> $O/t.log
python tools/lmp_step_bench.py > $O/ls0.txt 2>&1
SHAPE=262144,128,256 EDAK_LMP_NN=2 python tools/lmp_step_bench.py > $O/ls2.txt 2>&1
SHAPE=262144,128,256 EDAK_LMP_NN=3 python tools/lmp_step_bench.py > $O/ls3.txt 2>&1
SHAPE=262144,128,128 python tools/lmp_step_bench.py > $O/ls128.txt 2>&1
SHAPE=262144,128,128 EDAK_LMP_NN=2 python tools/lmp_step_bench.py > $O/ls128b.txt 2>&1
