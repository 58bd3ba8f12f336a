mkdir -p gpurun_out
for sh in 262144,128,86 262144,128,128 16384,128,100; do for f in 0 1; do SHAPE=$sh FLAGS=$f PROFILE=$f python tools/lmp_gemm_bench.py 2>/dev/null | grep -v Warn; done; done > gpurun_out/lmp_gemm_c5.txt 2>&1
