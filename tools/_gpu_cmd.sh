mkdir -p gpurun_out
CFG=4 MEMBERS=100 python tools/ab_knobs.py "EDAK_CIRC_OS_MINB=6" "EDAK_CIRC_OS_PREH=1" "EDAK_CIRC_OS_PREH=1+EDAK_CIRC_OS_MINB=4" "EDAK_CIRC_OS_MINB=8" > gpurun_out/ab_os4.txt 2>&1
CFG=5 MEMBERS=128 python tools/ab_knobs.py "EDAK_CIRC_OS2_MINB=1" "EDAK_CIRC_OS2_MINB=2" "EDAK_CIRC_OS2_MINB=3" "EDAK_CIRC_OS2_MINB=4" "EDAK_CIRC_OS_PREH=1" > gpurun_out/ab_os5.txt 2>&1
