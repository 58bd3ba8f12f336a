mkdir -p gpurun_out/it
O=gpurun_out/it
CFG=5 python tools/ab_knobs.py "" "EDAK_CIRC_OS16P=3" "EDAK_CIRC_OS16P=2" > $O/ab_osp5.txt 2>&1
CFG=4 python tools/ab_knobs.py "" "EDAK_CIRC_OS16P=6" "EDAK_CIRC_OS16P=4" > $O/ab_osp4.txt 2>&1
CFG=5 REPS=3 python tools/ab_pass.py "" "EDAK_CIRC_OS16P=3" > $O/abp_osp5.txt 2>&1
CFG=4 REPS=5 python tools/ab_pass.py "" "EDAK_CIRC_OS16P=6" > $O/abp_osp4.txt 2>&1
