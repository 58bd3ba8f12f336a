# Round-end evidence on one B200: per-config sweep ncu record (first: the
# bench reads it), GPU tests, bench (ours + reference arm), launch lists
# (cfg4 bench, cfg5 pass) and a full ncu capture of the top cfg4 kernels.
# Outputs under gpurun_out/r2f/.
mkdir -p gpurun_out/r2f
O=gpurun_out/r2f
M=dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
python tools/sweep_ncu.py 4 > $O/sw4.log 2>&1 && ncu --metrics $M --clock-control none -k regex:'k_ad|k_tl' -s 4 -c 4 --csv --log-file $O/sweep_ncu_cfg4.csv python tools/sweep_ncu.py 4 > $O/ncu4.log 2>&1
python tools/sweep_ncu.py 5 > $O/sw5.log 2>&1 && ncu --metrics $M --clock-control none -k regex:'k_ad|k_tl' -s 2 -c 2 --csv --log-file $O/sweep_ncu_cfg5.csv python tools/sweep_ncu.py 5 > $O/ncu5.log 2>&1
python tools/ncu_to_json.py cfg4=$O/sweep_ncu_cfg4.csv cfg5=$O/sweep_ncu_cfg5.csv > $O/ncu_to_json.log 2>&1
cp profiles/r2_sweep_ncu.json $O/r2_sweep_ncu.json
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --per-config "" > $O/ncu_launch4.log 2>&1
CFG=5 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches_cfg5.csv python tools/prof_pass.py > $O/ncu_launch5.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:'k_ad_tile|k_tl_tile|k_lmp_nn|k_lmp_tn|k_circ_os16|k_svd_bjacobi' -s 60 -c 8 -o $O/cfg4_top python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --per-config "" > $O/ncu_full.log 2>&1
echo done >> $O/ncu_full.log
