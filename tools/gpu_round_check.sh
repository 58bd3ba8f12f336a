mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_r2b.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2b.log
python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r2b.json 2> gpurun_out/bench_ref_r2b.err
M=dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
python tools/sweep_ncu.py 4 > gpurun_out/sw4.log 2>&1 && python tools/sweep_ncu.py 5 > gpurun_out/sw5.log 2>&1 && ncu --metrics $M --clock-control none -k regex:'k_ad|k_tl' -s 4 -c 4 --csv --log-file gpurun_out/sweep_ncu_cfg4.csv python tools/sweep_ncu.py 4 > gpurun_out/ncu4.log 2>&1 && ncu --metrics $M --clock-control none -k regex:'k_ad|k_tl' -s 2 -c 2 --csv --log-file gpurun_out/sweep_ncu_cfg5.csv python tools/sweep_ncu.py 5 > gpurun_out/ncu5.log 2>&1
echo ncu_rc=$?
