# Round-2 (armed LEAD passes) measurement pass for profiles/: bench, launch list, ncu
# captures of the main line and of the STREAM schedule.  Run under gpurun from the repo root.
set -x
timeout 900 python bench.py > gpurun_out/r2b_bench.log 2>&1; echo "rc $?" >> gpurun_out/r2b_bench.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2b_launches_run.log 2>&1; echo "rc $?" >> gpurun_out/r2b_launches_run.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 3 -c 1 -o gpurun_out/r2b_ncu_c4_main python tools/run_cfg.py C4 4 > gpurun_out/r2b_ncu_main.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 3 -c 1 -o gpurun_out/r2b_ncu_c4_stream python tools/run_cfg.py C4 4 schedule=stream > gpurun_out/r2b_ncu_stream.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 2 -c 1 -o gpurun_out/r2b_ncu_c3_armed python tools/run_cfg.py C3 3 > gpurun_out/r2b_ncu_c3.log 2>&1
