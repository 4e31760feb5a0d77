# Round-2 measurement pass (the driver's own runs are authoritative; this is for profiles/)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_gputests.log 2>&1; echo "rc $?" >> gpurun_out/r2f_gputests.log
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1; echo "rc $?" >> gpurun_out/r2f_bench.log
BENCH_FORCE_DIST=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29561 RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 timeout 900 python bench.py --steps 5 --no-cpu --no-extras > gpurun_out/r2f_bench_dist1.log 2>&1; echo "rc $?" >> gpurun_out/r2f_bench_dist1.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2f_bench_reference.log 2>&1; echo "rc $?" >> gpurun_out/r2f_bench_reference.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2f_launches_run.log 2>&1; echo "rc $?" >> gpurun_out/r2f_launches_run.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 3 -c 1 -o gpurun_out/r2f_ncu_c4_main python tools/run_cfg.py C4 4 > gpurun_out/r2f_ncu_main.log 2>&1
timeout 120 python tools/dbg_stable.py C5 > gpurun_out/r2f_dbg_c5.log 2>&1
