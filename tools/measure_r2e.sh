# Round-2 re-entry measurement pass for profiles/ (current kernels): launch list of the bench,
# ncu captures of the main line, the C5 stable call and the C3 armed fixpoint, reference arm.
# Run under gpurun from the repo root.
set -x
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2e_bench_reference.log 2>&1; echo "rc $?" >> gpurun_out/r2e_bench_reference.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2e_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2e_launches_run.log 2>&1; echo "rc $?" >> gpurun_out/r2e_launches_run.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 3 -c 1 -o gpurun_out/r2e_ncu_c4_main python tools/run_cfg.py C4 4 > gpurun_out/r2e_ncu_main.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:st_fixpoint -s 2 -c 1 -o gpurun_out/r2e_ncu_c5_stable python tools/run_cfg.py C5 3 stable=1 > gpurun_out/r2e_ncu_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 2 -c 1 -o gpurun_out/r2e_ncu_c3_armed python tools/run_cfg.py C3 3 > gpurun_out/r2e_ncu_c3.log 2>&1
ls -la gpurun_out/
