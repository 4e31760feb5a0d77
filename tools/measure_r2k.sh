# Final measurement pass of round 2 (compact stable kernels, small-program kernel): GPU suite,
# bench (both arms), launch list, ncu captures of the new kernels.  Run under gpurun.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2k_gputests.log 2>&1; echo "rc $?" >> gpurun_out/r2k_gputests.log
timeout 900 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "rc $?" >> gpurun_out/r2k_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2k_bench_reference.log 2>&1; echo "rc $?" >> gpurun_out/r2k_bench_reference.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2k_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2k_smoke.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2k_launches_run.log 2>&1; echo "rc $?" >> gpurun_out/r2k_launches_run.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:st_compact_kernel -s 2 -c 1 -o gpurun_out/r2k_ncu_c5_compact python tools/run_cfg.py C5 3 stable=1 > gpurun_out/r2k_ncu_c5.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lm_small_kernel -s 2 -c 1 -o gpurun_out/r2k_ncu_c1_small python tools/run_cfg.py C1 4 > gpurun_out/r2k_ncu_c1.log 2>&1
timeout 300 python tools/ab_small.py > gpurun_out/r2k_ab_small.log 2>&1
timeout 300 python tools/ab_compact.py > gpurun_out/r2k_ab_compact.log 2>&1
timeout 300 python tools/ab_search.py > gpurun_out/r2k_ab_search.log 2>&1
ls -la gpurun_out/ | grep r2k
tail -3 gpurun_out/r2k_gputests.log
