# Round-2 closing check at HEAD (after the on-demand T buffers and the per-SM CTA count of the compact kernels): GPU suite, smoke, bench (both arms).  Run under gpurun.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_gputests.log 2>&1; echo "rc $?" >> gpurun_out/r2n_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2n_smoke.log
timeout 900 python bench.py > gpurun_out/r2n_bench.log 2>&1; echo "rc $?" >> gpurun_out/r2n_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2n_bench_reference.log 2>&1; echo "rc $?" >> gpurun_out/r2n_bench_reference.log
tail -3 gpurun_out/r2n_gputests.log; tail -2 gpurun_out/r2n_smoke.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2n_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2n_launches_run.log 2>&1; echo "rc $?" >> gpurun_out/r2n_launches_run.log
