# Round-2 final-session measurement pass at HEAD: GPU suite, bench (both arms), phase stamps.
# Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_gputests.log 2>&1; echo "rc $?" >> gpurun_out/r2g_gputests.log
timeout 900 python bench.py > gpurun_out/r2g_bench.log 2>&1; echo "rc $?" >> gpurun_out/r2g_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2g_bench_reference.log 2>&1; echo "rc $?" >> gpurun_out/r2g_bench_reference.log
timeout 300 python tools/dbg_cluster.py C1 > gpurun_out/r2g_dbg_cluster_c1.log 2>&1
timeout 300 python tools/dbg_stable.py > gpurun_out/r2g_dbg_stable.log 2>&1
tail -3 gpurun_out/r2g_gputests.log
