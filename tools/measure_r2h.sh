# Round-2 final measurement pass with the compact stable kernel: GPU suite, bench (both arms).
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_gputests.log 2>&1; echo "rc $?" >> gpurun_out/r2h_gputests.log
timeout 900 python bench.py > gpurun_out/r2h_bench.log 2>&1; echo "rc $?" >> gpurun_out/r2h_bench.log
tail -3 gpurun_out/r2h_gputests.log; tail -c 600 gpurun_out/r2h_bench.log
