# Round-2 closing check at HEAD: GPU suite, smoke, bench (both arms).  Run under gpurun.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2l_gputests.log 2>&1; echo "rc $?" >> gpurun_out/r2l_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; echo "rc $?" >> gpurun_out/r2l_smoke.log
timeout 900 python bench.py > gpurun_out/r2l_bench.log 2>&1; echo "rc $?" >> gpurun_out/r2l_bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2l_bench_reference.log 2>&1; echo "rc $?" >> gpurun_out/r2l_bench_reference.log
tail -3 gpurun_out/r2l_gputests.log; tail -2 gpurun_out/r2l_smoke.log
