# compact stable kernels: parity on both paths, then the C5 timing A/B and phase stamps
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -x -q -k "stable or guess or paper_layout or search or cluster_launches or random_normal" > gpurun_out/st_compact_tests.log 2>&1; echo "rc $?" >> gpurun_out/st_compact_tests.log
tail -5 gpurun_out/st_compact_tests.log
timeout 300 python tools/ab_compact.py > gpurun_out/st_compact_ab.log 2>&1; tail -20 gpurun_out/st_compact_ab.log
timeout 300 python tools/dbg_compact.py > gpurun_out/st_compact_dbg.log 2>&1; tail -4 gpurun_out/st_compact_dbg.log
timeout 300 python tools/ab_search.py > gpurun_out/st_search_ab.log 2>&1; tail -4 gpurun_out/st_search_ab.log
