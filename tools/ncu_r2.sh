set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -x -q -k "stable or guess or search or c5 or normal or paper_layout" > gpurun_out/r2_t10.log 2>&1; echo "rc $?" >> gpurun_out/r2_t10.log
timeout 120 python tools/dbg_stable.py C5 > gpurun_out/r2_dbg_c5b.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lm_cluster_kernel -s 2 -c 1 -o gpurun_out/r2_ncu_c1_cluster python tools/run_cfg.py C1 3 > gpurun_out/r2_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 3 -c 1 -o gpurun_out/r2_ncu_c4_main python tools/run_cfg.py C4 4 > gpurun_out/r2_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lm_full_kernel -s 3 -c 1 -o gpurun_out/r2_ncu_c4_stream python tools/run_cfg.py C4 4 schedule=stream > gpurun_out/r2_ncu3.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:st_fixpoint -s 2 -c 1 -o gpurun_out/r2_ncu_c5_stable python tools/run_cfg.py C5 3 stable=1 > gpurun_out/r2_ncu4.log 2>&1
