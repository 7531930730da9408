mkdir -p gpurun_out/r02
timeout 1200 python tools/overlap_timeline.py > gpurun_out/r02/overlap_timeline_c5_p8.json 2> gpurun_out/r02/overlap_timeline.err; echo tl=$?
tail -3 gpurun_out/r02/overlap_timeline.err
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dist.py -m gpu -q -x -k "spmm_acc or column_blocked or partitioned" > gpurun_out/g15_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/g15_tests.log
