mkdir -p gpurun_out
export HG_KERNEL_LIST=gpurun_out/g2_kernels.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge_cases.py tests/test_gpu_models.py -m gpu -q -rf -x -k "gemm or linear or dense_math or trace or parity or graph_step or smoke" > gpurun_out/g2_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/g2_tests.log
timeout 600 python bench.py --no-sweep --no-small --no-cpu-baseline > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; echo bench_rc=$?
head -c 600 gpurun_out/g2_bench.json
