mkdir -p gpurun_out/r02
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_edge_cases.py tests/test_gpu_models.py -m gpu -q -x -k "gemm or linear or dense_math or trace or parity or graph_step" > gpurun_out/g5_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/g5_tests.log
python tools/gemm_bench.py > gpurun_out/r02/gemm_bench_v2.jsonl 2>&1; echo gb=$?
cat gpurun_out/r02/gemm_bench_v2.jsonl
