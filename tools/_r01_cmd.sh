python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gat.json 2>gpurun_out/bench_gat.err
python bench.py --workload gin-products --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gin.json 2>gpurun_out/bench_gin.err
python bench.py > gpurun_out/bench_gcn.json 2>gpurun_out/bench_gcn.err
