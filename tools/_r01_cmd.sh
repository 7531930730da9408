python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gat.json 2>gpurun_out/bench_gat.err
python bench.py --workload gat-pubmed --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gatp.json 2>gpurun_out/bench_gatp.err
