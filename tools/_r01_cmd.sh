python -m pytest tests/test_gpu_kernels.py -q -x -k "pack or schedule or spmm" > gpurun_out/t_pack.log 2>&1; tail -1 gpurun_out/t_pack.log
python bench.py > gpurun_out/bench_gcn.json 2>gpurun_out/bench_gcn.err
python bench.py --workload gat-pubmed --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gatp.json 2>gpurun_out/bench_gatp.err
python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gat.json 2>gpurun_out/bench_gat.err
