python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "gat or attention or dist or acceptance" > gpurun_out/pytest_gat.log 2>&1; tail -1 gpurun_out/pytest_gat.log
python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gat.json 2>gpurun_out/bench_gat.err
timeout 1200 ncu --set full --clock-control none -k regex:"k_gat_(fwd|bwd)_all" -c 2 -o /tmp/gat python tools/ncu_target.py --workload gat-rmat --epochs 1 > /tmp/ncu_gat.log 2>&1
python tools/ncu_summary.py /tmp/gat.ncu-rep "fast GAT attention fwd / bwd after the one-chunk row path, RMAT-24 layer 1" > gpurun_out/ncu_gat2.md
