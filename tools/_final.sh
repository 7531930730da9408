P=gpurun_out/r02/final; mkdir -p $P
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $P/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo tests=$?; tail -1 $P/pytest_gpu.log
( time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench_gcn.json ) 2> $P/bench_gcn.err; echo gcn=$?
( time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/bench_reference_arm.json ) 2> $P/bench_ref.err; echo ref=$?
timeout 900 python bench.py --workload gin-products --steps 10 --warmup 3 --no-cpu-baseline > $P/bench_gin_products.json 2>/dev/null; echo gin=$?
timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > $P/bench_gat_rmat.json 2>/dev/null; echo gat=$?
timeout 900 python bench.py --workload gat-pubmed --steps 20 --warmup 3 --no-cpu-baseline > $P/bench_gat_pubmed.json 2>/dev/null; echo pub=$?
tail -3 $P/bench_ref.err $P/bench_gcn.err
