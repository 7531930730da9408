mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g8_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/g8_tests.log
python tools/gemm_bench.py > gpurun_out/r02/gemm_bench_v4.jsonl 2>&1
timeout 600 python bench.py --no-sweep --no-small --no-cpu-baseline > gpurun_out/r02/bench_gcn_v2.json 2>/dev/null; echo gcn=$?
timeout 600 python bench.py --workload gin-products --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gin_v2.json 2>/dev/null; echo gin=$?
timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_rmat_v2.json 2>/dev/null; echo gat=$?
for f in gcn_v2 gin_v2 gat_rmat_v2; do python -c "
import json; d=json.loads(open('gpurun_out/r02/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'])"; done
