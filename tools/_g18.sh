mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g18_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/g18_tests.log
for v in 1 0; do
HG_FUSED_FOLLOWUP=$v timeout 600 python bench.py --no-small --no-cpu-baseline --no-sweep > gpurun_out/r02/bench_gcn_ff$v.json 2>/dev/null
HG_FUSED_FOLLOWUP=$v timeout 600 python bench.py --workload gin-products --steps 10 --no-cpu-baseline --no-sweep > gpurun_out/r02/bench_gin_ff$v.json 2>/dev/null
HG_FUSED_FOLLOWUP=$v timeout 900 python bench.py --workload gat-rmat --steps 5 --no-cpu-baseline --no-sweep > gpurun_out/r02/bench_gat_ff$v.json 2>/dev/null
for f in gcn_ff$v gin_ff$v gat_ff$v; do python -c "
import json; d=json.loads(open('gpurun_out/r02/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step_eager'], d['e2e']['value'])"; done
done
