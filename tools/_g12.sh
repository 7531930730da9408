mkdir -p gpurun_out/r02
timeout 1200 python -m pytest tests -m gpu -q -x -k "spmm or gat or trace or parity or smoke" > gpurun_out/g12_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/g12_tests.log
for v in roll noroll; do
  if [ $v = noroll ]; then export HG_LIB=tools/exp/variants/norolling/libhalfgnn.so; fi
  timeout 600 python bench.py --no-small --no-cpu-baseline > gpurun_out/r02/bench_gcn_$v.json 2>/dev/null
  timeout 600 python bench.py --workload gin-products --steps 10 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/r02/bench_gin_$v.json 2>/dev/null
  timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_$v.json 2>/dev/null
  HG_FUSED_GAT=0 timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gatunf_$v.json 2>/dev/null
  for f in gcn_$v gin_$v gat_$v gatunf_$v; do python -c "
import json; d=json.loads(open('gpurun_out/r02/bench_$f.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', d['value'], d['ms_per_step_eager'], d['e2e']['value'], r.get('gather_ceiling') and r['gather_ceiling']['frac'], {k:v['ms'] for k,v in d.get('spmm_sweep_reddit',{}).items()})"; done
done
