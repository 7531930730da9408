mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests -m gpu -q -x -k "gat_fused or gat_attention or gat_core or trace" > gpurun_out/g9_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/g9_tests.log
timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_rmat_v4.json 2>gpurun_out/r02/bench_gat_rmat_v4.err; echo gat=$?
HG_FUSED_GAT=0 timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_rmat_v4_unfused.json 2>/dev/null; echo gat=$?
for f in gat_rmat_v4 gat_rmat_v4_unfused; do python -c "
import json; d=json.loads(open('gpurun_out/r02/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step_eager'], d['e2e']['value'])"; done
