mkdir -p gpurun_out/r02
timeout 900 python bench.py --workload gat-pubmed --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_pubmed_v4.json 2>/dev/null; echo pub=$?
HG_FUSED_GAT=0 timeout 900 python bench.py --workload gat-pubmed --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_pubmed_v4_unfused.json 2>/dev/null; echo pub=$?
for f in gat_pubmed_v4 gat_pubmed_v4_unfused; do python -c "
import json; d=json.loads(open('gpurun_out/r02/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step_eager'], d['e2e']['value'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fast -s 0 -c 1 -o gpurun_out/r02/ncu_att_fused python tools/ncu_target.py --workload gat-rmat --epochs 1 > /dev/null 2>&1; echo ncu=$?
HG_FUSED_GAT=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fast -s 0 -c 1 -o gpurun_out/r02/ncu_att_unfused python tools/ncu_target.py --workload gat-rmat --epochs 1 > /dev/null 2>&1; echo ncu=$?
