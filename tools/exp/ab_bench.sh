#!/bin/bash
# A/B: the GCN C3 bench line under each library variant (tools/exp/variants/*).
# usage: tools/exp/ab_bench.sh [workload] [variant ...]
wl=${1:-gcn-reddit}; shift
for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="tools/exp/variants/$v/libhalfgnn.so"; fi
  HG_LIB=$lib timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --no-sweep --no-small \
    --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); r=d['roofline']; g=r.get('gather_ceiling') or {}
print(json.dumps({'variant':'$v','ms':d['value'],'eager':d['ms_per_step_eager'],
  'spmm_ms':g.get('spmm_ms_per_step'),'probe_ms':g.get('probe_ms_per_step'),'l2frac':(r.get('l2') or {}).get('frac')}))"
done
