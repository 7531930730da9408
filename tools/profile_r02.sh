# round-2 profiling pass (one B200): launch lists, per-call DRAM traffic, --set full captures
# usage: gpurun -- bash tools/profile_r02.sh   (outputs in gpurun_out/r02/prof, copied to profiles/r02)
P=gpurun_out/r02/prof; mkdir -p $P; T=/tmp/hgprof; mkdir -p $T
for w in gcn-reddit gin-products gat-rmat; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launch_$w.csv python tools/ncu_target.py --workload $w --epochs 3 > /dev/null 2>&1; echo launch_$w=$?
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmm_fast --csv --log-file $P/traffic_$w.csv python tools/ncu_target.py --workload $w --epochs 2 > /dev/null 2>&1; echo traffic_$w=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $P/launch_bench_gcn.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-small --no-cpu-baseline > /dev/null 2>&1; echo lb=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fast -s 8 -c 1 -o $T/full_spmm_c3 python tools/ncu_target.py --workload gcn-reddit --epochs 3 > /dev/null 2>&1; echo fs=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm" -s 4 -c 4 -o $T/full_gemm_c3 python tools/ncu_target.py --workload gcn-reddit --epochs 3 > /dev/null 2>&1; echo fg=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm" -s 0 -c 2 -o $T/full_gemm_c5 python tools/gemm_bench.py --ncu --shapes 5 > /dev/null 2>&1; echo fg5=$?
for r in full_spmm_c3 full_gemm_c3 full_gemm_c5; do
  python tools/ncu_summary.py $T/$r.ncu-rep "$r" > $P/$r.md 2>&1
  ncu -i $T/$r.ncu-rep --page raw --csv > $P/$r.raw.csv 2>/dev/null
done
timeout 600 python tools/gemm_bench.py > $P/gemm_bench.jsonl 2>&1; echo gb=$?
ls -la $P
