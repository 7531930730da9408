mkdir -p gpurun_out/r02
for w in gcn-reddit gin-products gat-rmat; do
  ep=2; [ $w = gat-rmat ] && ep=2
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launch_$w.csv python tools/ncu_target.py --workload $w --epochs 3 > /dev/null 2>&1; echo ncu_$w=$?
done
timeout 900 python bench.py --workload gin-products --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gin.json 2> gpurun_out/r02/bench_gin.err; echo gin=$?
timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_rmat.json 2> gpurun_out/r02/bench_gat_rmat.err; echo gat=$?
timeout 900 python bench.py --workload gat-pubmed --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02/bench_gat_pubmed.json 2> gpurun_out/r02/bench_gat_pubmed.err; echo pub=$?
