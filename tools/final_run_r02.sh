# Round-2 consolidated run on one B200 (smoke, GPU tests, every bench line,
# the reference arm, launch lists, per-call traffic, one --set full SpMM capture).
# usage: gpurun -- bash tools/final_run_r02.sh   (outputs under gpurun_out/r02/)
R=${R:-5}
P=gpurun_out/r02/final$R; mkdir -p $P
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $P/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo tests=$?; tail -1 $P/pytest_gpu.log
( time timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench_gcn.json ) 2> $P/bench_gcn.err; echo gcn=$?
( time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/bench_reference_arm.json ) 2> $P/bench_ref.err; echo ref=$?
timeout 900 python bench.py --workload gin-products --steps 10 --warmup 3 --no-cpu-baseline > $P/bench_gin_products.json 2>/dev/null; echo gin=$?
timeout 900 python bench.py --workload gat-rmat --steps 5 --warmup 3 --no-cpu-baseline > $P/bench_gat_rmat.json 2>/dev/null; echo gat=$?
timeout 900 python bench.py --workload gat-pubmed --steps 20 --warmup 3 --no-cpu-baseline > $P/bench_gat_pubmed.json 2>/dev/null; echo pub=$?
Q=gpurun_out/r02/prof$R; mkdir -p $Q
for w in gcn-reddit gin-products gat-rmat; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $Q/launch_$w.csv python tools/ncu_target.py --workload $w --epochs 3 > /dev/null 2>&1; echo launch_$w=$?
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmm_fast --csv --log-file $Q/traffic_$w.csv python tools/ncu_target.py --workload $w --epochs 2 > /dev/null 2>&1; echo traffic_$w=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $Q/launch_bench_gcn.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-small --no-cpu-baseline > /dev/null 2>&1; echo lb=$?
T=/tmp/hgprof$R; mkdir -p $T
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_fast -s 4 -c 1 -f -o $T/full_spmm_c3 python tools/ncu_target.py --workload gcn-reddit --epochs 3 > /dev/null 2>&1; echo fs=$?
python tools/ncu_summary.py $T/full_spmm_c3.ncu-rep full_spmm_c3_reordered > $Q/full_spmm_c3.md 2>&1
ncu -i $T/full_spmm_c3.ncu-rep --page raw --csv > $Q/full_spmm_c3.raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -c 1 -f -o $T/full_gemm_dots_c5 python tools/ncu_target.py --workload gat-rmat --epochs 1 > /dev/null 2>&1; echo fg=$?
python tools/ncu_summary.py $T/full_gemm_dots_c5.ncu-rep full_gemm_dots_c5 > $Q/full_gemm_dots_c5.md 2>&1
ncu -i $T/full_gemm_dots_c5.ncu-rep --page raw --csv > $Q/full_gemm_dots_c5.raw.csv 2>/dev/null
