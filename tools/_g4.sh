mkdir -p gpurun_out/r02
python tools/gemm_bench.py > gpurun_out/r02/gemm_bench_v1.jsonl 2>&1; echo gb=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -c 4 -o gpurun_out/r02/ncu_gemm_v1 python tools/gemm_bench.py --ncu --shapes 5 > gpurun_out/r02/ncu_gemm_v1.log 2>&1; echo ncu=$?
timeout 600 python tools/exp/run_gather_tma.py > gpurun_out/r02/gather_tma.json 2>&1; echo tma=$?
