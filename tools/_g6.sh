mkdir -p gpurun_out/r02
python tools/gemm_bench.py --shapes 2,3,5 > gpurun_out/r02/gemm_bench_v3.jsonl 2>&1; cat gpurun_out/r02/gemm_bench_v3.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_wgrad -c 2 -o gpurun_out/r02/ncu_wgrad_v2 python tools/gemm_bench.py --ncu --shapes 3 > /dev/null 2>&1; echo ncu=$?
