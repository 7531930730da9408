mkdir -p gpurun_out/r02
for c in 1 2 3; do for bk in 64 128; do
 echo "ctas=$c bk=$bk $(HG_WG_CTAS=$c HG_WG_BK=$bk python tools/gemm_bench.py --shapes 0,3,5 2>&1 | python -c 'import json,sys; print([json.loads(l)["wgrad_nobias_us"] for l in sys.stdin.read().strip().splitlines()])' 2>&1 | tail -1)"
done; done > gpurun_out/r02/wgrad_sweep3.txt 2>&1
cat gpurun_out/r02/wgrad_sweep3.txt
