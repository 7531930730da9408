mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/g1_gputests.log 2>&1; echo tests_rc=$?
timeout 900 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g1_ref.json 2> gpurun_out/g1_ref.err; echo ref_rc=$?
tail -3 gpurun_out/g1_gputests.log
