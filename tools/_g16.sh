mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g16_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/g16_tests.log
timeout 900 python bench.py > gpurun_out/r02/bench_gcn_v3.json 2>gpurun_out/r02/bench_gcn_v3.err; echo gcn=$?
python -c "
import json; d=json.loads(open('gpurun_out/r02/bench_gcn_v3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step_eager'], d['e2e']['value'], d['gpu_launches'], d['parity'])"
export HG_KERNEL_LIST=gpurun_out/r02/kernels_step.txt; rm -f $HG_KERNEL_LIST
timeout 600 python -m pytest tests/test_gpu_models.py -m gpu -q -k dense_math > /dev/null 2>&1; echo kl=$?
