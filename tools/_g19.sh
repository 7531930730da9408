timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g19_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/g19_tests.log
