timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g13_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/g13_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
