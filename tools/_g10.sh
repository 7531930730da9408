mkdir -p gpurun_out/r02
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r02/launch_gat-rmat_fused_warm.csv python tools/ncu_target.py --workload gat-rmat --epochs 3 > /dev/null 2>&1; echo ncu=$?
HG_FUSED_GAT=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r02/launch_gat-rmat_unfused_warm.csv python tools/ncu_target.py --workload gat-rmat --epochs 3 > /dev/null 2>&1; echo ncu=$?
