python bench.py > gpurun_out/bench_gcn.json 2> gpurun_out/bench_gcn.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmm_fast --csv --log-file gpurun_out/traffic_gat-rmat.csv python tools/ncu_target.py --workload gat-rmat --epochs 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_spmm_fast|k_sddmm_fast" -c 3 -o /tmp/rm python tools/ncu_spmm_rmat.py 128 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/rm.ncu-rep "RMAT-24 F=128 aggregation: unit kernel + packed kernel (hg_spmm)" > gpurun_out/ncu_rmat_spmm.md
timeout 900 ncu --set full --clock-control none -k regex:k_sddmm_fast -c 1 -o /tmp/sd python tools/ncu_sddmm_rmat.py 128 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/sd.ncu-rep "RMAT-24 F=128 4-head SDDMM, persistent teams" > gpurun_out/ncu_rmat_sddmm.md
