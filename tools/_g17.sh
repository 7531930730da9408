mkdir -p gpurun_out/r02
bash tools/exp/ab_bench.sh gcn-reddit eb2occ4 eb4occ4 > gpurun_out/r02/ab_spmm_eb_occ.jsonl 2>&1
bash tools/exp/ab_bench.sh gin-products eb2occ4 eb4occ4 >> gpurun_out/r02/ab_spmm_eb_occ.jsonl 2>&1
cat gpurun_out/r02/ab_spmm_eb_occ.jsonl
