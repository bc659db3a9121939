cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"encode|pack" --csv --log-file gpurun_out/j4_launches.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/j4_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_kernel" -s 3 -c 1 -o gpurun_out/j4_pack python bench.py --steps 2 --warmup 3 --profile > gpurun_out/j4_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_v3" -s 3 -c 1 -o gpurun_out/j4_chain python bench.py --steps 2 --warmup 3 --profile > gpurun_out/j4_ncu3.log 2>&1
