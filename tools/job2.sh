cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/j2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j2_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/j2_bench.json 2> gpurun_out/j2_bench.err
for w in cfg1 cfg3; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/j2_cfgs.json 2>> gpurun_out/j2_bench.err; done
timeout 900 python bench.py --workload cfg4 --shard-global --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j2_cfg4sg.json 2> gpurun_out/j2_cfg4sg.err
