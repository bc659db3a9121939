cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/j3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j3_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/j3_bench.json 2> gpurun_out/j3_bench.err
APAX_ENC_SPLIT=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/j3_bench.json 2>> gpurun_out/j3_bench.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/j3_pytest_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j3_pytest_all.log
