cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_profiler.py tests/test_sharded_profile.py -x -q > gpurun_out/j18_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j18_pytest.log
timeout 900 python tools/time_profile.py gpurun_out/j18_profile.json > gpurun_out/j18_profile.log 2>&1
