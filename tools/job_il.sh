#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_il_graph.py > gpurun_out/il_graph.txt 2>&1
timeout 900 python -m pytest tests/test_k5.py tests/test_d3_errors.py tests/test_gpu_parity.py tests/test_range_decode.py tests/test_pipeline.py tests/test_cli.py -x -q -m gpu --timeout 300 > gpurun_out/il_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/il_pytest.log
timeout 600 python tools/fuzz_corrupt.py 300 7 > gpurun_out/il_fuzz.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/il_bench.json 2> gpurun_out/il_bench.err
