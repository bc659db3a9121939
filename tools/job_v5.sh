#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/v5_check.py small > gpurun_out/v5_small.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_small.txt
grep -q "ALL OK" gpurun_out/v5_small.txt || exit 0
timeout 300 python tools/v5_check.py > gpurun_out/v5_full.txt 2>&1; echo "rc=$?" >> gpurun_out/v5_full.txt
APAX_V5_RANK=0 timeout 300 python tools/v5_check.py > gpurun_out/v5_full_norank.txt 2>&1
TIMES_VARIANT=times5 TIMES_FN=apax_debug_cta_times5 timeout 300 python tools/cta_times.py cfg2 > gpurun_out/v5_times.txt 2>&1
